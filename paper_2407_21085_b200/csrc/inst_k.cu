// Instantiation unit: 15,15 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<15, 15>();
