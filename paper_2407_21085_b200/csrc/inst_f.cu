// Instantiation unit: 11,11 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<11, 11>();
