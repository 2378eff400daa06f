// Instantiation unit: 18,18 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<18, 18>();
