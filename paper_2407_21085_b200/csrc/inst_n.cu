// Instantiation unit: 19,19 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<19, 19>();
