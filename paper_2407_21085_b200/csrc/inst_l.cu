// Instantiation unit: 16,16 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<16, 16>();
