// Instantiation unit: 17,17 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<17, 17>();
