// Instantiation unit: 12,12 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<12, 12>();
