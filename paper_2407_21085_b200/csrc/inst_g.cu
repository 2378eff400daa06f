// Instantiation unit: 14,14 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<14, 14>();
