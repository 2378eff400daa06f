// Instantiation unit: 13,13 (one high-d kernel set per unit: parallel nvcc, see ops.h)
#include "inst.cuh"
template Ops make_ops<13, 13>();
