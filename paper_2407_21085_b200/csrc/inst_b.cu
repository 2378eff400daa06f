// Instantiation unit: 4,4 5,5 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<4, 4>();
template Ops make_ops<5, 5>();
