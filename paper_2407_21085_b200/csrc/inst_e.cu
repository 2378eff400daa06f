// Instantiation unit: 8,8 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<8, 8>();
