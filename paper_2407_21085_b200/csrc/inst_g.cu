// Instantiation unit: 14,14 15,15 16,16 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<14, 14>();
template Ops make_ops<15, 15>();
template Ops make_ops<16, 16>();
