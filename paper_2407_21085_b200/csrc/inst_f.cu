// Instantiation unit: 11,11 12,12 13,13 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<11, 11>();
template Ops make_ops<12, 12>();
template Ops make_ops<13, 13>();
