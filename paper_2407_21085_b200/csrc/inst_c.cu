// Instantiation unit: 6,6 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<6, 6>();
