// Instantiation unit: 7,7 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<7, 7>();
