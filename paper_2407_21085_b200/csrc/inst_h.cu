// Instantiation unit: 17,17 18,18 19,19 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<17, 17>();
template Ops make_ops<18, 18>();
template Ops make_ops<19, 19>();
