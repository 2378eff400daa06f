// Instantiation unit: 1,1 2,2 3,3 1,2 2,1 2,3 3,2 (generated layout, see ops.h)
#include "inst.cuh"
template Ops make_ops<1, 1>();
template Ops make_ops<2, 2>();
template Ops make_ops<3, 3>();
template Ops make_ops<1, 2>();
template Ops make_ops<2, 1>();
template Ops make_ops<2, 3>();
template Ops make_ops<3, 2>();
