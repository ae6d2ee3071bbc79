// dense_mode0.cu -- instantiation of the dense path for MODE 0 (see dense_impl.cuh).
#include "dense_launch.cuh"
PTDR_DEFINE_DENSE_MODE(0)
