// dense_mode2.cu -- instantiation of the dense path for MODE 2 (see dense_impl.cuh).
#include "dense_launch.cuh"
PTDR_DEFINE_DENSE_MODE(2)
