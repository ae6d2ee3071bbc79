// dense_mode4.cu -- instantiation of the dense path for MODE 4 (see dense_impl.cuh).
#include "dense_launch.cuh"
PTDR_DEFINE_DENSE_MODE(4)
