// dense_pipe_c3.cu -- instantiation of dense_pipe.cuh: tile 2^11, chunk width 2^4,
// 3 groups x 4 warps, 6 stages.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg3, 11, 4, 4, 3, 6, 0)
}  // namespace ptdr
