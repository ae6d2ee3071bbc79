// dense_pipe_c5.cu -- instantiation of dense_pipe.cuh: tile 2^11, chunk width 2^5,
// 3 groups x 4 warps, 6 stages.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg5, 11, 5, 4, 3, 6, 0)
}  // namespace ptdr
