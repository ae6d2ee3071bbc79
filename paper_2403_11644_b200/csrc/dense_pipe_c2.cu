// dense_pipe_c2.cu -- instantiation of dense_pipe.cuh: tile 2^11, chunk width 2^4,
// 4 groups x 4 warps, 6 stages.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg2, 11, 4, 4, 4, 6, 0)
}  // namespace ptdr
