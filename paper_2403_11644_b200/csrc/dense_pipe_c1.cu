// dense_pipe_c1.cu -- instantiation of dense_pipe.cuh: tile 2^12, chunk width 2^4,
// 2 groups x 8 warps, 3 stages.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg1, 12, 4, 8, 2, 3, 0)
}  // namespace ptdr
