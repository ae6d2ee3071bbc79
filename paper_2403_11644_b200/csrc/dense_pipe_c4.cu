// dense_pipe_c4.cu -- instantiation of dense_pipe.cuh: tile 2^12, chunk width 2^5,
// 2 groups x 8 warps, 3 stages.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg4, 12, 5, 8, 2, 3, 0)
}  // namespace ptdr
