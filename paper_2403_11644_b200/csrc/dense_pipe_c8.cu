// dense_pipe_c8.cu -- instantiation of dense_pipe.cuh: tile 2^12, chunk width 2^4,
// 2 groups x 8 warps, 2 stages, early stage release with 2 exchange rounds.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg8, 12, 4, 8, 2, 2, 2)
}  // namespace ptdr
