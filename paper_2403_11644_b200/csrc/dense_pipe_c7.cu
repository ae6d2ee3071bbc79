// dense_pipe_c7.cu -- instantiation of dense_pipe.cuh: tile 2^11, chunk width 2^4,
// 4 groups x 4 warps, 4 stages, early stage release with 2 exchange rounds.
#include "dense_pipe.cuh"
namespace ptdr {
PTDR_DEFINE_PIPE_CFG(pipe_cfg7, 11, 4, 4, 4, 4, 2)
}  // namespace ptdr
