// match_global.cu — match kernel instantiations that gather the train image's codes from
// global memory / L2 (images too large for one SM's shared memory).
#include "match_launch.cuh"

namespace chgpu {
cudaError_t launch_match_global(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    return launch_match_any<false>(P, smem, sm_count, stream, grid);
}
}  // namespace chgpu
