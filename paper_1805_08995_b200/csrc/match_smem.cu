// match_smem.cu — match kernel instantiations with the train image's codes in shared memory.
#include "match_launch.cuh"

namespace chgpu {
cudaError_t launch_match_smem(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    return launch_match_any<true>(P, smem, sm_count, stream, grid);
}
}  // namespace chgpu
