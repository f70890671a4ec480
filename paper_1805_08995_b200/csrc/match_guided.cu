// match_guided.cu — epipolar-guided instantiations of the match kernel.
#include "match_launch.cuh"

namespace chgpu {
cudaError_t launch_match_guided(const MatchParams& P, bool smem_train, size_t smem, int sm_count, cudaStream_t stream,
                                uint32_t* grid) {
    if (P.L == 6)
        return smem_train ? launch_match_variant<true, 6, true, true>(P, smem, sm_count, stream, grid)
                          : launch_match_variant<false, 6, true, true>(P, smem, sm_count, stream, grid);
    return smem_train ? launch_match_variant<true, 8, false, true>(P, smem, sm_count, stream, grid)
                      : launch_match_variant<false, 8, false, true>(P, smem, sm_count, stream, grid);
}
}  // namespace chgpu
