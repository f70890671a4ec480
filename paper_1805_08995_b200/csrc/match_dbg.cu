// match_dbg.cu — the match kernel's instantiations with the ranked-list output of the parity tests
// (chgpu_debug_ranked): the same source with DBG = true, so production launches carry no per-query pointer test.
#include "match_launch.cuh"

namespace chgpu {
cudaError_t launch_match_dbg(const MatchParams& P, bool smem_train, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    if (P.fmats != nullptr) {
        if (P.L == 6)
            return smem_train ? launch_match_variant<true, 6, true, true, kModeMatch, true>(P, smem, sm_count, stream, grid)
                              : launch_match_variant<false, 6, true, true, kModeMatch, true>(P, smem, sm_count, stream, grid);
        return smem_train ? launch_match_variant<true, 8, false, true, kModeMatch, true>(P, smem, sm_count, stream, grid)
                          : launch_match_variant<false, 8, false, true, kModeMatch, true>(P, smem, sm_count, stream, grid);
    }
    return smem_train ? launch_match_any<true, true>(P, smem, sm_count, stream, grid)
                      : launch_match_any<false, true>(P, smem, sm_count, stream, grid);
}
}  // namespace chgpu
