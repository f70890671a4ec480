// match_active.cu — the match kernel over the queries the join pass (join_kernels.cuh) found a candidate within tau for.
#include "match_launch.cuh"

namespace chgpu {
cudaError_t launch_match_active(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    if (P.fmats != nullptr) {  // epipolar-guided (the join's hit test is the unfiltered one: a superset, the band comes after)
        if (P.L == 6) return launch_match_variant<true, 6, true, true, kModeMatchActive>(P, smem, sm_count, stream, grid);
        return launch_match_variant<true, 8, false, true, kModeMatchActive>(P, smem, sm_count, stream, grid);
    }
    return launch_match_any<true, false, kModeMatchActive>(P, smem, sm_count, stream, grid);
}
}  // namespace chgpu
