// match_tiled.cu — instantiations for train images larger than the shared-memory tile (see match_kernels.cuh):
// the min pass and the top-k pass over (query image, tile) pairs, and the merge + verification kernel.
#include "match_launch.cuh"

namespace chgpu {

template <int MODE>
static cudaError_t launch_tiled_mode(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    switch (P.L) {
        case 4: return launch_match_variant<true, 4, true, false, MODE>(P, smem, sm_count, stream, grid);
        case 6: return launch_match_variant<true, 6, true, false, MODE>(P, smem, sm_count, stream, grid);
        case 8: return launch_match_variant<true, 8, true, false, MODE>(P, smem, sm_count, stream, grid);
        default: break;
    }
    if (P.L < 4) return launch_match_variant<true, 4, false, false, MODE>(P, smem, sm_count, stream, grid);
    if (P.L < 6) return launch_match_variant<true, 6, false, false, MODE>(P, smem, sm_count, stream, grid);
    return launch_match_variant<true, 8, false, false, MODE>(P, smem, sm_count, stream, grid);
}

cudaError_t launch_match_tiled(const MatchParams& P, int mode, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    if (mode == kModeTileMin) return launch_tiled_mode<kModeTileMin>(P, smem, sm_count, stream, grid);  // never filtered
    if (P.fmats != nullptr)  // epipolar-guided top-k pass: the table slots of match_guided.cu
        return P.L == 6 ? launch_match_variant<true, 6, true, true, kModeTileTopK>(P, smem, sm_count, stream, grid)
                        : launch_match_variant<true, 8, false, true, kModeTileTopK>(P, smem, sm_count, stream, grid);
    return launch_tiled_mode<kModeTileTopK>(P, smem, sm_count, stream, grid);
}

cudaError_t launch_tile_compact(const MatchParams& P, uint32_t ntile_pairs, cudaStream_t stream) {
    if (ntile_pairs == 0) return cudaSuccess;
    tile_compact_kernel<0><<<ntile_pairs, 256, 0, stream>>>(P, ntile_pairs);
    return cudaGetLastError();
}

cudaError_t launch_tile_merge(const MatchParams& P, uint32_t npairs, uint32_t max_nq, cudaStream_t stream) {
    if (npairs == 0 || max_nq == 0) return cudaSuccess;
    const dim3 grid(npairs, (max_nq + kMergeChunk - 1) / kMergeChunk);
    tile_merge_kernel<0><<<grid, kMergeThreads, 0, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace chgpu
