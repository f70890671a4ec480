// match_launch.cuh — launchers of the match kernel's instantiations.  The shared-memory and the
// global-gather variants live in separate translation units (match_smem.cu, match_global.cu)
// so that nvcc compiles them in parallel.
#pragma once

#include "match_kernels.cuh"

namespace chgpu {

// Launches match_kernel<SMEM_TRAIN, LT, EXACT> for P.L tables on `stream` as a persistent grid
// (one CTA per SM at most, never more CTAs than units).  smem = dynamic shared memory bytes.
cudaError_t launch_match_smem(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid);
cudaError_t launch_match_global(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid);
// Epipolar-guided instantiations (match_guided.cu): L == 6 exact, any other L through the LT = 8 generic.
cudaError_t launch_match_guided(const MatchParams& P, bool smem_train, size_t smem, int sm_count, cudaStream_t stream,
                                uint32_t* grid);
// The same kernels instantiated with the parity tests' ranked-list output (P.dbg_ranked / P.dbg_count; match_dbg.cu).
cudaError_t launch_match_dbg(const MatchParams& P, bool smem_train, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid);
// Tiled train images (match_tiled.cu): mode = kModeTileMin / kModeTileTopK over (query image, tile) pairs with the
// tile's codes in shared memory, then the per-query merge + verification over the original pairs.
cudaError_t launch_match_tiled(const MatchParams& P, int mode, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid);
cudaError_t launch_tile_compact(const MatchParams& P, uint32_t ntile_pairs, cudaStream_t stream);  // P.pairs = tile pairs
cudaError_t launch_tile_merge(const MatchParams& P, uint32_t npairs, uint32_t max_nq, cudaStream_t stream);
// The match kernel over the hit queries the join pass listed (P.act / P.nact; match_active.cu): train codes in shared memory.
cudaError_t launch_match_active(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid);
// Table slots (LT) the launchers pick for L tables; the staging area is sized with it.
inline int match_table_slots(uint32_t L, bool guided) { return guided ? (L == 6 ? 6 : 8) : (L <= 4 ? 4 : (L <= 6 ? 6 : 8)); }

template <bool SMEM, int LT, bool EXACT, bool GUIDED = false, int MODE = kModeMatch, bool DBG = false>
cudaError_t launch_match_variant(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid_out) {
    auto kfn = match_kernel<SMEM, LT, EXACT, GUIDED, MODE, DBG>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kMatchThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    const uint32_t cap = uint32_t(per_sm) * uint32_t(sm_count);
    const uint32_t grid = P.nunits < cap ? P.nunits : cap;
    *grid_out = grid;
    kfn<<<grid, kMatchThreads, smem, stream>>>(P);
    return cudaGetLastError();
}

template <bool SMEM, bool DBG = false, int MODE = kModeMatch>
cudaError_t launch_match_any(const MatchParams& P, size_t smem, int sm_count, cudaStream_t stream, uint32_t* grid) {
    switch (P.L) {
        case 4: return launch_match_variant<SMEM, 4, true, false, MODE, DBG>(P, smem, sm_count, stream, grid);
        case 6: return launch_match_variant<SMEM, 6, true, false, MODE, DBG>(P, smem, sm_count, stream, grid);
        case 8: return launch_match_variant<SMEM, 8, true, false, MODE, DBG>(P, smem, sm_count, stream, grid);
        default: break;
    }
    if (P.L < 4) return launch_match_variant<SMEM, 4, false, false, MODE, DBG>(P, smem, sm_count, stream, grid);
    if (P.L < 6) return launch_match_variant<SMEM, 6, false, false, MODE, DBG>(P, smem, sm_count, stream, grid);
    return launch_match_variant<SMEM, 8, false, false, MODE, DBG>(P, smem, sm_count, stream, grid);
}

}  // namespace chgpu
