// compact_kernels.cuh — per-pair record offsets and the ordered compaction of the match
// kernel's per-query scratch into the reference's MatchRecord stream.
#pragma once

#include "dev_types.cuh"

namespace chgpu {

// Exclusive scan of per-pair match counts -> record offsets (one CTA; npairs is a sub-batch).
__global__ void scan_counts_kernel(const uint32_t* __restrict__ counts, uint32_t npairs,
                                   unsigned long long* __restrict__ offsets /* npairs + 1 */,
                                   DevStats* stats) {
    __shared__ unsigned long long s_warp[32];
    __shared__ unsigned long long s_carry;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < npairs; base += blockDim.x) {
        const uint32_t i = base + tid;
        const unsigned long long v = i < npairs ? counts[i] : 0;
        unsigned long long incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, d);
            if (int(lane) >= d) incl += u;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long u = __shfl_up_sync(0xffffffffu, w, d);
                if (int(lane) >= d) w += u;
            }
            s_warp[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before = s_carry + (warp ? s_warp[warp - 1] : 0);
        if (i < npairs) offsets[i] = before + incl - v;
        __syncthreads();
        if (tid == blockDim.x - 1) s_carry = before + incl;
        __syncthreads();
    }
    if (tid == 0) {
        offsets[npairs] = s_carry;
        atomicAdd(&stats->matches, s_carry);
    }
}

__device__ __forceinline__ unsigned long long mix64_dev(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// One CTA per pair: ordered compaction of the per-query scratch into MatchRecord{u32 q, u32 t, f64 d^2}
// (feature_io.hpp:51-57), ascending q, at most one per query (matcher.cpp:191-192).  A thread owns kCompactPer
// consecutive queries, so a pass over kCompactThreads * kCompactPer queries is one warp scan + one scan over the warps
// (three barriers) with every thread's loads in flight at once.  Measured per 4,096 pairs of 8,192 queries (scripts/exp4.sh):
// 512 x 4: 98 us, 256 x 4: 99, 512 x 2: 109, 1024 x 4: 114, 512 x 8: 129, 1024 x 8: 168, 512 x 16: 194 (the old one-query-per-
// thread kernel with serial scans: 329).
#ifndef CHGPU_COMPACT_PER
#define CHGPU_COMPACT_PER 4
#endif
#ifndef CHGPU_COMPACT_THREADS
#define CHGPU_COMPACT_THREADS 512
#endif
constexpr int kCompactPer = CHGPU_COMPACT_PER;
constexpr int kCompactThreads = CHGPU_COMPACT_THREADS;
__global__ void __launch_bounds__(kCompactThreads) compact_kernel(const PairDesc* __restrict__ pairs, const DevImage* __restrict__ images,
                                                       const uint2* __restrict__ res, const unsigned long long* __restrict__ offsets,
                                                       uint4* __restrict__ records, uint32_t first_pair_global, DevStats* stats) {
    __shared__ uint32_t s_warp[32];
    const uint32_t pair = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const PairDesc pd = pairs[pair];
    const uint32_t nq = images[pd.slot_i].n;
    uint4* out = records + offsets[pair];
    const uint2* __restrict__ in = res + pd.res_off;
    unsigned long long csum = 0;
    uint32_t base = 0;  // records written by earlier passes (every thread keeps its own copy)
    for (uint32_t q0 = 0; q0 < nq; q0 += blockDim.x * kCompactPer) {
        const uint32_t qa = q0 + tid * kCompactPer;
        uint2 r[kCompactPer];
        uint32_t mask = 0;
#pragma unroll
        for (int k = 0; k < kCompactPer; ++k) {
            r[k] = qa + k < nq ? __ldcs(in + qa + k) : make_uint2(kNone, 0u);
            if (r[k].x != kNone) mask |= 1u << k;
        }
        const uint32_t cnt = __popc(mask);
        uint32_t incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
            if (int(lane) >= d) incl += u;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < nwarps ? s_warp[lane] : 0u;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, w, d);
                if (int(lane) >= d) w += u;
            }
            s_warp[lane] = w;  // inclusive over the warps
        }
        __syncthreads();
        uint32_t pos = base + (warp ? s_warp[warp - 1] : 0u) + incl - cnt;
        base += s_warp[nwarps - 1];
#pragma unroll
        for (int k = 0; k < kCompactPer; ++k)
            if (mask & (1u << k)) {
                const uint32_t q = qa + k;
                const unsigned long long db = (unsigned long long)__double_as_longlong(double(r[k].y));
                out[pos++] = make_uint4(q, r[k].x, uint32_t(db), uint32_t(db >> 32));
                csum += mix64_dev(mix64_dev((unsigned long long)(first_pair_global + pair) << 32 | q) ^
                                  ((unsigned long long)r[k].x << 32 | r[k].y));
            }
        __syncthreads();  // s_warp is rewritten by the next pass
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, d);
    if (lane == 0 && csum) atomicAdd(&stats->checksum, csum);
}

}  // namespace chgpu
