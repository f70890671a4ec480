// match_kernels.cuh — K3 (pair matching) and the ordered compaction of its results.
//
// K3 is a persistent kernel: one CTA per SM pulls work units (pair, query range) from a global
// counter.  For each unit the train image's 128-bit codes are brought into shared memory with
// one bulk async copy (cp.async.bulk + mbarrier, the sm_90+/sm_100 TMA path), then every warp
// owns one query point at a time:
//
//   1. bucket lookup   : lanes t < L read the query's table-t code and the two CSR offsets of
//                        that bucket in the train image; a warp scan flattens the L buckets
//                        into one index space [0, R)                     (matcher.cpp:164-169)
//   2. Hamming scan    : lane l evaluates raw candidates l, l+32, ...; key = distance<<24 | id
//                        (train code gathered from shared memory, 4x LOP3 + 4x POPC)
//                                                                         (matcher.cpp:68-84)
//   3. ranking         : the ranked list is the first n keys in ascending (distance, id) order
//                        with EQUAL KEYS COLLAPSED — the same point reached through several
//                        tables has the same key, so the reference's sort+unique
//                        (matcher.cpp:170-171) is implicit.  Keys are pulled one at a time with
//                        a warp-wide REDUX.MIN over "keys greater than the previous one"; the
//                        threshold tau and the re-rank fallback (matcher.cpp:176-189) only
//                        decide where the pulling stops, so no histogram has to be stored.
//   4. verification    : 8 lanes per candidate row, __vabsdiffu4 + __dp4a (exact u32 squared
//                        distance), best / second with rank-order tie-break, Lowe ratio in
//                        fp64 exactly as matcher.cpp:115-137.
//
// Results go to a per-query scratch (train id, d^2); compact_kernel turns them into the
// reference's MatchRecord stream, ascending query index inside every pair.
#pragma once

#include "dev_types.cuh"

namespace chgpu {

constexpr int kMatchThreads = 1024;
constexpr int kKeySlots = 10;  // 320 raw candidates per pass (max observed 309 at N=8192, L=6, m=8)

struct MatchParams {
    const DevImage* images;
    const PairDesc* pairs;
    uint2* res;                 // per query: (train id | kNone, d^2)
    uint32_t* pair_counts;      // matches per pair
    DevStats* stats;
    unsigned int* unit_counter;
    uint32_t nunits;
    uint32_t chunks_per_pair;
    uint32_t m, L;
    uint32_t top_k, tau, min_ranked, long_bits;
    double ratio_sq;            // cfg.ratio * cfg.ratio, formed on the host in fp64
    uint32_t* dbg_ranked;       // optional: n_i x top_k
    uint32_t* dbg_count;        // optional: n_i
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// Bulk global -> shared copy completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ uint32_t hamming128(const uint4& a, const uint4& b) {
    return __popc(a.x ^ b.x) + __popc(a.y ^ b.y) + __popc(a.z ^ b.z) + __popc(a.w ^ b.w);
}

// Sum over 4 byte lanes of (a_i - b_i)^2, exact in u32.
__device__ __forceinline__ uint32_t sqdiff4(uint32_t a, uint32_t b) {
    const uint32_t ad = __vabsdiffu4(a, b);
    return __dp4a(ad, ad, 0u);
}

// Smallest key strictly greater than `prev` over the warp's key slots (+ one extra slot).
template <int SLOTS>
__device__ __forceinline__ uint32_t next_key(const uint32_t (&key)[SLOTS], uint32_t extra, uint32_t prev,
                                             bool first) {
    uint32_t lmin = kNone;
#pragma unroll
    for (int i = 0; i < SLOTS; ++i) {
        const uint32_t k = key[i];
        if (first || k > prev) lmin = min(lmin, k);
    }
    if (first || extra > prev) lmin = min(lmin, extra);
    return __reduce_min_sync(0xffffffffu, lmin);
}

template <bool SMEM_TRAIN, int LT>
__global__ void __launch_bounds__(kMatchThreads, 1) match_kernel(const MatchParams P) {
    extern __shared__ __align__(16) uint4 s_long[];
    __shared__ unsigned int s_unit;
    __shared__ __align__(8) uint64_t s_bar;

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t kWarps = kMatchThreads / 32;
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t nb1 = (1u << P.m) + 1;

    if (SMEM_TRAIN && tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t bar_parity = 0;
    uint32_t resident = kNone;

    // per-warp statistics, flushed once per unit
    for (;;) {
        if (tid == 0) s_unit = atomicAdd(P.unit_counter, 1u);
        __syncthreads();
        const uint32_t unit = s_unit;
        if (unit >= P.nunits) break;
        const uint32_t pair = unit / P.chunks_per_pair, chunk = unit % P.chunks_per_pair;
        const PairDesc pd = P.pairs[pair];
        const DevImage I = P.images[pd.slot_i];
        const DevImage J = P.images[pd.slot_j];

        if (SMEM_TRAIN && resident != pd.slot_j && J.n != 0) {
            if (tid == 0) {
                // generic-proxy reads of the previous train image are complete (barrier below);
                // order them before the async-proxy writes.
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint32_t bytes = J.n * 16u;
                mbar_expect_tx(&s_bar, bytes);
                for (uint32_t off = 0; off < bytes; off += 65536u)
                    bulk_g2s(reinterpret_cast<unsigned char*>(s_long) + off,
                             reinterpret_cast<const unsigned char*>(J.longs) + off, min(65536u, bytes - off), &s_bar);
            }
            mbar_wait(&s_bar, bar_parity);
            bar_parity ^= 1;
            resident = pd.slot_j;
        }

        // query range of this unit: chunks are multiples of 32 queries
        const uint32_t qc = (((I.n + P.chunks_per_pair - 1) / P.chunks_per_pair) + 31u) & ~31u;
        const uint32_t q0 = min(I.n, chunk * qc), q1 = min(I.n, q0 + qc);

        uint32_t st_raw = 0, st_vq = 0, st_dist = 0, st_match = 0;

        for (uint32_t q = q0 + warp; q < q1; q += kWarps) {
            uint32_t out_t = kNone, out_d = 0;
            if (J.n != 0) {
                // ---- 1. bucket lookup ------------------------------------------------------
                uint32_t lo = 0, len = 0;
                if (lane < P.L) {
                    const uint32_t code = __ldg(I.shorts + uint64_t(q) * P.L + lane);
                    const uint32_t* o = J.offs + lane * nb1 + code;
                    lo = __ldg(o);
                    len = __ldg(o + 1) - lo;
                }
                uint32_t incl = len;
#pragma unroll
                for (int d = 1; d < LT; d <<= 1) {
                    const uint32_t u = __shfl_up_sync(FULL, incl, d);
                    if (int(lane) >= d) incl += u;
                }
                const uint32_t R = __shfl_sync(FULL, incl, LT - 1);
                const uint32_t excl = incl - len;
                const uint32_t bias = lane * J.n + lo - excl;  // flat index r -> points[r + bias]
                uint32_t pre[LT], bs[LT];
#pragma unroll
                for (int t = 0; t < LT; ++t) {
                    pre[t] = __shfl_sync(FULL, excl, t);
                    bs[t] = __shfl_sync(FULL, bias, t);
                }
                st_raw += R;

                if (R != 0) {
                    const uint4 ql = __ldg(I.longs + q);
                    uint32_t mykey = kNone;  // lane r holds the r-th ranked key
                    uint32_t n = 0;          // ranked count
                    uint32_t wmax = 0;       // multi-pass only: largest key seen
                    const bool single = R <= 32u * kKeySlots;

                    for (uint32_t base = 0; base < R; base += 32u * kKeySlots) {
                        // ---- 2. Hamming scan ------------------------------------------------
                        uint32_t key[kKeySlots];
#pragma unroll
                        for (int it = 0; it < kKeySlots; ++it) {
                            key[it] = kNone;
                            const uint32_t rb = base + it * 32u;
                            if (rb < R) {  // warp-uniform
                                // lanes past the end re-evaluate the last candidate: equal keys collapse
                                const uint32_t r = min(rb + lane, R - 1);
                                uint32_t b = bs[0];
#pragma unroll
                                for (int t = 1; t < LT; ++t)
                                    if (r >= pre[t]) b = bs[t];
                                const uint32_t id = __ldg(J.points + (r + b));
                                uint4 c;
                                if (SMEM_TRAIN) c = s_long[id];
                                else c = __ldg(J.longs + id);
                                key[it] = (hamming128(c, ql) << 24) | id;
                            }
                        }
                        // ---- 3. ranking -----------------------------------------------------
                        if (single) {
                            uint32_t k0 = next_key(key, kNone, 0u, true);
                            if ((k0 >> 24) <= P.tau) {
                                if (lane == 0) mykey = k0;
                                n = 1;
                                bool fallback = false;
                                uint32_t prev = k0;
                                while (n < P.top_k) {
                                    const uint32_t nk = next_key(key, kNone, prev, false);
                                    if (nk == kNone) break;
                                    if (!fallback && (nk >> 24) > P.tau) {
                                        if (n >= P.min_ranked) break;
                                        fallback = true;  // threshold cut something and the ranking is too small
                                    }
                                    if (lane == n) mykey = nk;
                                    ++n;
                                    prev = nk;
                                }
                            }
                        } else {
                            // merge this pass into the running top-k (ascending, unique)
                            uint32_t lmax = 0;
#pragma unroll
                            for (int it = 0; it < kKeySlots; ++it)
                                if (key[it] != kNone) lmax = max(lmax, key[it]);
                            wmax = max(wmax, __reduce_max_sync(FULL, lmax));
                            const uint32_t old = mykey;
                            uint32_t prev = 0;
                            mykey = kNone;
                            for (uint32_t r = 0; r < P.top_k; ++r) {
                                const uint32_t nk = next_key(key, old, prev, r == 0);
                                if (nk == kNone) break;
                                if (lane == r) mykey = nk;
                                prev = nk;
                            }
                        }
                    }
                    if (!single) {
                        // thresholded size s, unique total (<= k); fallback rule as in the single-pass path
                        const uint32_t total = __popc(__ballot_sync(FULL, mykey != kNone));
                        const uint32_t s = __popc(__ballot_sync(FULL, mykey != kNone && (mykey >> 24) <= P.tau));
                        const bool anycut = (wmax >> 24) > P.tau;
                        if (s == 0) n = 0;
                        else if (s >= P.min_ranked || !anycut) n = s;
                        else n = total;
                    }

                    if (P.dbg_ranked != nullptr) {
                        if (lane < n) P.dbg_ranked[uint64_t(q) * P.top_k + lane] = mykey & 0xffffffu;
                        if (lane == 0) P.dbg_count[q] = n;
                    }

                    // ---- 4. verification (euclidean_verify, matcher.cpp:115-137) ----------
                    if (n >= 2) {
                        st_vq += 1;
                        st_dist += n;
                        const uint32_t sub = lane & 7, grp = lane >> 3;
                        const uint4 qa = __ldg(reinterpret_cast<const uint4*>(I.desc + uint64_t(q) * kDim) + sub);
                        uint32_t mydist = kNone;
                        for (uint32_t j0 = 0; j0 < n; j0 += 4) {
                            const uint32_t j = min(j0 + grp, n - 1);
                            const uint32_t id = __shfl_sync(FULL, mykey, j) & 0xffffffu;
                            const uint4 ta = __ldg(reinterpret_cast<const uint4*>(J.desc + uint64_t(id) * kDim) + sub);
                            uint32_t s = sqdiff4(qa.x, ta.x) + sqdiff4(qa.y, ta.y) + sqdiff4(qa.z, ta.z) +
                                         sqdiff4(qa.w, ta.w);
                            s += __shfl_xor_sync(FULL, s, 1);
                            s += __shfl_xor_sync(FULL, s, 2);
                            s += __shfl_xor_sync(FULL, s, 4);
                            const uint32_t v = __shfl_sync(FULL, s, ((lane - j0) & 3u) * 8u);
                            if (lane >= j0 && lane < j0 + 4 && lane < n) mydist = v;
                        }
                        // best = smallest d^2, ties to the earlier rank (strict '<' in the reference loop)
                        const uint32_t packed = lane < n ? ((mydist << 8) | lane) : kNone;
                        const uint32_t bestp = __reduce_min_sync(FULL, packed);
                        const uint32_t bl = bestp & 0xffu, best = bestp >> 8;
                        const uint32_t second = __reduce_min_sync(FULL, (lane < n && lane != bl) ? mydist : kNone);
                        const uint32_t bid = __shfl_sync(FULL, mykey, bl) & 0xffffffu;
                        if (second != 0u && double(best) < __dmul_rn(P.ratio_sq, double(second))) {
                            out_t = bid;
                            out_d = best;
                            st_match += 1;
                        }
                    }
                }
            }
            if (lane == 0) P.res[pd.res_off + q] = make_uint2(out_t, out_d);
        }

        if (lane == 0) {
            if (st_raw) atomicAdd(&P.stats->raw_candidates, (unsigned long long)st_raw);
            if (st_vq) atomicAdd(&P.stats->verified_queries, (unsigned long long)st_vq);
            if (st_dist) atomicAdd(&P.stats->distances, (unsigned long long)st_dist);
            if (st_match) atomicAdd(&P.pair_counts[pair], st_match);
        }
        __syncthreads();  // all warps done with s_long / s_unit before the next unit
    }
}

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
// (feature_io.hpp:51-57), ascending q, at most one per query (matcher.cpp:191-192).
__global__ void compact_kernel(const PairDesc* __restrict__ pairs, const DevImage* __restrict__ images,
                               const uint2* __restrict__ res, const unsigned long long* __restrict__ offsets,
                               uint4* __restrict__ records, uint32_t first_pair_global, DevStats* stats) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_base;
    const uint32_t pair = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const PairDesc pd = pairs[pair];
    const uint32_t nq = images[pd.slot_i].n;
    if (tid == 0) s_base = 0;
    __syncthreads();
    uint4* out = records + offsets[pair];
    unsigned long long csum = 0;
    for (uint32_t q0 = 0; q0 < nq; q0 += blockDim.x) {
        const uint32_t q = q0 + tid;
        uint2 r = make_uint2(kNone, 0);
        if (q < nq) r = res[pd.res_off + q];
        const bool hit = r.x != kNone;
        const uint32_t bal = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        uint32_t before = s_base;
        for (uint32_t w = 0; w < warp; ++w) before += s_warp[w];
        if (hit) {
            const uint32_t pos = before + __popc(bal & ((1u << lane) - 1u));
            const unsigned long long db = (unsigned long long)__double_as_longlong(double(r.y));
            out[pos] = make_uint4(q, r.x, uint32_t(db), uint32_t(db >> 32));
            csum += mix64_dev(mix64_dev((unsigned long long)(first_pair_global + pair) << 32 | q) ^
                              ((unsigned long long)r.x << 32 | r.y));
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t tot = 0;
            for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) tot += s_warp[w];
            s_base += tot;
        }
        __syncthreads();
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, d);
    if (lane == 0 && csum) atomicAdd(&stats->checksum, csum);
}

}  // namespace chgpu
