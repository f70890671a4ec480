// general_kernels.cuh — KG, the general match path: everything the reference accepts and the tuned kernels (K3, K3j, the
// tiles) are not laid out for.
//
//   * short codes of 13..32 bits (hashing.cpp:30-36 allows 1..32): a dense 2^m + 1 offset table per image does not exist
//     for them.  The bucket index of such an image is the reference's own form (build_bucket_index, matcher.cpp:27-51:
//     the points of a table sorted by (code, point)), stored as one u64 key  code << 16 | point  per entry and searched
//     by bisection (BucketIndex::bucket, matcher.cpp:19-25) — sparse_index_kernel builds it with a sorting network.
//   * top_k > 32 (validate, matcher.cpp:9-17 asks for >= 2 only): the tuned kernels keep the ranked list one entry per
//     lane.  Here the list is never stored: every ranked key is verified the moment it is pulled.
//   * match_pair_filtered with a HOST callback (matcher.hpp:92-105, hook matcher.cpp:172): the candidate lists of a pair
//     are formed on the device (cand_union_kernel: concatenate the L buckets, sort, unique — matcher.cpp:164-171), handed
//     to the caller's filter on the host, and whatever comes back is ranked and verified on the device from the explicit
//     lists.  The reference ranks such a list with a stable counting sort (fill_histogram, matcher.cpp:68-84): ties in
//     the distance keep the ORDER OF THE LIST, duplicates stay — so the key is  distance << 24 | position.
//
// One warp per query.  A candidate's key is  distance << 24 | id  (buckets; the same point reached through several
// tables has the same key, so pulling keys in strictly ascending order is the reference's sort + unique) or
// distance << 24 | position (explicit lists).  The ranked list is the first keys in ascending order, cut by the threshold
// and re-ranked without it by the rule of matcher.cpp:176-189; each is verified as it is pulled (euclidean_verify,
// matcher.cpp:115-137: exact integer distances, best / second with strict '<', Lowe ratio in fp64).  Keys are kept in a
// per-warp shared-memory cache when the query has at most kGenCacheKeys candidates and recomputed per pull otherwise.
// Lightly tuned (KG): this path exists so that no input the reference accepts fails on the device.
#pragma once

#include "match_kernels.cuh"

namespace chgpu {

constexpr int kGenThreads = 256;
constexpr uint32_t kGenWarps = kGenThreads / 32;
constexpr uint32_t kGenCacheKeys = 1024;  // per warp: 4 KB (32 KB per CTA: the occupancy of this latency-bound kernel matters more)
#ifndef CHGPU_GEN_CHAINS
#define CHGPU_GEN_CHAINS 4
#endif
constexpr uint32_t kGenChains = CHGPU_GEN_CHAINS;  // independent id -> code gather chains per lane while the keys are formed
constexpr uint32_t kGenBitmapWords = kMaxPoints / 32;  // cand_union_kernel: one bit per train point, per warp

struct GeneralParams {
    MatchParams base;  // images, pairs, res, pair_counts, stats, m, L, top_k, tau, min_ranked, ratio_sq, fmats, band_px, dbg_*
    uint32_t npairs;
    unsigned long long queries;            // of the sub-batch (PairDesc::res_off indexes them)
    uint32_t sparse;                       // the images carry sorted (code, point) keys instead of dense offsets
    uint32_t slice;                        // consecutive queries a warp takes per visit
    const unsigned long long* list_offs;   // explicit candidate lists of ONE pair: n_i + 1 offsets into list_ids, or nullptr
    const uint32_t* list_ids;
};

// The L bucket ranges of one query in the train image's index: table t covers entries [first_t, first_t + len_t) of the
// image's entry array (points / sorted keys, table-major).  Lane t resolves table t.  Kept in the form the flat candidate
// index needs: start[t] = len_0 + ... + len_(t-1) (the flat index of the table's first candidate), shift[t] = first_t - start[t].
struct BucketRanges {
    uint32_t start[kMaxTables], shift[kMaxTables];
    uint32_t total;
};
__device__ __forceinline__ BucketRanges resolve_ranges(const DevImage& I, const DevImage& J, uint32_t q, uint32_t L, uint32_t m,
                                                       bool sparse, uint32_t lane) {
    constexpr uint32_t FULL = 0xffffffffu;
    uint32_t a = 0, n = 0;
    if (lane < L) {
        const uint32_t code = __ldg(I.shorts + uint64_t(q) * L + lane);
        if (!sparse) {
            const uint32_t* o = J.offs + uint64_t(lane) * ((1u << m) + 1u) + code;
            a = __ldg(o);
            n = __ldg(o + 1) - a;
        } else {
            // BucketIndex::bucket (matcher.cpp:19-25) on the sorted keys: entries with this code form one run
            const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(J.offs) + uint64_t(lane) * J.n;
            const unsigned long long lo_key = (unsigned long long)code << 16, hi_key = lo_key | 0xffffull;
            uint32_t lo = 0, hi = J.n;
            while (lo < hi) {  // first entry >= lo_key
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(keys + mid) < lo_key) lo = mid + 1;
                else hi = mid;
            }
            a = lo;
            // first entry > hi_key: runs are short (n / 2^m points on average), so gallop from the start of the run
            // and bisect the last stride instead of bisecting the whole table again
            uint32_t step = 1;
            while (a + step <= J.n && __ldg(keys + a + step - 1) <= hi_key) step <<= 1;   // entry a + step - 1 is past the run
            lo = a + (step >> 1);                       // entries below lo belong to the run (or lo == a: maybe empty)
            hi = min(a + step - 1, J.n);                // entry hi is past the run (or the end of the table)
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(keys + mid) <= hi_key) lo = mid + 1;
                else hi = mid;
            }
            n = lo - a;
        }
        a += lane * J.n;
    }
    BucketRanges r;
    r.total = 0;
#pragma unroll
    for (int t = 0; t < kMaxTables; ++t) {
        r.start[t] = r.total;  // tables past L: start == total, never reached by an index below total
        r.shift[t] = __shfl_sync(FULL, a, t) - r.total;
        r.total += uint32_t(t) < L ? __shfl_sync(FULL, n, t) : 0u;
    }
    return r;
}
// point id behind flat candidate index i (< r.total) of the concatenated buckets
__device__ __forceinline__ uint32_t range_id(const BucketRanges& r, const DevImage& J, bool sparse, uint32_t i) {
    uint32_t shift = r.shift[0];  // the last table whose first candidate is not past i
#pragma unroll
    for (int t = 1; t < kMaxTables; ++t)
        if (i >= r.start[t]) shift = r.shift[t];
    const uint32_t e = i + shift;
    if (sparse) return uint32_t(__ldg(reinterpret_cast<const unsigned long long*>(J.offs) + e) & 0xffffull);
    return __ldg(J.points + e);
}

// pair whose queries contain entry g of the sub-batch's query space (PairDesc::res_off ascending; pairs without queries
// share their successor's offset and are skipped by taking the LAST pair with res_off <= g)
__device__ __forceinline__ uint32_t pair_of_query(const PairDesc* __restrict__ pairs, uint32_t npairs, unsigned long long g) {
    uint32_t lo = 0, hi = npairs;  // last k with res_off <= g
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pairs[mid].res_off <= g) lo = mid;
        else hi = mid;
    }
    return lo;
}

// HEADS: the pulls of a query with 33..256 keys come from per-lane sorted lists (below); false = the A/B reference.
// LISTS / SPARSE / GUIDED: explicit candidate lists, the sorted-key index, the epipolar band — build-time, because the
// per-key code otherwise re-tests them (ncu: ~100 of 1,530 instructions per query were branches on these three flags)
template <bool HEADS, bool LISTS, bool SPARSE, bool GUIDED>
__global__ void __launch_bounds__(kGenThreads, 4) general_match_kernel(const GeneralParams G) {
    extern __shared__ __align__(16) uint32_t s_keys_all[];  // kGenWarps x kGenCacheKeys
    constexpr uint32_t FULL = 0xffffffffu;
    const MatchParams& P = G.base;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the warp's key cache by 32-bit shared-window address, pinned in a register (the compiler otherwise re-derives the
    // window base in front of every access: 7 instructions per key read)
    uint32_t s_keys = smem_addr(s_keys_all + warp * kGenCacheKeys);
    asm volatile("" : "+r"(s_keys));
    constexpr bool explicit_lists = LISTS, sparse = SPARSE, guided = GUIDED;

    // every warp takes a contiguous run of the sub-batch's queries in short slices: the pair (and its two image records)
    // changes rarely along a run, so it is looked up once and then only advanced
    const unsigned long long total_warps = (unsigned long long)gridDim.x * kGenWarps;
    const unsigned long long my_warp = (unsigned long long)blockIdx.x * kGenWarps + warp;
    const unsigned long long kSlice = G.slice;  // queries per visit (host: 1..8, shorter when the sub-batch is small)
    // statistics of the queries of one visit (<= 8 queries of at most L n = 2^19 candidates each; uniform over the lanes)
    uint32_t st_raw = 0, st_vq = 0, st_dist = 0;
    uint32_t pair = kNone;
    PairDesc pd{};
    DevImage I{}, J{};
    unsigned long long pair_end = 0;  // first query past the current pair
    for (unsigned long long g0 = my_warp * kSlice; g0 < G.queries; g0 += total_warps * kSlice) {
    for (unsigned long long g = g0; g < min(g0 + kSlice, G.queries); ++g) {
        if (pair == kNone || g >= pair_end || g < pd.res_off) {
            pair = pair_of_query(P.pairs, G.npairs, g);
            pd = P.pairs[pair];
            I = P.images[pd.slot_i];
            J = P.images[pd.slot_j];
            pair_end = pd.res_off + I.n;
        }
        const uint32_t q = uint32_t(g - pd.res_off);
        uint32_t out_t = kNone, out_d = 0, n = 0;
        if (J.n != 0) {
            const uint4 ql = __ldg(I.longs + q);
            BucketRanges r{};
            unsigned long long list_lo = 0;
            uint32_t C;
            if (explicit_lists) {
                list_lo = G.list_offs[q];
                C = uint32_t(G.list_offs[q + 1] - list_lo);
            } else {
                r = resolve_ranges(I, J, q, P.L, P.m, sparse, lane);
                C = r.total;
                st_raw += C;  // matcher.cpp:168 (lane 0 adds the visit's total once)
            }
            EpiLine line{};
            if (guided) line = epipolar_band(P.fmats + uint64_t(pd.pair_idx) * 9, __ldg(I.kp + q));
            auto id_of = [&](uint32_t i) -> uint32_t {
                return explicit_lists ? __ldg(G.list_ids + list_lo + i) : range_id(r, J, sparse, i);
            };
            auto key_at = [&](uint32_t i) -> uint32_t {
                const uint32_t id = id_of(i);
                const uint32_t d = hamming128(__ldg(J.longs + id), ql);
                uint32_t key = (d << 24) | (explicit_lists ? i : id);
                if (guided) key = band_filter(key, line, J.kp, P.band_px);
                return key;
            };
            const bool cached = C <= kGenCacheKeys;
            // HEADS: a query with 33..256 cached keys that gets past the threshold has every lane sort ITS (at most 8) keys,
            // cache entries lane + 32 j, with a network in registers and write them back; from then on a lane keeps only the
            // head of its list (hv) and where it came from (hp), and a pull is the minimum over the 32 heads plus one reload
            // in the lanes that held it — 8 instructions instead of a pass over all cached keys
            bool heads = false;
            uint32_t hv = kNone, hp = 0;
            // smallest key above `prev` (first: smallest key at all), kNone when there is none
            auto pull = [&](uint32_t prev, bool first) -> uint32_t {
                uint32_t best = kNone;
                if (HEADS && heads) {
                    uint32_t g;
                    do {  // a point reached through several tables has its key in several lists: equal heads leave together, a
                          // repeat inside one list is pulled again and skipped (g == prev)
                        g = __reduce_min_sync(FULL, hv);
                        if (hv == g && g != kNone) {
                            hp += 128u;
                            hv = hp < s_keys + C * 4u ? lds32(hp) : kNone;
                        }
                    } while (g == prev);
                    return g;
                }
                if (cached) {
                    // keys <= prev wrap to the top of the u32 range (see next_key in match_kernels.cuh): one add-and-min per key
                    const uint32_t nb = first ? 0u : ~prev;
                    uint32_t acc = kNone;
#pragma unroll 4
                    for (uint32_t i = lane; i < C; i += 32) acc = min(acc, lds32(s_keys + i * 4u) + nb);
                    const uint32_t g = __reduce_min_sync(FULL, acc);
                    if (first) return g;
                    return g >= nb - 1u ? kNone : g - nb;
                }
                for (uint32_t i = lane; i < C; i += 32) {
                    const uint32_t k = key_at(i);
                    if ((first || k > prev) && k < best) best = k;
                }
                return __reduce_min_sync(FULL, best);
            };
            __syncwarp();  // the previous query's cache is no longer read
            // keys of all candidates, kGenChains independent gather chains (id -> code) per lane in flight; the smallest on the way
            uint32_t kmin = kNone;
            for (uint32_t i0 = 0; i0 < C; i0 += 32u * kGenChains) {
                uint32_t kc[kGenChains];
#pragma unroll
                for (uint32_t u = 0; u < kGenChains; ++u) {
                    const uint32_t i = i0 + 32u * u + lane;
                    kc[u] = i < C ? key_at(i) : kNone;
                }
#pragma unroll
                for (uint32_t u = 0; u < kGenChains; ++u) {
                    const uint32_t i = i0 + 32u * u + lane;
                    if (cached && i < C) sts32(s_keys + i * 4u, kc[u]);
                    kmin = min(kmin, kc[u]);
                }
            }
            __syncwarp();
            uint32_t nk = __reduce_min_sync(FULL, kmin);

            uint32_t best = kNone, second = kNone, best_id = kNone;
            bool unthresholded = false;  // the re-rank of matcher.cpp:183-189 is under way
            if (nk != kNone && (nk >> 24) <= P.tau) {
                // this lane's 4 bytes of the query row
                const uint32_t qrow = __ldg(reinterpret_cast<const uint32_t*>(I.desc + uint64_t(q) * kDim) + lane);
                if (HEADS && cached && C > 32u && C <= 256u) {
                    heads = true;
                    uint32_t hk[8];
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j) hk[j] = lane + 32u * j < C ? lds32(s_keys + (lane + 32u * j) * 4u) : kNone;
                    auto cx = [&](int a, int b) {
                        const uint32_t lo = min(hk[a], hk[b]), hi = max(hk[a], hk[b]);
                        hk[a] = lo;
                        hk[b] = hi;
                    };
                    // 19-exchange sorting network for 8 keys
                    cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7); cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7); cx(1, 2); cx(5, 6);
                    cx(0, 4); cx(3, 7); cx(1, 5); cx(2, 6); cx(1, 4); cx(3, 6); cx(2, 4); cx(3, 5); cx(3, 4);
                    // back to the lane's own entries (no other lane reads them while the lists are in use)
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (lane + 32u * j < C) sts32(s_keys + (lane + 32u * j) * 4u, hk[j]);
                    hp = s_keys + lane * 4u;
                    hv = hk[0];
                }
                for (;;) {
                    // rank n: verified at once (euclidean_verify's loop body, matcher.cpp:124-133); the row travels while the
                    // next key is pulled
                    const uint32_t id = explicit_lists ? __ldg(G.list_ids + list_lo + (nk & 0xffffffu)) : (nk & 0xffffffu);
                    const uint32_t trow = __ldg(reinterpret_cast<const uint32_t*>(J.desc + uint64_t(id) * kDim) + lane);
                    if (P.dbg_ranked != nullptr && lane == 0) P.dbg_ranked[uint64_t(q) * P.top_k + n] = id;
                    ++n;
                    const uint32_t nxt = n == P.top_k ? kNone : pull(nk, false);
                    const uint32_t d = __reduce_add_sync(FULL, sqdiff4(qrow, trow));
                    if (d < best) {
                        second = best;
                        best = d;
                        best_id = id;
                    } else if (d < second) {
                        second = d;
                    }
                    if (nxt == kNone) break;  // the list is full, or no key is left
                    nk = nxt;
                    if (!unthresholded && (nk >> 24) > P.tau) {
                        // the threshold cut something; a ranking too small for the ratio test is redone without it
                        if (n < P.min_ranked) unthresholded = true;
                        else break;
                    }
                }
            }
            if (n >= 2) {
                st_vq += 1;
                st_dist += n;
                if (second != 0u && double(best) < __dmul_rn(P.ratio_sq, double(second))) {
                    out_t = best_id;
                    out_d = best;
                    if (lane == 0) atomicAdd(&P.pair_counts[pair], 1u);
                }
            }
        }
        if (P.dbg_count != nullptr && lane == 0) P.dbg_count[q] = n;
        if (lane == 0) __stcs(P.res + g, make_uint2(out_t, out_d));
    }
    // one atomic per visit and counter
    if (lane == 0) {
        if (st_raw) atomicAdd(&P.stats->raw_candidates, (unsigned long long)st_raw);
        if (st_vq) atomicAdd(&P.stats->verified_queries, (unsigned long long)st_vq);
        if (st_dist) atomicAdd(&P.stats->distances, (unsigned long long)st_dist);
    }
    st_raw = st_vq = st_dist = 0;
    }
}

// Candidate lists of one pair (matcher.cpp:164-171): per query the L buckets concatenated, sorted, made unique — through a
// bitmap over the train image's point ids in shared memory (one bit per point, per warp).  out == nullptr: counts[q] = size
// of the list; otherwise the list of query q goes to out[offsets[q] ...], ascending ids.
__global__ void __launch_bounds__(kGenThreads) cand_union_kernel(const DevImage* __restrict__ images, uint32_t slot_i, uint32_t slot_j,
                                                                 uint32_t m, uint32_t L, uint32_t sparse, uint32_t* __restrict__ counts,
                                                                 const unsigned long long* __restrict__ offsets,
                                                                 uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) uint32_t s_bits_all[];  // kGenWarps x kGenBitmapWords
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* bits = s_bits_all + warp * kGenBitmapWords;
    const DevImage I = images[slot_i];
    const DevImage J = images[slot_j];
    const uint32_t words = (J.n + 31) / 32;
    for (uint32_t w = lane; w < words; w += 32) bits[w] = 0;
    __syncwarp();
    for (uint32_t q = blockIdx.x * kGenWarps + warp; q < I.n; q += gridDim.x * kGenWarps) {
        uint32_t total = 0;
        if (J.n != 0) {
            const BucketRanges r = resolve_ranges(I, J, q, L, m, sparse != 0, lane);
            uint32_t wmin = kNone, wmax = 0;
            for (uint32_t i = lane; i < r.total; i += 32) {
                const uint32_t id = range_id(r, J, sparse != 0, i);
                atomicOr(bits + (id >> 5), 1u << (id & 31));
                wmin = min(wmin, id >> 5);
                wmax = max(wmax, id >> 5);
            }
            wmin = __reduce_min_sync(FULL, wmin);
            wmax = __reduce_max_sync(FULL, wmax);
            __syncwarp();
            if (r.total != 0) {
                uint32_t* dst = out ? out + offsets[q] : nullptr;
                for (uint32_t w0 = wmin; w0 <= wmax; w0 += 32) {
                    const uint32_t w = w0 + lane;
                    uint32_t word = w <= wmax ? bits[w] : 0u;
                    if (w <= wmax) bits[w] = 0;
                    const uint32_t c = __popc(word);
                    uint32_t incl = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t u = __shfl_up_sync(FULL, incl, d);
                        if (int(lane) >= d) incl += u;
                    }
                    if (dst) {
                        uint32_t at = total + incl - c;
                        while (word) {
                            dst[at++] = w * 32u + uint32_t(__ffs(word) - 1);
                            word &= word - 1;
                        }
                    }
                    total += __shfl_sync(FULL, incl, 31);
                }
            }
            __syncwarp();
        }
        if (!out && lane == 0) counts[q] = total;
    }
}

// Sparse bucket index of one (image, table): keys  code << 16 | point  sorted ascending = the reference's sort of (code,
// point) pairs (matcher.cpp:34-37).  A bitonic network whose every compare-exchange is ascending (the first step of each
// merge mirrors its block), so the positions past n behave as +infinity without being stored: an exchange whose upper
// partner lies past n is a no-op.
constexpr int kSparseThreads = 1024;
__global__ void __launch_bounds__(kSparseThreads) sparse_index_kernel(const DevImage* __restrict__ images, const uint32_t* __restrict__ slots,
                                                                      uint32_t L) {
    const DevImage img = images[slots[blockIdx.x]];
    const uint32_t t = blockIdx.y, n = img.n;
    if (n == 0) return;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(img.offs) + uint64_t(t) * n;
    for (uint32_t p = threadIdx.x; p < n; p += kSparseThreads)
        keys[p] = ((unsigned long long)__ldg(img.shorts + uint64_t(p) * L + t) << 16) | p;
    uint32_t npow = 1;
    while (npow < n) npow <<= 1;
    auto exchange = [&](uint32_t lo, uint32_t hi) {
        if (hi < n) {
            const unsigned long long a = keys[lo], b = keys[hi];
            if (a > b) {
                keys[lo] = b;
                keys[hi] = a;
            }
        }
    };
    for (uint32_t k = 2; k <= npow; k <<= 1) {
        __syncthreads();
        const uint32_t half = k >> 1;
        for (uint32_t x = threadIdx.x; x < npow / 2; x += kSparseThreads) {
            const uint32_t base = (x / half) * k, o = x % half;
            exchange(base + o, base + k - 1u - o);
        }
        for (uint32_t j = k >> 2; j > 0; j >>= 1) {
            __syncthreads();
            for (uint32_t x = threadIdx.x; x < npow / 2; x += kSparseThreads) {
                const uint32_t lo = (x / j) * 2u * j + (x % j);
                exchange(lo, lo + j);
            }
        }
    }
}

// the instantiation for a run's flags (HEADS = false only as the A/B reference of the plain bucket run)
using GeneralKernel = void (*)(const GeneralParams);
inline GeneralKernel general_kernel_for(bool heads, bool lists, bool sparse, bool guided) {
    if (lists) {  // explicit lists: the bucket index is not read (SPARSE is irrelevant)
        return guided ? general_match_kernel<true, true, false, true> : general_match_kernel<true, true, false, false>;
    }
    if (sparse) return guided ? general_match_kernel<true, false, true, true> : general_match_kernel<true, false, true, false>;
    if (guided) return general_match_kernel<true, false, false, true>;
    return heads ? general_match_kernel<true, false, false, false> : general_match_kernel<false, false, false, false>;
}

}  // namespace chgpu
