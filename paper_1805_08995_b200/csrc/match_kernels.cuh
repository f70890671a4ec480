// match_kernels.cuh — K3, the pair-matching kernel.
//
// K3 is a persistent kernel: one CTA per SM pulls work units (pair, query range) from a global
// counter.  For each unit the train image's 128-bit codes and its dense bucket offsets are
// brought into shared memory with bulk async copies (cp.async.bulk + mbarrier, the sm_90+/sm_100
// TMA path), then every warp owns one query point at a time:
//
//   1. bucket lookup   : kBatch queries at a time, ONE QUERY PER LANE: the lane reads its query's L
//                        table codes and long code from global memory, resolves the L CSR ranges
//                        [first, last] in the train image's bucket index (shared memory) and parks
//                        everything the warp-wide steps below need in a per-warp staging record
//                        (matcher.cpp:164-169).  The query-side global round trip is paid once per
//                        batch; the per-query code reads the record with uniform shared loads.
//   2. Hamming scan    : 32 candidates per step, one per lane: id = ids[...], train code gathered
//                        from shared memory (LDS.128), 4x LOP3 + 4x POPC,
//                        key = distance<<24 | id                              (matcher.cpp:68-84)
//                        Step t covers the first 32 entries of table t's bucket; its ids were
//                        PREFETCHED while the previous query was ranked and verified.  The entries
//                        past 32 of all buckets form one flat index space walked by up to
//                        kOverSlots further steps; the table a flat index falls in comes from a
//                        staged lane mask (segment = popc(mask & lanes<=l)), not a compare chain.
//                        The bucket lists are stored in a bank-friendly order (see DevImage::scan),
//                        so 8 consecutive entries gather from 8 different bank groups.
//                        Queries whose buckets overflow that (large images) take rounds of 32
//                        entries per table: a first pass keeps only the smallest key, and only
//                        queries with a candidate within tau pay for a second, merging pass.
//   3. ranking         : the ranked list is the first n keys in ascending (distance, id) order
//                        with EQUAL KEYS COLLAPSED — the same point reached through several
//                        tables has the same key, so the reference's sort+unique
//                        (matcher.cpp:170-171) is implicit.  Keys are pulled one at a time:
//                        every lane folds its slots with min(acc, key - (prev+1)) (one
//                        VIADDMNMX per slot; keys <= prev wrap to the top of the u32 range) and
//                        a warp-wide REDUX.MIN picks the winner.  The threshold tau and the
//                        re-rank fallback (matcher.cpp:176-189) only decide where the pulling
//                        stops, so no histogram has to be stored.
//   4. verification    : 4 lanes per candidate row, __vabsdiffu4 + __dp4a (exact u32 squared
//                        distance), best / second with rank-order tie-break, Lowe ratio in
//                        fp64 exactly as matcher.cpp:115-137.  (-DCHGPU_VERIFY_MMA: the same distances
//                        from a Gram matrix on the integer tensor-core path, mma.sync m16n8k16 u8;
//                        measured slower, kept as an A/B switch.)
//
// Results go to a per-query scratch (train id, d^2); compact_kernel (compact_kernels.cuh) turns
// them into the reference's MatchRecord stream, ascending query index inside every pair.
#pragma once

#include <utility>

#include "dev_types.cuh"

namespace chgpu {

// Compile-time loop: f(std::integral_constant<int, 0>{}), ..., f(std::integral_constant<int, N-1>{}).
template <class F, int... Is>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

#ifndef CHGPU_MATCH_THREADS
#define CHGPU_MATCH_THREADS 896
#endif
#ifndef CHGPU_OVER_SLOTS
#define CHGPU_OVER_SLOTS 3
#endif
#ifndef CHGPU_VERIFY_LANES
#define CHGPU_VERIFY_LANES 4
#endif
#ifndef CHGPU_VERIFY_TILES
#define CHGPU_VERIFY_TILES 2  // tensor-core verification: 7-candidate tiles per round (1 or 2)
#endif
constexpr int kMatchThreads = CHGPU_MATCH_THREADS;
constexpr uint32_t kVerifyLanes = CHGPU_VERIFY_LANES;  // lanes per descriptor row in the verification (2, 4 or 8)
static_assert(kVerifyLanes == 2 || kVerifyLanes == 4 || kVerifyLanes == 8, "lanes per row");
// bucket lists in the bank-friendly scan order (default) or, for A/B measurements, the canonical one
#ifdef CHGPU_SCAN_CANONICAL
#define CH_IDS(img) (img).points
#else
#define CH_IDS(img) (img).scan
#endif
constexpr int kOverSlots = CHGPU_OVER_SLOTS;  // register slots for bucket entries past the first 32 of every table
static_assert(kOverSlots >= 1 && kOverSlots <= 3, "the staging record carries three overflow segment masks");

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
    uint32_t smem_long_bytes;   // SMEM_TRAIN: bytes reserved for the train codes (offsets follow)
    double ratio_sq;            // cfg.ratio * cfg.ratio, formed on the host in fp64
    const double* fmats;        // GUIDED: 9 doubles per pair, row-major fundamental matrix (I -> lines in J)
    double band_px;             // GUIDED: epipolar band half-width in pixels
    uint32_t* dbg_ranked;       // optional: n_i x top_k
    uint32_t* dbg_count;        // optional: n_i
    // tiled train images (MODE 1 / 2 and tile_merge_kernel)
    uint32_t* gmin;             // per query (res indexing): smallest key over all tiles
    unsigned long long* gdone;  // per query: bit t set once tile t's list is written
    uint32_t* lists;            // per query: list_stride keys, tile t's top_k keys at [t * top_k, (t + 1) * top_k)
    uint32_t list_stride;
    uint32_t tile_points;       // point ids per tile
    uint16_t* act;              // per (query image, tile) pair, at PairDesc::act_off: the queries the top-k pass visits ...
    uint32_t* nact;             // ... and how many (tile_compact_kernel)
};

// Train images too large for the shared-memory tile are matched tile by tile: every id range of
// tile_points points is a small train image of its own (own bucket index over local ids, built by the
// same bucket_build_kernel on a slice of the codes), so the kernel below runs unchanged on (query image,
// tile) pairs and only its output differs:
//   MODE 1 (kTileMin)   scan: the smallest key of the tile joins gmin[query] (atomicMin).  Most queries have no
//                       candidate within tau in any tile and are finished after this pass.  A tile that itself
//                       has one writes its list (below) right away and marks it in gdone[query].
//   MODE 2 (kTileTopK)  queries with gmin within tau, tiles not yet marked (tile_compact_kernel lists them per
//                       (query image, tile) pair, so the pass walks a dense list): the tile's top_k smallest
//                       distinct keys, no threshold, global point ids, go to lists[query][tile].
// tile_merge_kernel then merges the lists of a query, applies the threshold / re-rank rule of
// matcher.cpp:176-189 to the merged ranking and verifies it exactly like MODE 0 does.
constexpr int kModeMatch = 0, kModeTileMin = 1, kModeTileTopK = 2;
// kModeMatchActive: kModeMatch over the queries the join pass (join_kernels.cuh) found a candidate within tau for — the
// pair's list P.act / P.nact, ascending query indices; every other query keeps the "no match" of the initialised scratch
// and the raw-candidate statistic has been taken by the join pass.
constexpr int kModeMatchActive = 3;

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
// Shared-memory loads by 32-bit shared-window address (keeps the address arithmetic to one LEA).
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
template <uint32_t OFF>
__device__ __forceinline__ uint2 lds64_at(uint32_t base) {  // [base + OFF], 8-byte aligned
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+%3];" : "=r"(v.x), "=r"(v.y) : "r"(base), "n"(OFF));
    return v;
}
template <uint32_t OFF>
__device__ __forceinline__ uint4 lds128_at(uint32_t base) {  // [base + OFF], 16-byte aligned
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+%5];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(base), "n"(OFF));
    return v;
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint2 lds64x(uint32_t addr) {  // two adjacent u32 (need not be 8-byte aligned)
    uint2 v;
    asm volatile("ld.shared.u32 %0, [%2];\n\tld.shared.u32 %1, [%2+4];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

// Read-once global loads that must not displace the train image's bucket lists from L1.
__device__ __forceinline__ uint4 ldg_stream128(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldg_stream32(const void* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t hamming128(const uint4& a, const uint4& b) {
#ifdef CHGPU_CSA_POPC
    // carry-save adder over three of the four xor words: 3 POPC + 2 LOP3 instead of 4 POPC
    const uint32_t x = a.x ^ b.x, y = a.y ^ b.y, z = a.z ^ b.z, w = a.w ^ b.w;
    const uint32_t s = x ^ y ^ z, c = (x & y) | (z & (x ^ y));
    return __popc(s) + __popc(w) + 2u * __popc(c);
#else
    return __popc(a.x ^ b.x) + __popc(a.y ^ b.y) + __popc(a.z ^ b.z) + __popc(a.w ^ b.w);
#endif
}

// Sum over 4 byte lanes of (a_i - b_i)^2, exact in u32.
__device__ __forceinline__ uint32_t sqdiff4(uint32_t a, uint32_t b) {
    const uint32_t ad = __vabsdiffu4(a, b);
    return __dp4a(ad, ad, 0u);
}

// Warp-wide smallest key over all slots (+ one extra value).
template <int SLOTS>
__device__ __forceinline__ uint32_t first_key(const uint32_t (&key)[SLOTS], uint32_t extra) {
    uint32_t lmin = extra;
#pragma unroll
    for (int i = 0; i < SLOTS; ++i) lmin = min(lmin, key[i]);
    return __reduce_min_sync(0xffffffffu, lmin);
}

// Warp-wide smallest key strictly greater than `prev`, or kNone when there is none.
// key - (prev + 1) in u32 arithmetic: keys <= prev (and empty kNone slots) wrap to values
// >= kNone - prev - 1, which no key > prev can reach (valid keys are < 2^31 + 2^24).
template <int SLOTS>
__device__ __forceinline__ uint32_t next_key(const uint32_t (&key)[SLOTS], uint32_t extra, uint32_t prev) {
    const uint32_t nb = ~prev;  // -(prev + 1)
#ifndef CHGPU_SERIAL_PULL
    // two independent min chains (half the dependency depth, one more instruction: +0.3 % measured)
    uint32_t acc = extra + nb, acc2 = key[0] + nb;
#pragma unroll
    for (int i = 1; i < SLOTS; ++i) {
        if (i & 1) acc = min(acc, key[i] + nb);
        else acc2 = min(acc2, key[i] + nb);
    }
    acc = min(acc, acc2);
#else
    uint32_t acc = extra + nb;
#pragma unroll
    for (int i = 0; i < SLOTS; ++i) acc = min(acc, key[i] + nb);
#endif
    const uint32_t g = __reduce_min_sync(0xffffffffu, acc);
    return g >= nb - 1u ? kNone : g - nb;
}

// This lane's own smallest key strictly greater than `prev` (no warp exchange), or kNone.
template <int SLOTS>
__device__ __forceinline__ uint32_t lane_next_key(const uint32_t (&key)[SLOTS], uint32_t prev) {
    const uint32_t nb = ~prev;
    uint32_t acc = nb - 1u, acc2 = key[0] + nb;  // kNone + nb; see next_key for the wrap argument
#pragma unroll
    for (int i = 1; i < SLOTS; ++i) {
        if (i & 1) acc = min(acc, key[i] + nb);
        else acc2 = min(acc2, key[i] + nb);
    }
    acc = min(acc, acc2);
    return acc >= nb - 1u ? kNone : acc - nb;
}

// next_key that also hands back what every lane found on its own: *lane_min = this lane's smallest key > prev (or kNone).
template <int SLOTS>
__device__ __forceinline__ uint32_t next_key_keep(const uint32_t (&key)[SLOTS], uint32_t prev, uint32_t& lane_min) {
    lane_min = lane_next_key(key, prev);
    return __reduce_min_sync(0xffffffffu, lane_min);
}

// Hamming key of one candidate id: distance<<24 | id.
template <bool SMEM_TRAIN>
__device__ __forceinline__ uint32_t key_of(uint32_t id, const uint4& ql, uint32_t s_long, const uint4* __restrict__ g_long) {
    uint4 c;
    if (SMEM_TRAIN) c = lds128(s_long + id * 16u);
    else c = __ldg(g_long + id);
#ifdef CHGPU_CSA_POPC
    return (hamming128(c, ql) << 24) | id;
#else
    // distance << 24 | id with the shift folded into two multiply-adds (id < 2^24: '+' carries nothing)
    const uint32_t t = __popc(c.x ^ ql.x) + __popc(c.y ^ ql.y) + __popc(c.z ^ ql.z);
    const uint32_t k = __popc(c.w ^ ql.w) * 0x1000000u + id;
    return t * 0x1000000u + k;
#endif
}

// One step of the Hamming scan: candidate `first + lane` of the bucket-major id list, clamped
// to `last` (lanes past the end re-evaluate the last candidate: equal keys collapse).
template <bool SMEM_TRAIN>
__device__ __forceinline__ uint32_t scan_step(const uint16_t* __restrict__ pts, uint32_t first, uint32_t last,
                                              uint32_t lane, const uint4& ql, uint32_t s_long,
                                              const uint4* __restrict__ g_long) {
    const uint32_t id = __ldg(pts + min(first + lane, last));
    return key_of<SMEM_TRAIN>(id, ql, s_long, g_long);
}

// Per-warp staging of the bucket lookups of kBatch consecutive queries of the warp (shared memory),
// one record per query:
//   +0   ql uint4
//   +16  hdr = tover (capped at 255) | empty-table mask << 8 | base1 << 16 | base2 << 24
//   +20  M0, M1, M2: for overflow step s, bit l set iff flat overflow index 32 s + l starts a table's segment
//   +32  LT x {first, last} entry of the query's bucket in table t (`last` clamped to `first` when empty:
//        such lanes read a neighbour's entry, discarded later)
//   +32+8LT  adj[k], k-th table WITH overflow: flat overflow index r of that segment -> ids[r + adj]
// tover = entries past the first 32 of every bucket, summed over the tables; base_s = segments that start
// before step s.  Lane l of step s belongs to segment base_s + popc(M_s & lanes<=l) - 1.
constexpr uint32_t kBatch = 16;
__host__ __device__ constexpr uint32_t stage_record_bytes(int LT) { return (32u + uint32_t(LT) * 12u + 15u) & ~15u; }
__host__ __device__ constexpr uint32_t stage_bytes_per_warp(int LT) { return kBatch * stage_record_bytes(LT); }

// Epipolar band of one query (guided_match_pair, geometry.cpp:234-250): l = F (x, y, 1)^T, candidates
// farther than band_px from the line are dropped between lookup and ranking; a degenerate line leaves the
// query unguided.  fp64, every operation individually rounded, in the order the oracle states (chor.h).
struct EpiLine {
    double a, b, c, inv_norm;
    bool active;
};
__device__ __forceinline__ EpiLine epipolar_band(const double* __restrict__ F, float4 kp) {
    const double x = double(kp.x), y = double(kp.y);
    EpiLine l;
    l.a = __dadd_rn(__dadd_rn(__dmul_rn(__ldg(F + 0), x), __dmul_rn(__ldg(F + 1), y)), __ldg(F + 2));
    l.b = __dadd_rn(__dadd_rn(__dmul_rn(__ldg(F + 3), x), __dmul_rn(__ldg(F + 4), y)), __ldg(F + 5));
    // third component: the order Eigen >= 3.3 gives it (see oracle/chor.h): F20 x + (F21 y + F22)
    l.c = __dadd_rn(__dmul_rn(__ldg(F + 6), x), __dadd_rn(__dmul_rn(__ldg(F + 7), y), __ldg(F + 8)));
    l.active = !(l.a == 0.0 && l.b == 0.0);
    l.inv_norm = l.active ? __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dmul_rn(l.a, l.a), __dmul_rn(l.b, l.b)))) : 0.0;
    return l;
}
__device__ __forceinline__ uint32_t band_filter(uint32_t key, const EpiLine& l, const float4* __restrict__ kp_j, double band_px) {
    if (!l.active || key == kNone) return key;
    const float4 t = __ldg(kp_j + (key & 0xffffffu));
    const double d = __dmul_rn(fabs(__dadd_rn(__dadd_rn(__dmul_rn(l.a, double(t.x)), __dmul_rn(l.b, double(t.y))), l.c)), l.inv_norm);
    return d > band_px ? kNone : key;
}

#ifndef CHGPU_VERIFY_MMA
// Verification of a ranked list (euclidean_verify, matcher.cpp:115-137), SIMT form (the default; the tensor-core
// form below, -DCHGPU_VERIFY_MMA, issues 14 fewer instructions per query and is 2.4 % SLOWER on the B200: DESIGN.md): lane r holds the r-th ranked key
// (id in the low 24 bits), n >= 2 entries.  kVerifyLanes lanes per candidate row (128 / kVerifyLanes bytes
// each), 32 / kVerifyLanes rows per round; exact u32 squared distances; best = smallest d^2 with ties to the
// earlier rank (strict '<' in the reference loop); Lowe ratio in fp64 with the reference's operand order.
__device__ __forceinline__ bool verify_ranked(const uint8_t* __restrict__ desc_i, const uint8_t* __restrict__ desc_j,
                                              uint32_t q, uint32_t n, uint32_t mykey, uint32_t lane, double ratio_sq,
                                              uint32_t& out_t, uint32_t& out_d) {
    constexpr uint32_t FULL = 0xffffffffu;
#ifndef CHGPU_NO_VERIFY_SHORTCUT
    // Shortcut (exact): usually the first ranked candidate is the match and the rest are far away.  Lanes 0-7 form its
    // full distance F (16 bytes each); lane pairs 8+2j, 9+2j form the distance of candidate j + 1 over its FIRST 32
    // dimensions only, P_c <= d^2_c (one 32-byte sector per candidate instead of four).  If F < ratio^2 * min P_c then
    // F < P_c <= d^2_c for every other candidate (ratio^2 < 1): the first candidate is the strict best, `second` >=
    // min P_c > 0, and by the monotonicity of the rounded product the reference's test best < ratio^2 * second holds:
    // the record is (id_0, F), exactly the reference's.  Otherwise nothing is decided and the full evaluation below runs.
    if (n <= 13u) {
        const bool whole = lane < 8u;
        const uint32_t cj = whole ? 0u : ((lane - 8u) >> 1) + 1u;  // rank of the candidate this lane works on
        const uint32_t piece = whole ? lane : (lane & 1u);          // which 16 bytes of the rows
        const uint32_t cid = __shfl_sync(FULL, mykey, min(cj, n - 1)) & 0xffffffu;
        const uint4 qa = __ldg(reinterpret_cast<const uint4*>(desc_i + uint64_t(q) * kDim) + piece);
        const uint4 ta = __ldg(reinterpret_cast<const uint4*>(desc_j + uint64_t(cid) * kDim) + piece);
        uint32_t s = sqdiff4(qa.x, ta.x) + sqdiff4(qa.y, ta.y) + sqdiff4(qa.z, ta.z) + sqdiff4(qa.w, ta.w);
        s += __shfl_xor_sync(FULL, s, 1);                        // pairs: P_c complete
        uint32_t f = s + __shfl_xor_sync(FULL, s, 2);
        f += __shfl_xor_sync(FULL, f, 4);                        // lanes 0-7: F complete
        const uint32_t full0 = __shfl_sync(FULL, f, 0);
        const uint32_t pmin = __reduce_min_sync(FULL, (!whole && cj < n) ? s : kNone);
        if (double(full0) < __dmul_rn(ratio_sq, double(pmin))) {
            out_t = __shfl_sync(FULL, mykey, 0) & 0xffffffu;
            out_d = full0;
            return true;
        }
    }
#endif
    constexpr uint32_t VL = kVerifyLanes, ROWS = 32u / VL, PIECES = 8u / VL;
    const uint32_t part = lane % VL, cand = lane / VL;
    const uint4* __restrict__ qrow = reinterpret_cast<const uint4*>(desc_i + uint64_t(q) * kDim) + part * PIECES;
    uint4 qa[PIECES];
#pragma unroll
    for (uint32_t w = 0; w < PIECES; ++w) qa[w] = __ldg(qrow + w);
    uint32_t mydist = kNone;
    for (uint32_t j0 = 0; j0 < n; j0 += ROWS) {
        const uint32_t jj = min(j0 + cand, n - 1);
        const uint32_t cid = __shfl_sync(FULL, mykey, jj) & 0xffffffu;
        const uint4* __restrict__ trow = reinterpret_cast<const uint4*>(desc_j + uint64_t(cid) * kDim) + part * PIECES;
        uint32_t s = 0;
#pragma unroll
        for (uint32_t w = 0; w < PIECES; ++w) {
            const uint4 ta = __ldg(trow + w);
            s += sqdiff4(qa[w].x, ta.x) + sqdiff4(qa[w].y, ta.y) + sqdiff4(qa[w].z, ta.z) + sqdiff4(qa[w].w, ta.w);
        }
#pragma unroll
        for (uint32_t d = 1; d < VL; d <<= 1) s += __shfl_xor_sync(FULL, s, d);
        const uint32_t v = __shfl_sync(FULL, s, ((lane - j0) % ROWS) * VL);
        if (lane >= j0 && lane < j0 + ROWS && lane < n) mydist = v;
    }
    const uint32_t packed = lane < n ? ((mydist << 8) | lane) : kNone;
    const uint32_t bestp = __reduce_min_sync(FULL, packed);
    const uint32_t bl = bestp & 0xffu, best = bestp >> 8;
    const uint32_t second = __reduce_min_sync(FULL, (lane < n && lane != bl) ? mydist : kNone);
    const uint32_t bid = __shfl_sync(FULL, mykey, bl) & 0xffffffu;
    if (second != 0u && double(best) < __dmul_rn(ratio_sq, double(second))) {
        out_t = bid;
        out_d = best;
        return true;
    }
    return false;
}
#else
// One tensor-core step of the verification: D(16x8, s32) += A(16x16, u8, row) * B(16x8, u8, col)
// (warp-level mma.sync; SASS IMMA.16816.U8.U8).
__device__ __forceinline__ void mma_u8_16816(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm("mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(b0));
}
// Gram matrix of 8 descriptor rows, one row per fragment group g, thread t of the group holding bytes [32 t, 32 t + 32)
// of its row as two LDG.128 results.  The fragment registers of mma.sync are taken as loaded (no repacking): an A
// pair (a0 | a1) is an even / odd word pair of ONE row, so fragment row g is the row's even words E_g and fragment
// row g + 8 its odd words O_g; with B = the even word the upper half of D accumulates E_g . E_c, with B = the odd word
// the lower half accumulates O_g . O_c (the other halves are mixed products nobody reads).  The K order is free as
// long as A and B agree.  After the 8 steps  G[g][c] = e[c & 1] + o[2 + (c & 1)]  in thread t == c >> 1.
__device__ __forceinline__ void gram8_u8(int (&e)[4], int (&o)[4], const uint4& x0, const uint4& x1) {
    mma_u8_16816(e, x0.x, x0.y, x0.x);
    mma_u8_16816(o, x0.x, x0.y, x0.y);
    mma_u8_16816(e, x0.z, x0.w, x0.z);
    mma_u8_16816(o, x0.z, x0.w, x0.w);
    mma_u8_16816(e, x1.x, x1.y, x1.x);
    mma_u8_16816(o, x1.x, x1.y, x1.y);
    mma_u8_16816(e, x1.z, x1.w, x1.z);
    mma_u8_16816(o, x1.z, x1.w, x1.w);
}

// Verification of a ranked list (euclidean_verify, matcher.cpp:115-137): lane r holds the r-th ranked key
// (id in the low 24 bits), n >= 2 entries.  Exact u32 squared distances; best = smallest d^2 with ties to the
// earlier rank (strict '<' in the reference loop); Lowe ratio in fp64 with the reference's operand order.
//
// The distances come from the integer tensor-core path: 7 candidate rows and the query row (row 7) form an
// 8 x 128 u8 matrix X; its Gram matrix G = X X^T (u8 x u8 -> s32, every product and sum exact) holds all three
// terms of |x_r - q|^2 = G[r][r] - 2 G[r][7] + G[7][7].  Two such tiles (14 candidates) per round, their four
// row loads per thread in flight together.  The thread that holds G[r][r] (t == r >> 1) fetches G[r][7] from
// thread 3 of its group and keeps (d^2 << 8 | rank) of its candidates; best and second come out of two
// warp-wide minima over those, so the distances never have to be moved to "their" lane.
__device__ __forceinline__ bool verify_ranked(const uint8_t* __restrict__ desc_i, const uint8_t* __restrict__ desc_j,
                                              uint32_t q, uint32_t n, uint32_t mykey, uint32_t lane, double ratio_sq,
                                              uint32_t& out_t, uint32_t& out_d) {
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t g = lane >> 2, t = lane & 3;  // fragment coordinates: row of the tile, 32-byte slice of the row
    const uint4* __restrict__ qrow = reinterpret_cast<const uint4*>(desc_i + uint64_t(q) * kDim) + t * 2;
    const bool own = g != 7 && t == (g >> 1);  // this thread receives G[g][g] of both tiles
    uint32_t m1 = kNone, m2 = kNone;           // smallest and second smallest (d^2 << 8 | rank) seen by this thread
#if CHGPU_VERIFY_TILES == 2
    for (uint32_t j0 = 0; j0 < n; j0 += 14) {
        // tile A: candidates j0 .. j0 + 6, tile B: j0 + 7 .. j0 + 13 (past the end: the last one again)
        const uint32_t ra = j0 + g, rb = ra + 7;
        const uint32_t ia = __shfl_sync(FULL, mykey, min(ra, n - 1)) & 0xffffffu;
        const uint32_t ib = __shfl_sync(FULL, mykey, min(rb, n - 1)) & 0xffffffu;
        const uint4* __restrict__ pa = g == 7 ? qrow : reinterpret_cast<const uint4*>(desc_j + uint64_t(ia) * kDim) + t * 2;
        const uint4* __restrict__ pb = g == 7 ? qrow : reinterpret_cast<const uint4*>(desc_j + uint64_t(ib) * kDim) + t * 2;
        const uint4 a0 = __ldg(pa), a1 = __ldg(pa + 1), b0 = __ldg(pb), b1 = __ldg(pb + 1);
        int ea[4] = {0, 0, 0, 0}, oa[4] = {0, 0, 0, 0}, eb[4] = {0, 0, 0, 0}, ob[4] = {0, 0, 0, 0};
        gram8_u8(ea, oa, a0, a1);
        gram8_u8(eb, ob, b0, b1);
        const int a_even = ea[0] + oa[2], a_odd = ea[1] + oa[3];  // G_A[g][2t], G_A[g][2t+1]
        const int b_even = eb[0] + ob[2], b_odd = eb[1] + ob[3];
        const int cross_a = __shfl_sync(FULL, a_odd, lane | 3u), cross_b = __shfl_sync(FULL, b_odd, lane | 3u);  // G[g][7]
        const int qq = __shfl_sync(FULL, a_odd, 31);                                                             // G[7][7]
        const int diag_a = (g & 1) ? a_odd : a_even, diag_b = (g & 1) ? b_odd : b_even;
        const uint32_t da = uint32_t(diag_a + qq - 2 * cross_a), db = uint32_t(diag_b + qq - 2 * cross_b);
        const uint32_t pka = (own && ra < n) ? ((da << 8) | ra) : kNone;
        const uint32_t pkb = (own && rb < n) ? ((db << 8) | rb) : kNone;
        m2 = min(m2, max(m1, pka));
        m1 = min(m1, pka);
        m2 = min(m2, max(m1, pkb));
        m1 = min(m1, pkb);
    }
#else
    for (uint32_t j0 = 0; j0 < n; j0 += 7) {  // one tile per round: candidates j0 .. j0 + 6
        const uint32_t ra = j0 + g;
        const uint32_t ia = __shfl_sync(FULL, mykey, min(ra, n - 1)) & 0xffffffu;
        const uint4* __restrict__ pa = g == 7 ? qrow : reinterpret_cast<const uint4*>(desc_j + uint64_t(ia) * kDim) + t * 2;
        const uint4 a0 = __ldg(pa), a1 = __ldg(pa + 1);
        int ea[4] = {0, 0, 0, 0}, oa[4] = {0, 0, 0, 0};
        gram8_u8(ea, oa, a0, a1);
        const int a_even = ea[0] + oa[2], a_odd = ea[1] + oa[3];
        const int cross_a = __shfl_sync(FULL, a_odd, lane | 3u);
        const int qq = __shfl_sync(FULL, a_odd, 31);
        const int diag_a = (g & 1) ? a_odd : a_even;
        const uint32_t da = uint32_t(diag_a + qq - 2 * cross_a);
        const uint32_t pka = (own && ra < n) ? ((da << 8) | ra) : kNone;
        m2 = min(m2, max(m1, pka));
        m1 = min(m1, pka);
    }
#endif
    const uint32_t bestp = __reduce_min_sync(FULL, m1);
    const uint32_t secondp = __reduce_min_sync(FULL, m1 == bestp ? m2 : m1);
    const uint32_t bl = bestp & 0xffu, best = bestp >> 8, second = secondp >> 8;
    const uint32_t bid = __shfl_sync(FULL, mykey, bl) & 0xffffffu;
    if (second != 0u && double(best) < __dmul_rn(ratio_sq, double(second))) {
        out_t = bid;
        out_d = best;
        return true;
    }
    return false;
}
#endif

// Shortcut for the common shape of a matching query (exact): exactly one candidate k0 within tau, so the
// reference re-ranks without the threshold (matcher.cpp:176-189) and verifies k0 plus the top_k - 1 next keys.  Instead of
// pulling those keys one warp reduction at a time, every lane looks at its OWN slots: a1 < a2 < a3 = its three smallest
// keys above k0.  With M3 = min over the lanes of a3: if at least top_k - 1 DISTINCT a1 values lie below M3, then the
// (top_k - 1)-th smallest key above k0 lies below M3 as well, so every key of the reference's ranked list is some lane's a1
// or a2 (a third key of any lane is >= M3).  The a1 / a2 candidates therefore form a SUPERSET of the list's runners-up, and
// the smallest 16-dimension partial distance over that superset is a lower bound of the reference's `second`.  The test
// F < ratio^2 * bound (F = full distance of k0's point) then proves, as in verify_ranked's shortcut, that k0's point is the
// strict best and passes the reference's ratio test: the record is (id(k0), F) and the ranked list has exactly top_k
// entries (the statistics need that number).  When the count is short or the test fails nothing is decided: the caller
// goes on with the exact pulls and the full verification.
// Loads of the shortcut, issued as early as their addresses are known so that they travel under the arithmetic that
// follows: the pieces of the full distance (query row and k0's row, 8 lanes x 16 bytes) when k0 is known, ...
struct FirstRow {
    uint4 q, t;
};
__device__ __forceinline__ FirstRow load_first_row(const uint8_t* __restrict__ desc_i, const uint8_t* __restrict__ desc_j,
                                                   uint32_t q, uint32_t k0, uint32_t lane) {
    const uint32_t piece = lane & 7u;
    FirstRow r;
    r.q = __ldg(reinterpret_cast<const uint4*>(desc_i + uint64_t(q) * kDim) + piece);
    r.t = __ldg(reinterpret_cast<const uint4*>(desc_j + uint64_t(k0 & 0xffffffu) * kDim) + piece);
    return r;
}

template <int SLOTS>
__device__ __forceinline__ bool rerank_shortcut(const uint32_t (&key)[SLOTS], uint32_t k0, uint32_t a1, uint32_t top_k,
                                                const FirstRow& first, const uint8_t* __restrict__ desc_j, uint32_t lane,
                                                double ratio_sq, uint32_t& out_t, uint32_t& out_d) {
    constexpr uint32_t FULL = 0xffffffffu;
    // ... and the first 16 dimensions of every lane's a1 point before a2, a3 and the count are worked out (a lane without a
    // key re-reads k0's row: no new sector)
    const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(desc_j + uint64_t((a1 == kNone ? k0 : a1) & 0xffffffu) * kDim));
    const uint32_t a2r = lane_next_key(key, a1), a2 = a1 == kNone ? kNone : a2r;
    const uint32_t a3r = lane_next_key(key, a2), a3 = a2 == kNone ? kNone : a3r;
    const uint32_t m3 = __reduce_min_sync(FULL, a3);
    const uint32_t same = __match_any_sync(FULL, a1);
    const bool leader = (same & ((1u << lane) - 1u)) == 0u;  // lowest lane holding this a1
    const uint32_t distinct_below = __popc(__ballot_sync(FULL, leader && a1 < m3));
    if (distinct_below + 1u < top_k) return false;
#ifdef CHGPU_SHORTCUT_STATS
    out_d = 1;  // experiment: the count check passed
#endif
    // the query's first 16 dimensions sit in the lanes with piece 0
    uint4 q0;
    q0.x = __shfl_sync(FULL, first.q.x, 0);
    q0.y = __shfl_sync(FULL, first.q.y, 0);
    q0.z = __shfl_sync(FULL, first.q.z, 0);
    q0.w = __shfl_sync(FULL, first.q.w, 0);
    uint32_t p2 = kNone;  // only keys below M3 can be on the list: few lanes have such an a2
    if (a2 < m3) {
        const uint4 t2 = __ldg(reinterpret_cast<const uint4*>(desc_j + uint64_t(a2 & 0xffffffu) * kDim));
        p2 = sqdiff4(q0.x, t2.x) + sqdiff4(q0.y, t2.y) + sqdiff4(q0.z, t2.z) + sqdiff4(q0.w, t2.w);
    }
    const uint32_t p1 = a1 < m3 ? sqdiff4(q0.x, t1.x) + sqdiff4(q0.y, t1.y) + sqdiff4(q0.z, t1.z) + sqdiff4(q0.w, t1.w) : kNone;
    const uint32_t bound = __reduce_min_sync(FULL, min(p1, p2));
    uint32_t f = sqdiff4(first.q.x, first.t.x) + sqdiff4(first.q.y, first.t.y) + sqdiff4(first.q.z, first.t.z) +
                 sqdiff4(first.q.w, first.t.w);
    f += __shfl_xor_sync(FULL, f, 1);
    f += __shfl_xor_sync(FULL, f, 2);
    f += __shfl_xor_sync(FULL, f, 4);
    if (double(f) < __dmul_rn(ratio_sq, double(bound))) {
        out_t = k0 & 0xffffffu;
        out_d = f;
        return true;
    }
    return false;
}

// LT = number of table slots unrolled in registers (>= L); EXACT: L == LT, no per-table guards;
// GUIDED: the epipolar band filter above is applied to every candidate.
// DBG: the parity tests' ranked-list output (dbg_ranked / dbg_count); a separate instantiation so that production launches
// carry no per-query pointer test.
template <bool SMEM_TRAIN, int LT, bool EXACT, bool GUIDED, int MODE = kModeMatch, bool DBG = false>
__global__ void __launch_bounds__(kMatchThreads, 1) match_kernel(const MatchParams P) {
    extern __shared__ __align__(16) unsigned char s_raw[];  // [train codes | bucket offsets | lookup staging]
    __shared__ unsigned int s_unit;
    __shared__ __align__(8) uint64_t s_bar;

    constexpr int KS = LT + kOverSlots;
    constexpr bool kMatch = MODE == kModeMatch || MODE == kModeMatchActive;    // the reference's match semantics
    constexpr bool kActive = MODE == kModeTileTopK || MODE == kModeMatchActive;  // walks the pair's active-query list
    constexpr uint32_t kWarps = kMatchThreads / 32;
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nb1 = (1u << P.m) + 1;
    const uint32_t L = EXACT ? uint32_t(LT) : P.L;
    const uint32_t obytes = SMEM_TRAIN ? ((L * nb1 * 4u + 15u) & ~15u) : 0u;  // the arena pads every array to 256 B
    // shared-window addresses, pinned in registers (the compiler would otherwise re-derive
    // them from SR_CgaCtaId in front of every gather)
    uint32_t s_long = smem_addr(s_raw);
    asm volatile("" : "+r"(s_long));
    uint32_t s_offs = s_long + P.smem_long_bytes;
    asm volatile("" : "+r"(s_offs));
    uint32_t s_stage = s_offs + obytes + warp * stage_bytes_per_warp(LT);
    asm volatile("" : "+r"(s_stage));
    constexpr uint32_t kRec = stage_record_bytes(LT), kAdj = 32u + uint32_t(LT) * 8u;
    const uint32_t le_mask = (2u << lane) - 1u;  // lanes <= this one

    if (SMEM_TRAIN && tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t bar_parity = 0;
    uint32_t resident = kNone;
    // The re-rank shortcut pays when its partial-distance bound usually holds (uniform descriptors: 72 % of the attempts
    // decide the query) and costs when it rarely does (SIFT-shaped descriptors: the first 16 dimensions of a random pair
    // are too close for the bound, 0.5 %).  Every warp keeps score and stops trying once, after 64 attempts, fewer than
    // half have decided their query; a launch starts over.  Results never depend on it — only who computes them.
    uint32_t sc_try = 0, sc_ok = 0;

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
                mbar_expect_tx(&s_bar, bytes + obytes);
                for (uint32_t off = 0; off < bytes; off += 65536u)
                    bulk_g2s(s_raw + off, reinterpret_cast<const unsigned char*>(J.longs) + off,
                             min(65536u, bytes - off), &s_bar);
                for (uint32_t off = 0; off < obytes; off += 65536u)
                    bulk_g2s(s_raw + P.smem_long_bytes + off, reinterpret_cast<const unsigned char*>(J.offs) + off,
                             min(65536u, obytes - off), &s_bar);
            }
            mbar_wait(&s_bar, bar_parity);
            bar_parity ^= 1;
            resident = pd.slot_j;
        }

        // query range of this unit: chunks are multiples of 32 queries
        // (MODE 2 walks positions of the pair's active-query list instead of query indices)
        const uint32_t nq_unit = kActive ? __ldg(P.nact + pair) : I.n;
        const uint32_t qc = (((nq_unit + P.chunks_per_pair - 1) / P.chunks_per_pair) + 31u) & ~31u;
        const uint32_t q0 = min(nq_unit, chunk * qc), q1 = min(nq_unit, q0 + qc);
        const uint16_t* __restrict__ act = kActive ? P.act + pd.act_off : nullptr;
        uint32_t qa_lane = 0;  // MODE 2: the query index behind batch position `lane`
        const uint16_t* __restrict__ ids = CH_IDS(J);

        uint32_t st_raw = 0, st_vq = 0, st_dist = 0, st_match = 0;

        if (J.n == 0) {
            if (MODE == kModeMatch)  // (kModeMatchActive: the scratch was initialised with "no match")
                for (uint32_t q = q0 + tid; q < q1; q += kMatchThreads) __stcs(P.res + pd.res_off + q, make_uint2(kNone, 0u));
        } else {
            // ---- 1. bucket lookup, kBatch queries at a time, one query per lane -------------------
            // (matcher.cpp:164-169).  Lane i resolves the L table ranges of the warp's (base+i)-th query
            // and parks them, with the query's long code, in the warp's staging area: the global-memory
            // round trip for the query-side data is paid once per batch, not once per query.
            auto lookup_batch = [&](uint32_t qb) {
                const uint32_t qpos = qb + lane * kWarps;
                const bool live = lane < kBatch && qpos < q1;
                uint32_t q = qpos;
                if (kActive) {
                    q = live ? uint32_t(__ldg(act + qpos)) : 0u;
                    qa_lane = q;
                }
                if (live) {
                    const uint32_t* __restrict__ qcodes = I.shorts + uint64_t(q) * L;
                    const uint32_t rec = s_stage + lane * kRec;
                    sts128(rec, __ldg(I.longs + q));
                    uint32_t total = 0, pre = 0, empty = 0, nseg = 0, m0 = 0, m1 = 0, m2 = 0;
#pragma unroll
                    for (int t = 0; t < LT; ++t) {
                        uint32_t a = 0, b = 0;
                        if (EXACT || t < int(L)) {
                            const uint32_t code = __ldg(qcodes + t);
                            if (SMEM_TRAIN) {
                                const uint2 o = lds64x(s_offs + (t * nb1 + code) * 4u);
                                a = o.x;
                                b = o.y;
                            } else {
                                const uint32_t* o = J.offs + t * nb1 + code;
                                a = __ldg(o);
                                b = __ldg(o + 1);
                            }
                        }
                        const uint32_t len = b - a;
                        const uint32_t first = (EXACT || t < int(L)) ? t * J.n + a : 0u;  // unused slots: entry 0, discarded
                        total += len;
                        if (len == 0) empty |= 1u << t;
                        sts64(rec + 32u + t * 8u, first, first + max(len, 1u) - 1u);
                        if (len > 32u) {
                            sts32(rec + kAdj + nseg * 4u, first + 32u - pre);
                            ++nseg;
                            const uint32_t bit = 1u << (pre & 31u);
                            if (pre < 32u) m0 |= bit;
                            else if (pre < 64u) m1 |= bit;
                            else if (pre < 96u) m2 |= bit;
                            pre += len - 32u;
                        }
                    }
                    const uint32_t base1 = __popc(m0), base2 = base1 + __popc(m1);
                    sts128(rec + 16u, make_uint4(min(pre, 255u) | (empty << 8) | (base1 << 16) | (base2 << 24), m0, m1, m2));
                    if (!kActive) st_raw += total;  // per lane; reduced over the warp when the unit ends
                }
                __syncwarp();
            };
            // ids of the first 32 entries of each of a query's buckets, one per lane (lanes past the end
            // re-read the last entry: equal keys collapse)
            auto load_ids = [&](uint32_t rec, uint32_t (&out)[LT]) {
                static_for<LT>([&](auto T) {
                    constexpr int t = decltype(T)::value;
                    const uint2 fl = lds64_at<32u + t * 8u>(rec);
                    out[t] = __ldg(ids + min(fl.x + lane, fl.y));
                });
            };

            uint32_t idn[LT];  // prefetched ids of the NEXT query
            uint32_t q = q0 + warp;
            if (q < q1) {
                lookup_batch(q);
                load_ids(s_stage, idn);
            }
            for (uint32_t j = 0; q < q1; ++j, q += kWarps) {
                const uint32_t slot = j & (kBatch - 1);
                const uint32_t rec = s_stage + slot * kRec;
                uint32_t out_t = kNone, out_d = 0;
                const uint4 ql = lds128_at<0>(rec);
                const uint4 hdr = lds128_at<16>(rec);  // tover | empty << 8 | base1 << 16 | base2 << 24, M0, M1, M2
                const uint32_t tover = hdr.x & 0xffu;
                uint32_t id[LT];
#pragma unroll
                for (int t = 0; t < LT; ++t) id[t] = idn[t];
                // the next query's ids travel while this one is scanned, ranked and verified
                if (slot != kBatch - 1 && q + kWarps < q1) load_ids(rec + kRec, idn);

                uint32_t mykey = kNone;  // lane r holds the r-th ranked key
                uint32_t n = 0;          // ranked count
                bool decided = false;    // the re-rank shortcut has produced the record (out_t, out_d): no verification
#ifdef CHGPU_SHORTCUT_STATS
                bool attempted = false;
#endif
                // GUIDED: the band can only remove candidates, so a query whose UNFILTERED smallest key is beyond tau
                // ranks nothing either way; the line and the filter are evaluated only for the others.
                EpiLine line{};

                constexpr bool skip = false;
                bool emit = MODE == kModeTileTopK;  // this (query, tile) writes its list
                const uint32_t qa = kActive ? __shfl_sync(FULL, qa_lane, slot) : q;  // the query's index
                if (skip) {
                } else if (tover <= 32u * kOverSlots) {
                    // ---- 2. Hamming scan: the first 32 entries of every bucket, one table per slot,
                    //         then the entries past 32 of all buckets flattened into the last slots
                    uint32_t key[KS];
#pragma unroll
                    for (int s = 0; s < kOverSlots; ++s) key[LT + s] = kNone;
                    if (tover != 0) {
                        // id for now; its key below.  r + adj is a u32 sum (adj never wraps: pre < first + 32)
                        const uint32_t seg_mask[3] = {hdr.y, hdr.z, hdr.w};
                        {
                            const uint32_t seg = __popc(seg_mask[0] & le_mask) - 1u;
                            const uint32_t r = min(lane, tover - 1u);
                            key[LT] = __ldg(ids + uint32_t(r + lds32(rec + kAdj + seg * 4u)));
                        }
                        if (tover > 32u) {  // a second / third overflow step is rare: keep it out of line
#pragma unroll
                            for (int s = 1; s < kOverSlots; ++s) {
                                if (uint32_t(s) * 32u < tover) {
                                    const uint32_t base = (hdr.x >> (8 + 8 * s)) & 0xffu;
                                    const uint32_t seg = base + __popc(seg_mask[s] & le_mask) - 1u;
                                    const uint32_t r = min(uint32_t(s) * 32u + lane, tover - 1u);
                                    key[LT + s] = __ldg(ids + uint32_t(r + lds32(rec + kAdj + seg * 4u)));
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int t = 0; t < LT; ++t) key[t] = key_of<SMEM_TRAIN>(id[t], ql, s_long, J.longs);
                    if ((hdr.x & 0xff00u) != 0) {  // empty buckets (rare)
#pragma unroll
                        for (int t = 0; t < LT; ++t)
                            if (hdr.x & (0x100u << t)) key[t] = kNone;
                    }
                    // nested: half of the queries have at most one overflow step and leave through one branch
                    if (tover != 0) {
                        key[LT] = key_of<SMEM_TRAIN>(key[LT], ql, s_long, J.longs);
                        if (kOverSlots > 1 && tover > 32u) {
                            key[LT + 1] = key_of<SMEM_TRAIN>(key[LT + 1], ql, s_long, J.longs);
                            if (kOverSlots > 2 && tover > 64u)
                                key[LT + kOverSlots - 1] = key_of<SMEM_TRAIN>(key[LT + kOverSlots - 1], ql, s_long, J.longs);
                        }
                    }
                    // ---- 3. ranking: pull straight out of the slots -------------------------------
                    uint32_t k0 = first_key(key, kNone);
                    if (GUIDED && (MODE == kModeTileTopK || (k0 >> 24) <= P.tau)) {
                        line = epipolar_band(P.fmats + uint64_t(pd.pair_idx) * 9, __ldg(I.kp + qa));
#pragma unroll
                        for (int i = 0; i < KS; ++i) key[i] = band_filter(key[i], line, J.kp, P.band_px);
                        k0 = first_key(key, kNone);
                    }
                    if (MODE == kModeTileMin) {
                        if (lane == 0 && k0 != kNone) atomicMin(P.gmin + pd.res_off + q, k0);
                        // the tile itself has a candidate within tau (guided runs filter first: top-k pass only)
                        emit = (k0 >> 24) <= P.tau && P.fmats == nullptr;
                    }
                    if (MODE == kModeTileMin && !emit) {
                    } else if (!kMatch) {
                        // the tile's top_k smallest distinct keys, whatever their distance
                        uint32_t prev = k0;
                        while (prev != kNone) {
                            if (lane == n) mykey = prev;
                            if (++n == P.top_k) break;
                            prev = next_key(key, kNone, prev);
                        }
                    } else if ((k0 >> 24) <= P.tau) {
                        if (lane == 0) mykey = k0;
                        n = 1;
                        // keys within tau, in order (usually this loop ends at its first pull)
                        uint32_t a1;  // this lane's own smallest key above k0
#ifndef CHGPU_NO_RERANK_SHORTCUT
                        const FirstRow first = load_first_row(I.desc, J.desc, qa, k0, lane);  // travels under the first pull
#endif
                        uint32_t nk = next_key_keep(key, k0, a1);
#ifndef CHGPU_NO_RERANK_SHORTCUT
                        // one candidate within tau, more beyond it: the re-rank case; most of these are decided without
                        // pulling the other top_k - 1 keys (not in the ranked-list instantiation, which reports them)
#ifdef CHGPU_SHORTCUT_STATS
                        attempted = !DBG && nk != kNone && (nk >> 24) > P.tau;
#endif
                        if (!DBG && nk != kNone && (nk >> 24) > P.tau && (sc_try < 64u || 2u * sc_ok >= sc_try)) {
                            ++sc_try;
                            if (rerank_shortcut(key, k0, a1, P.top_k, first, J.desc, lane, P.ratio_sq, out_t, out_d)) {
                                ++sc_ok;
                                decided = true;
                                n = P.top_k;
                            }
                        }
#endif
                        if (!decided) {
                            while ((nk >> 24) <= P.tau) {  // (beyond the threshold, or kNone: no key left)
                                if (lane == n) mykey = nk;
                                if (++n == P.top_k) break;
                                nk = next_key(key, kNone, nk);
                            }
                            // the threshold cut something and the ranking is too small: re-rank without it
                            if (n < P.top_k && nk != kNone && n < P.min_ranked) {
                                do {
                                    if (lane == n) mykey = nk;
                                    ++n;
                                    if (n == P.top_k) break;
                                    nk = next_key(key, kNone, nk);
                                } while (nk != kNone);
                            }
                        }
                    }
                } else {
                    // ---- long buckets: rounds of 32 entries per table ----------------------------
                    uint32_t maxlen = 0;
                    uint32_t lo[LT], len[LT];
                    static_for<LT>([&](auto T) {
                        constexpr int t = decltype(T)::value;
                        const uint2 fl = lds64_at<32u + t * 8u>(rec);
                        lo[t] = fl.x;
                        len[t] = (hdr.x & (0x100u << t)) ? 0u : fl.y - fl.x + 1u;
                        maxlen = max(maxlen, len[t]);
                    });
                    // pass 1: smallest and largest key only — most queries have nothing within tau
                    uint32_t lmin = kNone, lmax = 0;
                    for (uint32_t off = 0; MODE != kModeTileTopK && off < maxlen; off += 32u) {
#pragma unroll
                        for (int t = 0; t < LT; ++t)
                            if (off < len[t]) {
                                const uint32_t k = scan_step<SMEM_TRAIN>(ids, lo[t] + off, lo[t] + len[t] - 1u, lane, ql,
                                                                         s_long, J.longs);
                                lmin = min(lmin, k);  // GUIDED: unfiltered (lmax is then taken in pass 2)
                                if (k != kNone) lmax = max(lmax, k);
                            }
                    }
                    const uint32_t gmin = __reduce_min_sync(FULL, lmin);
                    if (MODE == kModeTileMin) {
                        if (lane == 0 && gmin != kNone) atomicMin(P.gmin + pd.res_off + q, gmin);
                        emit = (gmin >> 24) <= P.tau && P.fmats == nullptr;
                    }
                    if (MODE == kModeTileMin && !emit) {
                    } else if (!kMatch || (gmin >> 24) <= P.tau) {
                        // pass 2: merge every round into the running top-k (ascending, unique)
                        if (GUIDED) {
                            line = epipolar_band(P.fmats + uint64_t(pd.pair_idx) * 9, __ldg(I.kp + qa));
                            lmax = 0;
                        }
                        for (uint32_t off = 0; off < maxlen; off += 32u) {
                            uint32_t key[LT];
#pragma unroll
                            for (int t = 0; t < LT; ++t) {
                                key[t] = kNone;
                                if (off < len[t]) {
                                    key[t] = scan_step<SMEM_TRAIN>(ids, lo[t] + off, lo[t] + len[t] - 1u, lane, ql, s_long,
                                                                   J.longs);
                                    if (GUIDED) {
                                        key[t] = band_filter(key[t], line, J.kp, P.band_px);
                                        if (key[t] != kNone) lmax = max(lmax, key[t]);
                                    }
                                }
                            }
                            // a round whose smallest key is beyond a full list's last entry changes nothing
                            const uint32_t kth = __shfl_sync(FULL, mykey, P.top_k - 1);
                            uint32_t prev = first_key(key, kNone);
                            if (prev > kth) continue;
                            const uint32_t old = mykey;
                            prev = min(prev, __shfl_sync(FULL, old, 0));
                            mykey = kNone;
                            for (uint32_t r = 0; r < P.top_k && prev != kNone; ++r) {
                                if (lane == r) mykey = prev;
                                prev = next_key(key, old, prev);
                            }
                        }
                        // thresholded size s, unique total (<= k); fallback rule as in the single-round path
                        const bool anycut = (__reduce_max_sync(FULL, lmax) >> 24) > P.tau;
                        const uint32_t tot = __popc(__ballot_sync(FULL, mykey != kNone));
                        const uint32_t s = __popc(__ballot_sync(FULL, mykey != kNone && (mykey >> 24) <= P.tau));
                        n = (kMatch && (s >= P.min_ranked || !anycut)) ? s : tot;
                        if (GUIDED && kMatch && s == 0) n = 0;  // the band removed everything within tau: no ranking, no fallback
                    }
                }

                if (!kMatch && emit) {
                    if (lane < P.top_k)
                        P.lists[(pd.res_off + qa) * P.list_stride + pd.tile_idx * P.top_k + lane] = lane < n ? mykey + pd.tile_base : kNone;
                    if (MODE == kModeTileMin && lane == 0) atomicOr(P.gdone + pd.res_off + q, 1ull << pd.tile_idx);
                }

                if (DBG && kMatch) {
                    if (lane < n) P.dbg_ranked[uint64_t(qa) * P.top_k + lane] = mykey & 0xffffffu;
                    if (lane == 0) P.dbg_count[qa] = n;
                }

                // ---- 4. verification (euclidean_verify, matcher.cpp:115-137) ------------------
#ifdef CHGPU_SHORTCUT_STATS
                // experiment (scripts/exp7.sh): verified_queries = re-rank cases, distances = count checks passed, matches of
                // the pair counts = accepted by the shortcut
                if (kMatch && attempted) {
                    st_vq += 1;
                    st_dist += (decided || out_d == 1) ? 1 : 0;
                    st_match += decided ? 1 : 0;
                }
                if (false) {
#else
                if (kMatch && n >= 2) {
#endif
                    st_vq += 1;
                    st_dist += n;
                    if (decided || verify_ranked(I.desc, J.desc, qa, n, mykey, lane, P.ratio_sq, out_t, out_d)) st_match += 1;
                }
                if (kMatch && lane == 0) __stcs(P.res + pd.res_off + qa, make_uint2(out_t, out_d));

                // batch boundary: resolve the next kBatch queries (this one's ranges are in registers)
                if (slot == kBatch - 1 && q + kWarps < q1) {
                    __syncwarp();
                    lookup_batch(q + kWarps);
                    load_ids(s_stage, idn);
                }
            }
        }

        st_raw = __reduce_add_sync(FULL, st_raw);
        if (lane == 0) {
            if (st_raw) atomicAdd(&P.stats->raw_candidates, (unsigned long long)st_raw);
            if (st_vq) atomicAdd(&P.stats->verified_queries, (unsigned long long)st_vq);
            if (st_dist) atomicAdd(&P.stats->distances, (unsigned long long)st_dist);
            if (st_match) atomicAdd(&P.pair_counts[pair], st_match);
        }
        __syncthreads();  // all warps done with the train tile / s_unit before the next unit
    }
}

// Merge + verification for tiled train images: one warp per query of the pair.  The query's T lists
// (T = tiles of the train image, top_k keys each, global ids, kNone padded) are merged 32 entries at a time
// into the ascending, duplicate-free top_k — the ranked list the reference builds over the whole image —
// then cut by the threshold / re-rank rule (matcher.cpp:176-189) and verified (matcher.cpp:106-137).
// Whether the threshold cut anything can be read off the lists: a tile with a candidate beyond tau that is
// not in its list has a full list within tau, and then the merged ranking is full as well.
// The queries the top-k pass visits for every (query image, tile) pair: gmin within tau and the tile's list not
// yet written by the min pass.  One warp per pair, ballot compaction in query order.
template <int kInstance>
__global__ void __launch_bounds__(256) tile_compact_kernel(const MatchParams P, uint32_t ntile_pairs) {
    // one CTA per (query image, tile) pair: every warp takes a contiguous run of the queries (a multiple of 32), counts its
    // active ones, the CTA turns the counts into offsets, and the warp writes its part of the list in query order
    __shared__ uint32_t s_count[8];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tp = blockIdx.x;
    if (tp >= ntile_pairs) return;
    const PairDesc pd = P.pairs[tp];
    const uint32_t nq = P.images[pd.slot_i].n;
    const uint32_t run = ((nq + 8u * 32u - 1u) / (8u * 32u)) * 32u;
    const uint32_t q0 = min(nq, warp * run), q1 = min(nq, q0 + run);
    auto active = [&](uint32_t q) {
        return q < q1 && (__ldg(P.gmin + pd.res_off + q) >> 24) <= P.tau && !((__ldg(P.gdone + pd.res_off + q) >> pd.tile_idx) & 1ull);
    };
    uint32_t count = 0;
    for (uint32_t q = q0; q < q1; q += 32) count += __popc(__ballot_sync(0xffffffffu, active(q + lane)));
    if (lane == 0) s_count[warp] = count;
    __syncthreads();
    uint32_t base = 0, total = 0;
#pragma unroll
    for (uint32_t w = 0; w < 8; ++w) {
        const uint32_t c = s_count[w];
        if (w < warp) base += c;
        total += c;
    }
    uint16_t* __restrict__ out = P.act + pd.act_off + base;
    uint32_t at = 0;
    for (uint32_t q = q0; q < q1; q += 32) {
        const bool f = active(q + lane);
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (f) out[at + __popc(bal & ((1u << lane) - 1u))] = uint16_t(q + lane);
        at += __popc(bal);
    }
    if (threadIdx.x == 0) P.nact[tp] = total;
}

// Ascending bitonic sort of one value per lane (kNone sinks to the top lanes), and the last stage alone for a
// sequence that is already bitonic.
__device__ __forceinline__ uint32_t warp_bitonic_merge32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (uint32_t j = 16; j > 0; j >>= 1) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
        v = (lane & j) == 0 ? min(v, o) : max(v, o);
    }
    return v;
}
__device__ __forceinline__ uint32_t warp_sort32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (uint32_t k = 2; k < 32; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
            const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
            v = keep_min ? min(v, o) : max(v, o);
        }
    }
    return warp_bitonic_merge32(v, lane);
}

constexpr int kMergeThreads = 256;
constexpr uint32_t kMergeChunk = 1024;  // queries per CTA
template <int kInstance>
__global__ void __launch_bounds__(kMergeThreads) tile_merge_kernel(const MatchParams P) {
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t pair = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const PairDesc pd = P.pairs[pair];
    const DevImage I = P.images[pd.slot_i];
    const DevImage J = P.images[pd.slot_j];
    const uint32_t q0 = blockIdx.y * kMergeChunk, q1 = min(I.n, q0 + kMergeChunk);
    const uint32_t entries = ((J.n + P.tile_points - 1) / P.tile_points) * P.top_k;
    uint32_t st_vq = 0, st_dist = 0, st_match = 0;
    for (uint32_t q = q0 + warp; q < q1; q += kMergeThreads / 32) {
        uint32_t out_t = kNone, out_d = 0, n = 0, mykey = kNone;
        if ((__ldg(P.gmin + pd.res_off + q) >> 24) <= P.tau) {
            const uint32_t* __restrict__ list = P.lists + (pd.res_off + q) * P.list_stride;
            // keys of different tiles differ in the id and a tile's list has no duplicates: a plain sort merges them.
            // 32 entries per round, one per lane: sort the round, keep the 32 smallest of it and the running list
            // (min(a[l], b[31 - l]) is bitonic), re-sort that with the last bitonic stage.
            bool cut = false;
            for (uint32_t e0 = 0; e0 < entries; e0 += 32) {
                const uint32_t v = e0 + lane < entries ? __ldg(list + e0 + lane) : kNone;
                cut |= v != kNone && (v >> 24) > P.tau;
                const uint32_t sorted = warp_sort32(v, lane);
                if (e0 == 0) {
                    mykey = sorted;
                } else {
                    const uint32_t mirrored = __shfl_sync(FULL, sorted, 31u - lane);
                    mykey = warp_bitonic_merge32(min(mykey, mirrored), lane);
                }
            }
            if (lane >= P.top_k) mykey = kNone;
            const bool anycut = __any_sync(FULL, cut);
            const uint32_t tot = __popc(__ballot_sync(FULL, mykey != kNone));
            const uint32_t s = __popc(__ballot_sync(FULL, mykey != kNone && (mykey >> 24) <= P.tau));
            n = (s >= P.min_ranked || !anycut) ? s : tot;
            if (s == 0) n = 0;  // guided runs: the band removed everything within tau (no ranking, no fallback)
        }
        if (P.dbg_ranked != nullptr) {
            if (lane < n) P.dbg_ranked[uint64_t(q) * P.top_k + lane] = mykey & 0xffffffu;
            if (lane == 0) P.dbg_count[q] = n;
        }
        if (n >= 2) {
            st_vq += 1;
            st_dist += n;
            if (verify_ranked(I.desc, J.desc, q, n, mykey, lane, P.ratio_sq, out_t, out_d)) st_match += 1;
        }
        if (lane == 0) __stcs(P.res + pd.res_off + q, make_uint2(out_t, out_d));
    }
    if (lane == 0) {
        if (st_vq) atomicAdd(&P.stats->verified_queries, (unsigned long long)st_vq);
        if (st_dist) atomicAdd(&P.stats->distances, (unsigned long long)st_dist);
        if (st_match) atomicAdd(&P.pair_counts[pair], st_match);
    }
}

}  // namespace chgpu
