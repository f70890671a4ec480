// join_kernels.cuh — K3j, the tensor-core Hamming pass in front of the match kernel.
//
// 64 % of the queries of a pair have no candidate within the Hamming threshold tau and leave the match kernel after a
// full scan of their buckets (matcher.cpp:164-175: no ranking, no verification, no record).  K3j finds out WHICH queries
// those are without visiting them one by one: a candidate of query q in table t is a train point with the same bucket
// code, so the candidate evaluations of a pair are the L * 2^m bucket-by-bucket cross products  queries(t, b) x
// train(t, b)  — small dense blocks of Hamming distances, which is matrix work:
//
//     |a AND b| for all pairs of a block  =  A B^T  over u8 operands  A[q][k] = bit k of a_q * 2^j(k),
//                                                                      B[c][k] = bit k of b_c * 2^(7 - j(k))
//     hamming(a, b) = popc(a) + popc(b) - 2 |a AND b|                  (products 2^7 where both bits are set)
//
// on the integer tensor-core path (mma.sync m16n8k32 u8 x u8 -> s32, SASS IMMA.16832.U8.U8; exact).  The operands are
// made in registers from the bucket-sorted code copies of the two images (DevImage::scodes): one LOP3 per fragment
// register — A = x & (0x01010101 << j), B = y' & (0x01010101 << (7 - j)) with y' = y with the bits of every byte
// reversed, stored next to y — so a byte of A is 0 or 2^j, the byte of B at the same K position 0 or 2^(7-j).  The K
// order is free as long as A and B agree.  No shared memory, no block-level synchronisation: one warp per bucket.
//
// Output: hit[q] = 1 iff some candidate of q has Hamming distance <= tau (a byte per query, set by whichever bucket finds
// one).  join_compact_kernel turns the flags of every pair into the ascending list of its hit queries, and the match
// kernel (MODE kModeMatchActive) runs lookup / scan / ranking / verification for those only; all other queries keep the
// "no match" the result scratch was initialised with.  The raw-candidate statistic (sum of |queries| x |train| over the
// buckets = sum over the queries of their bucket sizes, matcher.cpp:168) is accumulated here.
#pragma once

#include "dev_types.cuh"

namespace chgpu {

struct JoinParams {
    const DevImage* images;
    const PairDesc* pairs;
    uint32_t npairs;
    uint32_t m, L, tau;
    uint8_t* hit;            // per query of the sub-batch (PairDesc::res_off + q): set to 1, or ...
    uint32_t* hit_key;       // ... (tiled train images) the per-query minimum-key scratch of the tile passes, set to 0
    DevStats* stats;
    unsigned int* counter;   // work counter (units of 32 buckets)
};

#ifndef CHGPU_JOIN_OCC
#define CHGPU_JOIN_OCC 3
#endif
constexpr int kJoinThreads = 256;

__device__ __forceinline__ void mma_u8_16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                             uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One pass of join_bucket: MT m16 tiles of query rows (rows g + 8 j of the pass, j < 2 MT) against all train columns in
// tiles of 8.  Every tile of 8 columns is one 128-byte line of the reversed copies: the thread takes its column's code with
// one load (the bucket's lines were prefetched into L1 when the bucket was opened) and the popcounts of the two columns it
// receives with two byte loads.
template <int MT>
__device__ __forceinline__ void join_pass(const uint4* __restrict__ qc, const int16_t* __restrict__ qp,
                                          const uint16_t* __restrict__ qi, uint32_t r0, uint32_t nq,
                                          const uint4* __restrict__ tr, const int16_t* __restrict__ tp, uint32_t nt, int tau,
                                          uint8_t* __restrict__ hit, uint32_t* __restrict__ hit_key, uint32_t g, uint32_t tq) {
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t ma0 = 0x01010101u << (2u * tq), ma1 = ma0 << 1;   // A: bits 2tq, 2tq + 1 of every byte, value 2^j
    const uint32_t mb0 = 0x80808080u >> (2u * tq), mb1 = mb0 >> 1;   // B (bit-reversed bytes): the same bits, value 2^(7-j)
    uint32_t alo[2 * MT][4], ahi[2 * MT][4];  // [row slot][K step]: the row's word s masked to bits 2tq / 2tq + 1
    int thr[2 * MT], best[2 * MT];
#pragma unroll
    for (int j = 0; j < 2 * MT; ++j) {
        const uint32_t r = min(r0 + g + 8u * j, nq - 1);
        const uint4 x = __ldg(qc + r);
        // hamming <= tau  <=>  128 |a AND b| - 64 popc(b) >= 64 (popc(a) - tau)
        thr[j] = int(__ldg(qp + r)) - tau;  // spop holds 64 popc; tau comes in as 64 tau
        best[j] = int(0x80000000u);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            alo[j][s] = xw[s] & ma0;
            ahi[j][s] = xw[s] & ma1;
        }
    }
    const uint4* __restrict__ trp = tr + g;        // this thread's column of the tile
    const int16_t* __restrict__ tpp = tp + 2u * tq;  // the two columns whose results it receives
    const int left_c = int(nt) - int(g), left_a = int(nt) - int(2u * tq);
    for (int c0 = 0; c0 < int(nt); c0 += 8, trp += 8, tpp += 8) {
        uint4 y = make_uint4(0, 0, 0, 0);
        if (c0 < left_c) y = __ldg(trp);
        // penalties 64 popc(b) of the two columns this thread receives (2tq, 2tq + 1); past the end: never a hit
        const int pen_a = c0 < left_a ? -int(__ldg(tpp)) : -(1 << 28);
        const int pen_b = c0 + 1 < left_a ? -int(__ldg(tpp + 1)) : -(1 << 28);
        const uint32_t yw[4] = {y.x, y.y, y.z, y.w};
        uint32_t blo[4], bhi[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            blo[s] = yw[s] & mb0;
            bhi[s] = yw[s] & mb1;
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            int acc[4] = {0, 0, 0, 0};
#pragma unroll
            for (int s = 0; s < 4; ++s)  // K step s = code word s: 32 K positions = its 32 bits
                mma_u8_16832(acc, alo[2 * mt][s], alo[2 * mt + 1][s], ahi[2 * mt][s], ahi[2 * mt + 1][s], blo[s], bhi[s]);
            best[2 * mt] = max(acc[0] + pen_a, best[2 * mt]);  // (one add-and-max each)
            best[2 * mt] = max(acc[1] + pen_b, best[2 * mt]);
            best[2 * mt + 1] = max(acc[2] + pen_a, best[2 * mt + 1]);
            best[2 * mt + 1] = max(acc[3] + pen_b, best[2 * mt + 1]);
        }
    }
    // the four threads of a group hold different columns of the same rows
#pragma unroll
    for (int j = 0; j < 2 * MT; ++j) {
        best[j] = max(best[j], __shfl_xor_sync(FULL, best[j], 1));
        best[j] = max(best[j], __shfl_xor_sync(FULL, best[j], 2));
    }
    // thread tq of the group reports row slots tq and tq + 4 (as far as the pass has them)
#pragma unroll
    for (int base = 0; base < 2 * MT; base += 4) {
        int mine = best[base], mythr = thr[base];
#pragma unroll
        for (int j = base + 1; j < base + 4 && j < 2 * MT; ++j)
            if (int(tq) + base == j) {
                mine = best[j];
                mythr = thr[j];
            }
        const uint32_t slot = uint32_t(base) + tq, row = r0 + g + 8u * slot;
        if (slot < uint32_t(2 * MT) && row < nq && mine >= mythr) {
            const uint32_t qid = __ldg(qi + row);
            if (hit_key != nullptr) hit_key[qid] = 0u;
            else hit[qid] = 1;
        }
    }
}

// One bucket: nq queries (bucket-sorted codes qc, popcounts qp, ids qi) against nt train points (byte-bit-reversed codes tr,
// popcounts tp).  Fragment coordinates: g = lane >> 2 (row / column inside a tile), tq = lane & 3 (K slice).  Buckets hold
// 32 +- 6 points: up to 48 query rows go through ONE pass of 1, 2 or 3 row tiles, so the train-side work is done once.
__device__ __forceinline__ void join_bucket(const uint4* __restrict__ qc, const int16_t* __restrict__ qp,
                                            const uint16_t* __restrict__ qi, uint32_t nq, const uint4* __restrict__ tr,
                                            const int16_t* __restrict__ tp, uint32_t nt, int tau, uint8_t* __restrict__ hit,
                                            uint32_t* __restrict__ hit_key, uint32_t lane) {
    // the bucket's train-side lines into L1 (nt x 16 bytes of codes, nt popcount bytes): one prefetch instruction
    if (lane * 8u < nt) asm volatile("prefetch.global.L1 [%0];" ::"l"(tr + lane * 8u));
    if (lane == 31) asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
    const uint32_t g = lane >> 2, tq = lane & 3;
    uint32_t r0 = 0;
#ifndef CHGPU_JOIN_MAXMT2
    while (nq - r0 > 48) {
        join_pass<2>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
        r0 += 32;
    }
    const uint32_t left = nq - r0;  // 1 .. 48 rows: one pass of 1, 2 or 3 tiles
    if (left > 32) join_pass<3>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
    else if (left > 16) join_pass<2>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
    else join_pass<1>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
#else
    // A/B switch: at most two row tiles per pass (32 A-fragment registers instead of 48); buckets of 33-48 rows stream the
    // train columns twice.  Measured: the same at 3 CTAs per SM (4.82 against 4.84 ms), slower at 4 (5.11 ms).
    while (nq - r0 > 32) {
        join_pass<2>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
        r0 += 32;
    }
    if (nq - r0 > 16) join_pass<2>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
    else join_pass<1>(qc, qp, qi, r0, nq, tr, tp, nt, tau, hit, hit_key, g, tq);
#endif
}

__global__ void __launch_bounds__(kJoinThreads, CHGPU_JOIN_OCC) join_hits_kernel(const JoinParams P) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nb = 1u << P.m, nb1 = nb + 1, cells = P.L * nb, chunks = (cells + 31) / 32;
    const uint64_t units = uint64_t(P.npairs) * chunks;
    unsigned long long raw = 0;
    for (;;) {
        unsigned long long unit = 0;
        if (lane == 0) unit = atomicAdd(P.counter, 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= units) break;
        const uint32_t pair = uint32_t(unit / chunks), chunk = uint32_t(unit % chunks);
        const PairDesc pd = P.pairs[pair];
        const DevImage I = P.images[pd.slot_i];
        const DevImage J = P.images[pd.slot_j];
        if (I.n == 0 || J.n == 0) continue;
        // lane l owns bucket cell 32 chunk + l of this pair: its ranges in both images
        const uint32_t cell = chunk * 32 + lane;
        uint32_t t = 0, qa = 0, nq = 0, ta = 0, nt = 0;
        if (cell < cells) {
            t = cell / nb;
            const uint32_t b = cell % nb;
            qa = __ldg(I.offs + t * nb1 + b);
            nq = __ldg(I.offs + t * nb1 + b + 1) - qa;
            ta = __ldg(J.offs + t * nb1 + b);
            nt = __ldg(J.offs + t * nb1 + b + 1) - ta;
        }
        raw += (unsigned long long)nq * nt;
        uint32_t todo = __ballot_sync(0xffffffffu, nq != 0 && nt != 0);
        const uint64_t rev = uint64_t(P.L) * J.n;  // the reversed copies follow the plain ones
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t bt = __shfl_sync(0xffffffffu, t, src), bqa = __shfl_sync(0xffffffffu, qa, src),
                           bnq = __shfl_sync(0xffffffffu, nq, src), bta = __shfl_sync(0xffffffffu, ta, src),
                           bnt = __shfl_sync(0xffffffffu, nt, src);
            const uint64_t qo = uint64_t(bt) * I.n + bqa, to = uint64_t(bt) * J.n + bta;
            join_bucket(I.scodes + qo, I.spop + qo, I.points + qo, bnq, J.scodes + rev + to, J.spop + to, bnt, int(64u * P.tau),
                        P.hit + pd.res_off, P.hit_key ? P.hit_key + pd.res_off : nullptr, lane);
        }
    }
    // sum over the queries of their bucket sizes (raw_candidates, matcher.cpp:168)
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) raw += __shfl_xor_sync(0xffffffffu, raw, d);
    if (lane == 0 && raw) atomicAdd(&P.stats->raw_candidates, raw);
}

// The hit flags of every pair -> the ascending list of its hit queries (PairDesc::act_off, u16) and their number.  One CTA
// per pair (eight warps over contiguous runs of the queries), ballot compaction in query order.
__global__ void __launch_bounds__(256) join_compact_kernel(const DevImage* __restrict__ images, const PairDesc* __restrict__ pairs,
                                                           uint32_t npairs, const uint8_t* __restrict__ hit,
                                                           uint16_t* __restrict__ act, uint32_t* __restrict__ nact) {
    // one CTA per pair: every warp counts the hits of a contiguous run of the queries, the CTA turns the counts into
    // offsets, and the warp writes its part of the list in query order
    __shared__ uint32_t s_count[8];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t pair = blockIdx.x;
    if (pair >= npairs) return;
    const PairDesc pd = pairs[pair];
    const uint32_t nq = images[pd.slot_i].n;
    const uint8_t* __restrict__ h = hit + pd.res_off;
    const uint32_t run = ((nq + 8u * 32u - 1u) / (8u * 32u)) * 32u;
    const uint32_t q0 = min(nq, warp * run), q1 = min(nq, q0 + run);
    uint32_t count = 0;
    for (uint32_t q = q0; q < q1; q += 32) count += __popc(__ballot_sync(0xffffffffu, q + lane < q1 && h[q + lane] != 0));
    if (lane == 0) s_count[warp] = count;
    __syncthreads();
    uint32_t base = 0, total = 0;
#pragma unroll
    for (uint32_t w = 0; w < 8; ++w) {
        const uint32_t c = s_count[w];
        if (w < warp) base += c;
        total += c;
    }
    uint16_t* __restrict__ out = act + pd.act_off + base;
    uint32_t at = 0;
    for (uint32_t q = q0; q < q1; q += 32) {
        const bool f = q + lane < q1 && h[q + lane] != 0;
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (f) out[at + __popc(bal & ((1u << lane) - 1u))] = uint16_t(q + lane);
        at += __popc(bal);
    }
    if (threadIdx.x == 0) nact[pair] = total;
}

}  // namespace chgpu
