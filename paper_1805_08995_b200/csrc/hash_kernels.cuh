// hash_kernels.cuh — descriptor staging, centering sums, hash codes (K1) and bucket build (K2).
//
// All arithmetic that decides a hash bit is fp64 in the reference's exact operation order
// (reduce_dot, hashing.hpp:24-43): products rounded individually (__dmul_rn, never FMA), the
// first 7-N_r halving rounds as a pairwise tree, the last 2^N_r partial sums serially.
#pragma once

#include "dev_types.cuh"

namespace chgpu {

// ---------------------------------------------------------------------------------------------
// K0: split the 144-byte AoS records of a CHFT blob (feature_io.hpp:82-89) into SoA.
// One 16-byte chunk per thread: chunk 0 of a record is the keypoint, chunks 1..8 the descriptor.
__global__ void chft_split_kernel(const uint4* __restrict__ records, uint32_t n,
                                  uint4* __restrict__ desc, uint4* __restrict__ kp) {
    const uint64_t total = uint64_t(n) * 9;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t p = uint32_t(i / 9), c = uint32_t(i % 9);
        const uint4 v = __ldg(records + i);
        if (c == 0) kp[p] = v;
        else desc[uint64_t(p) * 8 + (c - 1)] = v;
    }
}

// The same split over a list of blobs in one launch (background loads split a whole block at once):
// blockIdx.y = file, blockIdx.x strides over its 16-byte chunks.
struct SplitJob {
    const uint4* records;
    uint4* desc;
    uint4* kp;
    uint32_t n;
    uint32_t pad;
};
__global__ void chft_split_batch_kernel(const SplitJob* __restrict__ jobs) {
    const SplitJob j = jobs[blockIdx.y];
    const uint64_t total = uint64_t(j.n) * 9;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t p = uint32_t(i / 9), c = uint32_t(i % 9);
        const uint4 v = __ldg(j.records + i);
        if (c == 0) j.kp[p] = v;
        else j.desc[uint64_t(p) * 8 + (c - 1)] = v;
    }
}

// K0 fused with the centering sums (the streaming loader's per-file kernel): blocks of 288 threads = 32 records
// x 9 chunks, so a thread keeps its chunk position while it strides over the records and can hold the 16 column
// sums of its descriptor chunk in registers; one shared-memory and one global (u64) atomic pass per block.
constexpr int kSplitSumThreads = 288;
__global__ void __launch_bounds__(kSplitSumThreads)
chft_split_sums_kernel(const uint4* __restrict__ records, uint32_t n, uint4* __restrict__ desc, uint4* __restrict__ kp,
                       unsigned long long* __restrict__ sums /*128*/) {
    __shared__ unsigned int s_acc[kDim];
    if (threadIdx.x < kDim) s_acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t c = threadIdx.x % 9, r_in = threadIdx.x / 9;
    uint32_t acc[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) acc[b] = 0;
    for (uint32_t p = blockIdx.x * 32 + r_in; p < n; p += gridDim.x * 32) {  // <= 65536 records: 255 * rows < 2^32
        const uint4 v = __ldg(records + uint64_t(p) * 9 + c);
        if (c == 0) {
            kp[p] = v;
        } else {
            desc[uint64_t(p) * 8 + (c - 1)] = v;
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int b = 0; b < 16; ++b) acc[b] += (w[b >> 2] >> (8 * (b & 3))) & 0xffu;
        }
    }
    if (c != 0) {
#pragma unroll
        for (int b = 0; b < 16; ++b) atomicAdd(&s_acc[(c - 1) * 16 + b], acc[b]);
    }
    __syncthreads();
    if (threadIdx.x < kDim && s_acc[threadIdx.x]) atomicAdd(&sums[threadIdx.x], (unsigned long long)s_acc[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// Centering pass: exact integer column sums (CenteringAccumulator::add, hashing.cpp:52-57).
// Each lane owns 4 adjacent byte columns of the 128-byte row; a warp reads whole rows.
__global__ void centering_sums_kernel(const uint8_t* __restrict__ desc, uint32_t n,
                                      unsigned long long* __restrict__ sums /*128*/) {
    __shared__ unsigned int s_acc[kDim];
    if (threadIdx.x < kDim) s_acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // 255 * rows_per_block must stay below 2^32: rows_per_block <= 2^20 is enforced by the launcher.
    unsigned int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    const uint32_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;
    const uint32_t r0 = blockIdx.x * rows_per_block;
    const uint32_t r1 = min(n, r0 + rows_per_block);
    for (uint32_t r = r0 + warp; r < r1; r += nwarps) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(desc + uint64_t(r) * kDim) + lane);
        a0 += w & 0xff;
        a1 += (w >> 8) & 0xff;
        a2 += (w >> 16) & 0xff;
        a3 += w >> 24;
    }
    atomicAdd(&s_acc[lane * 4 + 0], a0);
    atomicAdd(&s_acc[lane * 4 + 1], a1);
    atomicAdd(&s_acc[lane * 4 + 2], a2);
    atomicAdd(&s_acc[lane * 4 + 3], a3);
    __syncthreads();
    if (threadIdx.x < kDim) atomicAdd(&sums[threadIdx.x], (unsigned long long)s_acc[threadIdx.x]);
}

// The same sums over a list of resident images in one launch: blockIdx.y = image, blockIdx.x = row slice.
__global__ void centering_sums_batch_kernel(const DevImage* __restrict__ images, const uint32_t* __restrict__ slots,
                                            unsigned long long* __restrict__ sums /*128*/) {
    __shared__ unsigned int s_acc[kDim];
    const DevImage img = images[slots[blockIdx.y]];
    const uint32_t n = img.n;
    const uint32_t rows_per_block = (n + gridDim.x - 1) / gridDim.x;   // <= 65536 rows: 255 * rows < 2^32
    const uint32_t r0 = blockIdx.x * rows_per_block;
    const uint32_t r1 = min(n, r0 + rows_per_block);
    if (r0 >= r1) return;
    if (threadIdx.x < kDim) s_acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (uint32_t r = r0 + warp; r < r1; r += nwarps) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(img.desc + uint64_t(r) * kDim) + lane);
        a0 += w & 0xff;
        a1 += (w >> 8) & 0xff;
        a2 += (w >> 16) & 0xff;
        a3 += w >> 24;
    }
    atomicAdd(&s_acc[lane * 4 + 0], a0);
    atomicAdd(&s_acc[lane * 4 + 1], a1);
    atomicAdd(&s_acc[lane * 4 + 2], a2);
    atomicAdd(&s_acc[lane * 4 + 3], a3);
    __syncthreads();
    if (threadIdx.x < kDim) atomicAdd(&sums[threadIdx.x], (unsigned long long)s_acc[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// K1: hash codes.  One CTA = 64 points x all planes; 8 warps, each lane owns 2 points
// (lane, lane+32) and each warp 2 planes of the current 16-plane chunk, so one pass of the
// reduction DAG evaluates 4 dots with 2+2 shared-memory operands per product group.
//
// Shared memory: cT[128][64] centered descriptors (fp64, component-major => conflict-free),
// hs[16][128] plane chunk (broadcast reads), pbits[64][kPlaneWords] result bits.
constexpr int kHashTilePoints = 64;
constexpr int kHashChunkPlanes = 16;
constexpr int kHashThreads = 256;
constexpr int kPlaneWords = (kMaxTables * 32 + 128 + 31) / 32;  // 12 words cover L*m + n <= 384 planes

constexpr size_t hash_smem_bytes() {
    return sizeof(double) * (kDim * kHashTilePoints + kHashChunkPlanes * kDim) +
           sizeof(uint32_t) * kHashTilePoints * kPlaneWords;
}

// Node of the reduction DAG.  value(W, X) = sums[X] after the halving round of width W:
//   value(128, X) = c[X] * h[X]                       (rounded product)
//   value(W, X)   = value(2W, X) + value(2W, X + W)    (sums[i] += sums[i + width])
template <int W, int X>
__device__ __forceinline__ void dag_node(const double* __restrict__ c, const double* __restrict__ h,
                                         double (&o)[4]) {
    if constexpr (W == kDim) {
        const double c0 = c[X * kHashTilePoints], c1 = c[X * kHashTilePoints + 32];
        const double h0 = h[X], h1 = h[kDim + X];
        o[0] = __dmul_rn(c0, h0);
        o[1] = __dmul_rn(c0, h1);
        o[2] = __dmul_rn(c1, h0);
        o[3] = __dmul_rn(c1, h1);
    } else {
        double a[4], b[4];
        dag_node<W * 2, X>(c, h, a);
        dag_node<W * 2, X + W>(c, h, b);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = __dadd_rn(a[i], b[i]);
    }
}

// Serial tail: acc = sums[0]; acc += sums[1..T-1]  with T = 2^N_r.
template <int T, int J>
__device__ __forceinline__ void dag_tail(const double* __restrict__ c, const double* __restrict__ h,
                                         double (&acc)[4]) {
    if constexpr (J < T) {
        double v[4];
        dag_node<T, J>(c, h, v);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = (J == 0) ? v[i] : __dadd_rn(acc[i], v[i]);
        dag_tail<T, J + 1>(c, h, acc);
    }
}

__device__ __forceinline__ uint32_t take_bits(const uint32_t* w, uint32_t start, uint32_t len) {
    const uint32_t idx = start >> 5, sh = start & 31;
    uint64_t v = w[idx];
    if (sh + len > 32) v |= uint64_t(w[idx + 1]) << 32;
    v >>= sh;
    return len >= 32 ? uint32_t(v) : uint32_t(v) & ((1u << len) - 1u);
}

template <int RR>
__global__ void __launch_bounds__(kHashThreads)
hash_codes_kernel(const DevImage* __restrict__ images, const uint32_t* __restrict__ slots,
                  const double* __restrict__ planes /* (L*m + n) x 128: short planes then long */,
                  const double* __restrict__ centering /* 128 */, uint32_t m, uint32_t L, uint32_t nlong,
                  const unsigned int* __restrict__ guard_count /* nullable */, uint32_t guard_cap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // Launched behind the filtered kernel (K1f below) as its overflow path: it only runs when the
    // queue of undecided dots did not hold them all.
    if (guard_count != nullptr && *guard_count <= guard_cap) return;
    double* cT = reinterpret_cast<double*>(smem_raw);
    double* hs = cT + kDim * kHashTilePoints;
    uint32_t* pbits = reinterpret_cast<uint32_t*>(hs + kHashChunkPlanes * kDim);

    const DevImage img = images[slots[blockIdx.y]];
    const uint32_t p0 = blockIdx.x * kHashTilePoints;
    if (p0 >= img.n) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nplanes = L * m + nlong;

    // Stage: c[x][p] = double(desc[p][x]) - centering[x]   (center_descriptor, hashing.cpp:72-78)
    for (uint32_t i = tid; i < kHashTilePoints * (kDim / 4); i += kHashThreads) {
        const uint32_t p = i >> 5, x4 = i & 31;  // 32 words per descriptor row
        uint32_t w = 0;
        if (p0 + p < img.n) w = __ldg(reinterpret_cast<const uint32_t*>(img.desc + uint64_t(p0 + p) * kDim) + x4);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t x = x4 * 4 + b;
            cT[x * kHashTilePoints + p] = __dsub_rn(double((w >> (8 * b)) & 0xff), __ldg(centering + x));
        }
    }
    for (uint32_t i = tid; i < kHashTilePoints * kPlaneWords; i += kHashThreads) pbits[i] = 0;

    const double* c = cT + lane;
    const double* h = hs + (2 * warp) * kDim;
    for (uint32_t g0 = 0; g0 < nplanes; g0 += kHashChunkPlanes) {
        __syncthreads();  // previous chunk consumed (and, first time, cT / pbits staged)
        for (uint32_t i = tid; i < kHashChunkPlanes * kDim; i += kHashThreads) {
            const uint32_t g = g0 + i / kDim;
            hs[i] = g < nplanes ? __ldg(planes + uint64_t(g) * kDim + (i % kDim)) : 0.0;
        }
        __syncthreads();
        double acc[4];
        dag_tail<(1 << RR), 0>(c, h, acc);
        // Bit = (dot > 0.0), ties give 0 (hashing.cpp:80-99).
        const uint32_t ga = g0 + 2 * warp, gb = ga + 1;
        if (ga < nplanes) {
            if (acc[0] > 0.0) atomicOr(&pbits[lane * kPlaneWords + (ga >> 5)], 1u << (ga & 31));
            if (acc[2] > 0.0) atomicOr(&pbits[(lane + 32) * kPlaneWords + (ga >> 5)], 1u << (ga & 31));
        }
        if (gb < nplanes) {
            if (acc[1] > 0.0) atomicOr(&pbits[lane * kPlaneWords + (gb >> 5)], 1u << (gb & 31));
            if (acc[3] > 0.0) atomicOr(&pbits[(lane + 32) * kPlaneWords + (gb >> 5)], 1u << (gb & 31));
        }
    }
    __syncthreads();

    // Pack: short code t = planes [t*m, t*m+m), bit j at 1u<<j (hashing.cpp:80-88);
    // long code bit j = plane L*m + j, word j/32 of the uint4 (hashing.cpp:90-99).
    if (tid < kHashTilePoints && p0 + tid < img.n) {
        const uint32_t p = p0 + tid;
        uint32_t w[kPlaneWords + 1];
#pragma unroll
        for (int i = 0; i < kPlaneWords; ++i) w[i] = pbits[tid * kPlaneWords + i];
        w[kPlaneWords] = 0;
        for (uint32_t t = 0; t < L; ++t) img.shorts[uint64_t(p) * L + t] = take_bits(w, t * m, m);
        uint32_t lw[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t first = k * 32;
            lw[k] = first < nlong ? take_bits(w, L * m + first, min(32u, nlong - first)) : 0u;
        }
        img.longs[p] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// ---------------------------------------------------------------------------------------------
// K1f: hash codes through an fp32 filter with an a-priori error bound; the default hash path.
//
// A hash bit is the sign of the reference's fp64 value r = reduce_dot(c, h) (hashing.hpp:24-43), and
// it has to be reproduced exactly.  Almost every |r| is ~10^3 while its sign only needs ~10^-1 of
// accuracy, so the bulk of the work runs as an fp32 SIMT contraction and only the dots the bound
// cannot decide are re-evaluated by hash_fixup_kernel in the exact fp64 operation DAG.
//
//   acc  = fl32( sum_x d_x * fl32(h_x) )        d_x = descriptor byte, exact in fp32; 128 FFMA
//   v    = double(acc) - bias_g                 bias_g = sum_x centering_x h_x (host, fp64)
//   E    = A_p * ||h_g||_2 + 1e-30              A_p = (136 * 2^-24 + 2^-44) ||d_p||_2 + 2^-44 ||centering||_2
//
// With x the exact real value of sum_x (d_x - centering_x) h_x:  |v - x| <= 132 u32 ||d|| ||h|| + 131 u64
// ||centering|| ||h|| + u64 |v|  (gamma_128 of the FFMA chain plus one rounding of every h_x, Cauchy-Schwarz
// on sum |d_x h_x|; the host's bias sum; the final subtraction) and |r - x| <= 131 u64 (||d|| + ||centering||)
// ||h||  (one rounding of c_x = d_x - centering_x, the rounded products and at most 127 additions on any
// path of the DAG, for every N_r).  E exceeds their sum, hence |v| > E implies r != 0 and sign(r) = sign(v).
// Everything else — ties included — goes to the queue.  The host refuses the filter (exact kernel only)
// for planes or centerings that are not finite or exceed 1e30 / 1e6 in magnitude.
//
// One CTA = 128 points x all planes in chunks of 64; thread tile 8 points x 4 planes (32 accumulators),
// operands from shared memory: dT[128][128] fp32 descriptors component-major, hT[128][64] plane chunk.
constexpr int kFiltPoints = 128;
constexpr int kFiltPlanes = 64;
constexpr int kFiltThreads = 256;

struct HashFilterParams {
    const DevImage* images;
    const uint32_t* slots;
    const float* planes_t;      // [128][gpad] fp32-rounded planes, component-major, zero padded
    const double* bias;         // [gpad]
    const double* hnorm;        // [gpad] ||h_g||_2, rounded up
    double a_rel, a_abs;        // A_p = a_rel * ||d_p|| + a_abs
    uint32_t gpad, m, L, nlong;
    uint2* queue;               // undecided dots: (slot, point << 16 | plane)
    uint32_t queue_cap;
    unsigned int* queue_count;  // entries wanted (may exceed queue_cap: overflow)
};

constexpr size_t hash_filter_smem_bytes() {
    return sizeof(float) * kDim * (kFiltPoints + kFiltPlanes) + sizeof(double) * kFiltPoints +
           sizeof(uint32_t) * kFiltPoints * (kPlaneWords + 1);
}

__global__ void __launch_bounds__(kFiltThreads, 2) hash_filter_kernel(const HashFilterParams P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* dT = reinterpret_cast<float*>(smem_raw);
    float* hT = dT + kDim * kFiltPoints;
    double* Ap = reinterpret_cast<double*>(hT + kDim * kFiltPlanes);
    uint32_t* pbits = reinterpret_cast<uint32_t*>(Ap + kFiltPoints);
    uint32_t* dn2 = pbits + kFiltPoints * kPlaneWords;

    const uint32_t slot = P.slots[blockIdx.y];
    const DevImage img = P.images[slot];
    const uint32_t p0 = blockIdx.x * kFiltPoints;
    if (p0 >= img.n) return;
    const uint32_t tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const uint32_t nplanes = P.L * P.m + P.nlong;

    for (uint32_t i = tid; i < kFiltPoints * (kPlaneWords + 1); i += kFiltThreads) pbits[i] = 0;  // pbits and dn2
    __syncthreads();
    {   // stage: lane <-> point, so the component-major stores are conflict-free; two threads share a row
        const uint32_t p = tid & (kFiltPoints - 1), half = tid >> 7;
        const bool live = p0 + p < img.n;
        const uint4* row = reinterpret_cast<const uint4*>(img.desc + uint64_t(live ? p0 + p : 0) * kDim) + half * 4;
        uint32_t ss = 0;
#pragma unroll
        for (uint32_t w = 0; w < 4; ++w) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (live) v = __ldg(row + w);
            const uint32_t words[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (uint32_t b = 0; b < 16; ++b) {
                const uint32_t byte = (words[b >> 2] >> (8 * (b & 3))) & 0xffu;
                dT[(half * 64 + w * 16 + b) * kFiltPoints + p] = float(byte);
                ss += byte * byte;
            }
        }
        atomicAdd(&dn2[p], ss);
    }
    __syncthreads();
    if (tid < kFiltPoints) Ap[tid] = __dadd_ru(__dmul_ru(P.a_rel, __dsqrt_ru(double(dn2[tid]))), P.a_abs);

    for (uint32_t g0 = 0; g0 < nplanes; g0 += kFiltPlanes) {
        __syncthreads();  // previous chunk consumed (first time: Ap written)
        for (uint32_t i = tid; i < kDim * (kFiltPlanes / 4); i += kFiltThreads) {
            const uint32_t k = i / (kFiltPlanes / 4), c4 = i % (kFiltPlanes / 4);
            reinterpret_cast<float4*>(hT)[i] = __ldg(reinterpret_cast<const float4*>(P.planes_t + uint64_t(k) * P.gpad + g0) + c4);
        }
        __syncthreads();
        float acc[8][4];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
        const float* dcol = dT + ty * 8;
        const float* hcol = hT + tx * 4;
#pragma unroll 8
        for (int k = 0; k < kDim; ++k) {
            const float4 a0 = *reinterpret_cast<const float4*>(dcol + k * kFiltPoints);
            const float4 a1 = *reinterpret_cast<const float4*>(dcol + k * kFiltPoints + 4);
            const float4 b = *reinterpret_cast<const float4*>(hcol + k * kFiltPlanes);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
        // decide: sign certain iff |v| > E
        const uint32_t g = g0 + tx * 4;
        double bj[4], hj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bj[j] = __ldg(P.bias + g + j);
            hj[j] = __ldg(P.hnorm + g + j);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t p = ty * 8 + i;
            const double A = Ap[p];
            uint32_t nib = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double v = __dsub_rn(double(acc[i][j]), bj[j]);
                const double E = __dadd_ru(__dmul_ru(A, hj[j]), 1e-30);
                if (v > 0.0) nib |= 1u << j;
                if (!(fabs(v) > E) && g + j < nplanes && p0 + p < img.n) {
                    const unsigned int at = atomicAdd(P.queue_count, 1u);
                    if (at < P.queue_cap) P.queue[at] = make_uint2(slot, ((p0 + p) << 16) | (g + j));
                }
            }
            if (nib) atomicOr(&pbits[p * kPlaneWords + (g >> 5)], nib << (g & 31));
        }
    }
    __syncthreads();

    // pack exactly as hash_codes_kernel does
    if (tid < kFiltPoints && p0 + tid < img.n) {
        const uint32_t p = p0 + tid;
        uint32_t w[kPlaneWords + 1];
#pragma unroll
        for (int i = 0; i < kPlaneWords; ++i) w[i] = pbits[tid * kPlaneWords + i];
        w[kPlaneWords] = 0;
        for (uint32_t t = 0; t < P.L; ++t) img.shorts[uint64_t(p) * P.L + t] = take_bits(w, t * P.m, P.m);
        uint32_t lw[4];
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t first = k * 32;
            lw[k] = first < P.nlong ? take_bits(w, P.L * P.m + first, min(32u, P.nlong - first)) : 0u;
        }
        img.longs[p] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

struct HashFilterStats {
    unsigned long long undecided;  // dots sent to the exact path
    unsigned long long flipped;    // of those, bits the fp32 sign had wrong
    unsigned long long overflows;  // batches whose queue overflowed (recomputed by hash_codes_kernel)
};

// Exact re-evaluation of the undecided dots: one thread per queue entry walks the reference DAG
// (center_descriptor hashing.cpp:72-78, reduce_dot hashing.hpp:24-43) and corrects the stored bit.
__global__ void hash_fixup_kernel(const DevImage* __restrict__ images, const double* __restrict__ planes,
                                  const double* __restrict__ centering, const uint2* __restrict__ queue,
                                  uint32_t queue_cap, const unsigned int* __restrict__ queue_count, uint32_t m,
                                  uint32_t L, int reduce_rounds, HashFilterStats* __restrict__ stats) {
    const uint32_t want = *queue_count, n = min(want, queue_cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(&stats->undecided, (unsigned long long)want);
        if (want > queue_cap) atomicAdd(&stats->overflows, 1ull);
    }
    const uint32_t tail = 1u << reduce_rounds;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const uint2 q = queue[e];
        const DevImage img = images[q.x];
        const uint32_t p = q.y >> 16, g = q.y & 0xffffu;
        const uint8_t* d = img.desc + uint64_t(p) * kDim;
        const double* h = planes + uint64_t(g) * kDim;
        double s[kDim];
        for (int x = 0; x < kDim; ++x) s[x] = __dmul_rn(__dsub_rn(double(d[x]), centering[x]), h[x]);
        for (uint32_t width = kDim / 2; width >= tail; width >>= 1)
            for (uint32_t i = 0; i < width; ++i) s[i] = __dadd_rn(s[i], s[i + width]);
        double acc = s[0];
        for (uint32_t j = 1; j < tail; ++j) acc = __dadd_rn(acc, s[j]);
        const uint32_t bit = acc > 0.0 ? 1u : 0u;
        uint32_t* word;
        uint32_t pos;
        if (g < L * m) {
            word = img.shorts + uint64_t(p) * L + g / m;
            pos = g % m;
        } else {
            const uint32_t j = g - L * m;
            word = reinterpret_cast<uint32_t*>(img.longs + p) + (j >> 5);
            pos = j & 31;
        }
        if (((*word >> pos) & 1u) != bit) {
            atomicXor(word, 1u << pos);
            atomicAdd(&stats->flipped, 1ull);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// K2: bucket build.  One CTA per image, one warp per table: a stable counting sort of the
// image's points by m-bit code (build_bucket_index, matcher.cpp:27-51).  Points are consumed
// in ascending id order 32 at a time; __match_any_sync ranks equal codes inside the step, a
// shared-memory cursor per bucket carries the running position, so ids inside a bucket come
// out ascending exactly as the reference's sort of (code, point) pairs leaves them.
__global__ void bucket_build_kernel(const DevImage* __restrict__ images, const uint32_t* __restrict__ slots,
                                    uint32_t m, uint32_t L) {
    extern __shared__ uint32_t s_cursor[];  // L x 2^m
    const DevImage img = images[slots[blockIdx.x]];
    const uint32_t lane = threadIdx.x & 31, t = threadIdx.x >> 5;
    if (t >= L) return;
    const uint32_t nb = 1u << m, n = img.n;
    uint32_t* cur = s_cursor + t * nb;
    for (uint32_t b = lane; b < nb; b += 32) cur[b] = 0;
    __syncwarp();

    // Pass 1: histogram.
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t p = base + lane;
        const bool valid = p < n;
        const uint32_t code = valid ? __ldg(img.shorts + uint64_t(p) * L + t) : kNone;
        const uint32_t peers = __match_any_sync(0xffffffffu, code);
        if (valid && (__ffs(peers) - 1) == int(lane)) cur[code] += __popc(peers);
        __syncwarp();
    }
    // Exclusive scan of the histogram -> CSR offsets; cursors restart at the bucket starts.
    uint32_t* offs = img.offs + uint64_t(t) * (nb + 1);
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
        const uint32_t b = b0 + lane;
        const uint32_t v = b < nb ? cur[b] : 0;
        uint32_t incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, d);
            if (int(lane) >= d) incl += u;
        }
        if (b < nb) {
            offs[b] = carry + incl - v;
            cur[b] = carry + incl - v;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) offs[nb] = n;
    __syncwarp();

    // Pass 2: stable placement.
    uint16_t* pts = img.points + uint64_t(t) * n;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t p = base + lane;
        const bool valid = p < n;
        const uint32_t code = valid ? __ldg(img.shorts + uint64_t(p) * L + t) : kNone;
        const uint32_t peers = __match_any_sync(0xffffffffu, code);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        uint32_t start = 0;
        if (valid) start = cur[code];
        __syncwarp();
        if (valid) {
            pts[start + rank] = uint16_t(p);
            if (rank == 0) cur[code] = start + __popc(peers);
        }
        __syncwarp();
    }

    // Bucket-sorted copies of the long codes for the join pass (join_kernels.cuh): entry p of this table = the code of point
    // pts[p], plain and with the bits of every byte reversed, and its popcount.
    if (img.scodes != nullptr) {
        __syncwarp();
        uint4* sc = img.scodes + uint64_t(t) * n;             // plain copies: L x n
        uint4* sr = img.scodes + uint64_t(L + t) * n;         // reversed copies behind them: L x n
        int16_t* sp = img.spop + uint64_t(t) * n;
        for (uint32_t p = lane; p < n; p += 32) {
            const uint4 c = img.longs[pts[p]];
            sc[p] = c;
            sr[p] = make_uint4(__byte_perm(__brev(c.x), 0, 0x0123), __byte_perm(__brev(c.y), 0, 0x0123),
                               __byte_perm(__brev(c.z), 0, 0x0123), __byte_perm(__brev(c.w), 0, 0x0123));
            sp[p] = int16_t(64 * (__popc(c.x) + __popc(c.y) + __popc(c.z) + __popc(c.w)));
        }
    }

    // Pass 3: scan order.  The match kernel gathers the 16-byte codes of 8 consecutive bucket entries
    // with one quarter-warp LDS.128; the gather is conflict-free iff their ids differ mod 8.  Entries are
    // re-dealt by (rank inside the residue class, residue): the first min-count rounds hold all 8
    // residues.  Only the order inside a bucket changes, which no result depends on.  One bucket per lane.
    uint16_t* scan = img.scan + uint64_t(t) * n;
    // The match kernel reads entry `first` of a query's bucket even when the bucket is empty (its key is discarded
    // afterwards); for an empty bucket at the very end of the last table that is entry L n, one past the lists.  The arena
    // hands out recycled blocks, so that slot must hold a valid point id and not whatever the block held before (an id
    // beyond the shared-memory window would fault in the code gather).
    if (t == L - 1 && lane == 0) img.scan[uint64_t(L) * n] = 0;
    for (uint32_t b = lane; b < nb; b += 32) {
        const uint32_t lo = offs[b], hi = offs[b + 1], s = hi - lo;
        if (s <= 8 || s >= 256) {  // one octet, or counts that do not fit the packed bytes: keep the order
            for (uint32_t e = lo; e < hi; ++e) scan[e] = pts[e];
            continue;
        }
        unsigned long long cnt = 0, seen = 0;  // 8 x 8-bit counters, one per residue
        for (uint32_t e = lo; e < hi; ++e) cnt += 1ull << (8u * (pts[e] & 7u));
        for (uint32_t e = lo; e < hi; ++e) {
            const uint32_t id = pts[e], r = id & 7u;
            const uint32_t k = uint32_t(seen >> (8u * r)) & 0xffu;
            uint32_t pos = 0;
#pragma unroll
            for (uint32_t r2 = 0; r2 < 8; ++r2) {
                const uint32_t c = uint32_t(cnt >> (8u * r2)) & 0xffu;
                pos += min(c, k) + ((r2 < r && c > k) ? 1u : 0u);
            }
            scan[lo + pos] = uint16_t(id);
            seen += 1ull << (8u * r);
        }
    }
}

}  // namespace chgpu
