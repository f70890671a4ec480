// hash_tc.cuh — K1t: the hash filter on the 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Same contract as K1f (hash_kernels.cuh): decide every hash bit whose sign can be PROVEN, queue the rest for the exact
// fp64 re-evaluation (hash_fixup_kernel), so the codes are the reference's bit for bit (hashing.cpp:130-149).  What changes
// is the arithmetic of the filter — integer, hence exact, instead of an fp32 FFMA chain:
//
//   h_x  ~  H_x / S_g        H_x = rint(h_x * S_g),  S_g = 2^(22 - e_g),  2^e_g > max_x |h_x|      (host, once per family)
//   H_x  =  65536 l0 + 256 l1 + l2      three balanced int8 limbs (l0 in [-64, 64], l1, l2 in [-128, 127])
//   A_k  =  sum_x d_x l_k(x)            u8 x s8 -> s32 on the tensor cores: |A_k| <= 128 * 255 * 128, exact
//   v    =  fl64( (65536 A_0 + 256 A_1 + A_2) / S_g - bias_g )          bias_g = sum_x centering_x h_x (host)
//
// With x the exact real value of sum_x (d_x - centering_x) h_x and D1 = sum_x d_x:
//   |v - x| <= D1 * 2^(e_g - 23)  (one rounding of every h_x to a multiple of 1/S_g)  +  2^-52 ||c|| ||h||  (the host's
//   bias)  +  2^-53 |v|  (the one rounding of the subtraction; everything before it is exact in fp64), and the
//   reference's own value r satisfies |r - x| <= 131 * 2^-53 (||d|| + ||c||) ||h||  (K1f's analysis, any N_r).
//   E = alpha_g * D1 + beta_g,  alpha_g = (2^(e_g-23) + 2^-45 ||h_g||)(1 + 2^-40),  beta_g = (2^-45 ||c|| ||h_g|| + 1e-30)
//   (1 + 2^-40), both rounded up, exceeds the sum (||d||_2 <= D1), so |v| > E implies r != 0 and sign(r) = sign(v).
// The bound is ~45x tighter than the fp32 filter's (its 136 * 2^-24 ||d|| ||h|| came from the FFMA chain): fewer dots go to
// the exact path.
//
// One persistent CTA per SM (8 warps).  Per CTA, once: the three limb matrices (N_pad x 128 bytes each) and the per-plane
// constants into shared memory.  Per tile of 128 points: the descriptors as they lie in HBM (128-byte rows) into the
// SWIZZLE_128B K-major operand layout; then passes of 64 planes: 3 limbs x 4 K steps of tcgen05.mma (M = 128, N = 64,
// K = 32) into a TMEM buffer of 3 x 64 columns, the next pass's MMAs issued into the other buffer before this pass's
// epilogue starts; tcgen05.ld (lane = point, column = plane) -> fp64 decision -> 32 hash bits per thread and pass.
#pragma once

#include "hash_kernels.cuh"

namespace chgpu {

constexpr int kTcPoints = 128;      // points per tile (MMA M)
constexpr int kTcPassPlanes = 64;   // planes per pass (MMA N)
constexpr int kTcThreads = 256;
constexpr int kTcMaxPlanes = 256;   // N_pad ceiling: L*m + n <= 8*12 + 128 = 224

struct HashTcParams {
    const DevImage* images;
    const uint32_t* slots;
    const int8_t* limbs;        // [3][npad][128] row-major: limb k of plane g, component x
    const double* inv_scale;    // [npad] 1 / S_g
    const double* bias;         // [npad]
    const double* alpha;        // [npad]
    const double* beta;         // [npad]
    uint32_t npad, m, L, nlong;
    uint32_t count, tiles_max;  // images in this launch, tiles of the largest one
    uint2* queue;               // undecided dots: (slot, point << 16 | plane)
    uint32_t queue_cap;
    unsigned int* queue_count;
};

__host__ __device__ constexpr size_t hash_tc_smem_bytes(uint32_t npad) {
    return 1024 /* alignment slack */ + size_t(3) * npad * kDim + size_t(kTcPoints) * kDim + size_t(4) * npad * sizeof(double) +
           size_t(kTcPoints) * (kPlaneWords + 1) * sizeof(uint32_t) + 64;
}

namespace tc {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major operand tile, rows of 128 bytes, SWIZZLE_128B: 8-row atoms of 1,024 bytes, 16-byte chunk c of row r at c ^ (r & 7)
__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 1024u + (row & 7u) * 128u + (((chunk ^ row) & 7u) << 4);
}
// shared-memory matrix descriptor (sm_100): start address >> 4, leading / stride byte offsets >> 4, version 1, layout type
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout_type) {
    uint64_t d = 0;
    d |= uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout_type) << 61;
    return d;
}
// kind::i8 instruction descriptor: D = s32, A = unsigned 8-bit (the descriptors), B = signed 8-bit (the limbs), both K-major
__host__ __device__ constexpr uint32_t make_idesc_u8s8(uint32_t M, uint32_t N) {
    return (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// Bounded wait: a protocol error must end the kernel (trap), never hang the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spin = 0; spin < (1u << 28); ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
    }
    __trap();
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
          "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
}  // namespace tc

__global__ void __launch_bounds__(kTcThreads, 1) hash_filter_tc_kernel(const HashTcParams P) {
    extern __shared__ unsigned char smem_dyn[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base_s;
    // carve: [B limbs: 3 x npad x 128 | A tile: 128 x 128 | constants: 4 x npad doubles | pbits | dsum]
    unsigned char* base = smem_dyn + ((1024u - (tc::smem_u32(smem_dyn) & 1023u)) & 1023u);
    unsigned char* sB = base;
    unsigned char* sA = sB + size_t(3) * P.npad * kDim;
    double* cst = reinterpret_cast<double*>(sA + size_t(kTcPoints) * kDim);  // inv_scale | bias | alpha | beta
    uint32_t* pbits = reinterpret_cast<uint32_t*>(cst + size_t(4) * P.npad);
    uint32_t* dsum = pbits + kTcPoints * kPlaneWords;

    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t nplanes = P.L * P.m + P.nlong;
    const uint32_t npass = P.npad / kTcPassPlanes;

    // ---- once per CTA: limbs (swizzled), constants, barriers, TMEM --------------------------------------------
    for (uint32_t i = tid; i < 3u * P.npad * 8u; i += kTcThreads) {
        const uint32_t k = i / (P.npad * 8u), rc = i % (P.npad * 8u), r = rc >> 3, c = rc & 7u;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(P.limbs + (size_t(k) * P.npad + r) * kDim) + c);
        *reinterpret_cast<uint4*>(sB + size_t(k) * P.npad * kDim + tc::swz128(r, c)) = v;
    }
    for (uint32_t i = tid; i < P.npad; i += kTcThreads) {
        cst[i] = __ldg(P.inv_scale + i);
        cst[P.npad + i] = __ldg(P.bias + i);
        cst[2 * P.npad + i] = __ldg(P.alpha + i);
        cst[3 * P.npad + i] = __ldg(P.beta + i);
    }
    if (tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(&tmem_base_s)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = tc::make_idesc_u8s8(kTcPoints, kTcPassPlanes);
    const uint32_t a_addr = tc::smem_u32(sA), b_addr = tc::smem_u32(sB);
    uint32_t parity0 = 0, parity1 = 0;

    // the MMAs of one pass: limb k accumulates over the four K steps into columns [buf * 256 + k * 64, + 64)
    auto issue_pass = [&](uint32_t pass) {
        const uint32_t buf = pass & 1u;
#pragma unroll
        for (uint32_t k = 0; k < 3; ++k) {
            const uint32_t brow = b_addr + (k * P.npad + pass * kTcPassPlanes) * kDim;
#pragma unroll
            for (uint32_t ks = 0; ks < 4; ++ks)
                tc::umma_i8(tmem + buf * 256u + k * 64u, tc::make_desc(a_addr + ks * 32u, 16, 1024, 2),
                            tc::make_desc(brow + ks * 32u, 16, 1024, 2), idesc, ks > 0);
        }
        tc::umma_commit(&bar[buf]);
    };

    const uint32_t units = P.count * P.tiles_max;
    for (uint32_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
        const uint32_t slot = P.slots[unit / P.tiles_max];
        const DevImage img = P.images[slot];
        const uint32_t p0 = (unit % P.tiles_max) * kTcPoints;
        if (p0 >= img.n) continue;  // (uniform over the CTA)

        // ---- A tile: descriptor rows as they lie in HBM -> swizzled K-major operand; D1 = sum of the bytes of a row ----
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            const uint32_t row = (tid >> 3) + 32u * k, c = tid & 7u;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (p0 + row < img.n) v = __ldg(reinterpret_cast<const uint4*>(img.desc + uint64_t(p0 + row) * kDim) + c);
            *reinterpret_cast<uint4*>(sA + tc::swz128(row, c)) = v;
            uint32_t s = __dp4a(v.x, 0x01010101u, 0u);
            s = __dp4a(v.y, 0x01010101u, s);
            s = __dp4a(v.z, 0x01010101u, s);
            s = __dp4a(v.w, 0x01010101u, s);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            if (c == 0) dsum[row] = s;
        }
        for (uint32_t i = tid; i < kTcPoints * kPlaneWords; i += kTcThreads) pbits[i] = 0;
        // generic-proxy writes of the operand -> visible to the tensor core's async-proxy reads
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

        if (tid == 0) issue_pass(0);
        const uint32_t row = 32u * (warp & 3u) + lane, half = warp >> 2;  // this thread's point and 32-plane half of a pass
        const bool live = p0 + row < img.n;
        const double d1 = double(dsum[row]);
        for (uint32_t pass = 0; pass < npass; ++pass) {
            const uint32_t buf = pass & 1u;
            // the other buffer is free (its epilogue ended at the barrier that closed the previous iteration)
            if (tid == 0 && pass + 1 < npass) issue_pass(pass + 1);
            if (buf == 0) {
                tc::mbar_wait(&bar[0], parity0);
                parity0 ^= 1u;
            } else {
                tc::mbar_wait(&bar[1], parity1);
                parity1 ^= 1u;
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t word = 0;
#pragma unroll
            for (uint32_t sub = 0; sub < 2; ++sub) {
                uint32_t a0[16], a1[16], a2[16];
                const uint32_t col = buf * 256u + half * 32u + sub * 16u;
                const uint32_t taddr = tmem + ((32u * (warp & 3u)) << 16) + col;
                tc::tmem_ld16(taddr, a0);
                tc::tmem_ld16(taddr + 64u, a1);
                tc::tmem_ld16(taddr + 128u, a2);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const uint32_t g0 = pass * kTcPassPlanes + half * 32u + sub * 16u;
#pragma unroll
                for (uint32_t j = 0; j < 16; ++j) {
                    const uint32_t g = g0 + j;
                    // 65536 A0 + 256 A1 + A2: every term and every partial sum is an integer below 2^53: exact
                    const double t = fma(double(int32_t(a0[j])), 65536.0, fma(double(int32_t(a1[j])), 256.0, double(int32_t(a2[j]))));
                    const double v = fma(t, cst[g], -cst[P.npad + g]);  // exact product (power of two), one rounding
                    const double E = __fma_ru(cst[2 * P.npad + g], d1, cst[3 * P.npad + g]);
                    if (v > 0.0) word |= 1u << (sub * 16u + j);
                    if (!(fabs(v) > E) && g < nplanes && live) {
                        const unsigned int at = atomicAdd(P.queue_count, 1u);
                        if (at < P.queue_cap) P.queue[at] = make_uint2(slot, ((p0 + row) << 16) | g);
                    }
                }
            }
            const uint32_t w = pass * 2u + half;
            if (w < uint32_t(kPlaneWords)) pbits[row * kPlaneWords + w] = word;
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();  // this buffer may be overwritten by the pass after next; after the last pass: sA, pbits complete
        }

        // pack exactly as hash_codes_kernel does
        if (tid < kTcPoints && p0 + tid < img.n) {
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
        __syncthreads();  // pbits / dsum / sA are rewritten by the next unit
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace chgpu
