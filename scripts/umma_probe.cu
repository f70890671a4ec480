// umma_probe.cu — checks, on the B200, the pieces the tensor-core Hamming pass (csrc/tc_kernels.cuh) is built from:
//   * tcgen05.mma.cta_group::1.kind::i8 (int8 x int8 -> int32 in TMEM), M = 128, N = 16..256, K = 160 as five K = 32 steps,
//     operands K-major in shared memory in (mode 0) the un-swizzled "interleaved" canonical layout
//     ((8,n),2):((1,SBO),LBO) in 16-byte units, or (mode 1) SWIZZLE_128B for the first 128 bytes of K plus an interleaved
//     32-byte tail — written by ordinary threads (st.shared + fence.proxy.async), not by TMA;
//   * tcgen05.ld 32x32b.x32 read-back of the accumulator, lane = row, column = n;
//   * the issue rate of such MMA groups and of the TMEM loads (clock64 around loops on every SM).
// Results are compared with a host evaluation of the same integer products.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma_probe scripts/umma_probe.cu && /tmp/umma_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kM = 128, kK = 160, kNMax = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes, uint32_t layout_type) {
    uint64_t d = 0;
    d |= uint64_t((saddr & 0x3FFFFu) >> 4);
    d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;  // descriptor version (sm_100)
    d |= uint64_t(layout_type) << 61;
    return d;
}
// kind::i8, signed x signed -> s32, both operands K-major
__host__ __device__ constexpr uint32_t make_idesc(uint32_t M, uint32_t N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, "
        "%19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]),
          "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

// byte offset of (row r, K byte kb) inside an operand tile
//   mode 0: everything interleaved: 8-row groups of 10 core matrices (8 rows x 16 B, 128 B each): LBO = 128, SBO = 1280
//   mode 1: K bytes 0..127 SWIZZLE_128B (row pitch 128 B, 8-row atoms of 1024 B), K bytes 128..159 interleaved behind them
__host__ __device__ inline uint32_t tile_offset(int mode, int rows, int r, int kb) {
    if (mode == 0) return (r >> 3) * 1280 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15);
    if (kb < 128) return (r >> 3) * 1024 + (r & 7) * 128 + ((((kb >> 4) ^ (r & 7)) & 7) << 4) + (kb & 15);
    const int k2 = kb - 128;
    return rows * 128 + (r >> 3) * 256 + (k2 >> 4) * 128 + (r & 7) * 16 + (k2 & 15);
}

struct Timing {
    long long mma_cycles, ld_cycles;
};

__global__ void __launch_bounds__(128, 1) probe_kernel(const int8_t* A, const int8_t* B, int N, int mode, int32_t* D, int reps,
                                                       Timing* tm) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    unsigned char* sA = smem;                        // 128 x 160
    unsigned char* sB = smem + 32768;                // up to 256 x 160 (1024-aligned)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int i = tid; i < kM * kK; i += 128) sA[tile_offset(mode, kM, i / kK, i % kK)] = A[i];
    for (int i = tid; i < kNMax * kK; i += 128) {
        const int r = i / kK;
        sB[tile_offset(mode, kNMax, r, i % kK)] = r < N ? B[i] : 0;
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // generic-proxy writes of the operands -> visible to the tensor core's async-proxy reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    const uint32_t idesc = make_idesc(kM, uint32_t(N));
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);

    auto issue_group = [&](uint32_t dcol) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            uint64_t da, db;
            if (mode == 0) {
                da = make_desc(a0 + k * 256, 128, 1280, 0);
                db = make_desc(b0 + k * 256, 128, 1280, 0);
            } else if (k < 4) {
                da = make_desc(a0 + k * 32, 16, 1024, 2);
                db = make_desc(b0 + k * 32, 16, 1024, 2);
            } else {
                da = make_desc(a0 + kM * 128, 128, 256, 0);
                db = make_desc(b0 + kNMax * 128, 128, 256, 0);
            }
            umma_i8(tmem + dcol, da, db, idesc, k > 0);
        }
    };

    uint32_t parity = 0;
    if (tid == 0) {
        issue_group(0);
        umma_commit(&bar);
    }
    mbar_wait(&bar, parity);
    parity ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (blockIdx.x == 0) {
        for (int c0 = 0; c0 < N; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c0, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c0 + j < N) D[(warp * 32 + lane) * N + c0 + j] = int32_t(v[j]);
        }
    }
    // ---- timing: `reps` groups back to back (alternating two accumulator halves), then `reps` TMEM loads per warp ----
    __syncthreads();
    if (reps > 0) {
        long long t0 = clock64();
        if (tid == 0) {
            for (int r = 0; r < reps; ++r) issue_group((r & 1) * 256);
            umma_commit(&bar);
        }
        mbar_wait(&bar, parity);
        parity ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        long long t1 = clock64();
        uint32_t acc = 0;
        for (int r = 0; r < reps; ++r) {
            uint32_t v[32];
            tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + (r & 7) * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v[j];
        }
        long long t2 = clock64();
        if (acc == 0x12345678u) D[0] = 1;
        if (tid == 0) {
            tm[blockIdx.x].mma_cycles = t1 - t0;
            tm[blockIdx.x].ld_cycles = t2 - t1;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

int main() {
    std::vector<int8_t> A(kM * kK), B(kNMax * kK);
    uint32_t s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
    for (auto& v : A) v = int8_t(int(rnd() % 255) - 127);
    for (auto& v : B) v = int8_t(int(rnd() % 255) - 127);
    int8_t *dA, *dB;
    int32_t* dD;
    Timing* dT;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dD, kM * kNMax * 4));
    CK(cudaMalloc(&dT, sizeof(Timing) * sms));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    const size_t smem = 32768 + kNMax * kK + 1024;
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    printf("{\"probe\": \"umma_i8\", \"sms\": %d, \"results\": [\n", sms);
    bool first = true;
    for (int mode = 0; mode < 2; ++mode) {
        for (int N : {256, 160, 96, 16}) {
            CK(cudaMemset(dD, 0xff, kM * kNMax * 4));
            const int reps = 2000;
            probe_kernel<<<sms, 128, smem>>>(dA, dB, N, mode, dD, reps, dT);
            CK(cudaDeviceSynchronize());
            std::vector<int32_t> D(kM * N);
            std::vector<Timing> T(sms);
            CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(T.data(), dT, sizeof(Timing) * sms, cudaMemcpyDeviceToHost));
            long bad = 0;
            int first_bad = -1;
            for (int m = 0; m < kM; ++m)
                for (int n = 0; n < N; ++n) {
                    int32_t ref = 0;
                    for (int k = 0; k < kK; ++k) ref += int32_t(A[m * kK + k]) * int32_t(B[n * kK + k]);
                    if (ref != D[m * N + n]) {
                        if (first_bad < 0) first_bad = m * N + n;
                        ++bad;
                    }
                }
            double mma = 0, ld = 0;
            for (auto& t : T) {
                mma += double(t.mma_cycles);
                ld += double(t.ld_cycles);
            }
            printf("%s {\"mode\": %d, \"N\": %d, \"mismatches\": %ld, \"first_bad\": %d, \"cycles_per_group_of_5_mma\": %.1f, "
                   "\"cycles_per_tmem_ld_x32_with_4_warps\": %.1f}",
                   first ? "" : ",\n", mode, N, bad, first_bad, mma / sms / reps, ld / sms / reps);
            first = false;
        }
    }
    printf("\n]}\n");
    return 0;
}
