// imma_mix_probe.cu — does a stream of IMMA (mma.sync u8) on one warp of an SMSP take issue slots away from
// integer ALU work of the other warps of that SMSP?  Warps 0..3 (one per SMSP) run IMMA chains (or idle), warps
// 4..4+A-1 run independent LOP3/IADD chains; the ALU warps' rate is reported with the IMMA warps on and off.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imma_mix scripts/imma_mix_probe.cu && /tmp/imma_mix
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void mix(int iters, int imma_on, int k32, int* out, long long* alu_cycles, long long* imma_cycles) {
    const int warp = threadIdx.x >> 5;
    if (warp < 4) {
        int c[4][4] = {};
        uint32_t a0 = threadIdx.x * 2654435761u, a1 = a0 ^ 0x5bd1e995u, a2 = a0 + 77u, a3 = a1 + 99u, b0 = a0 >> 3, b1 = a1 >> 5;
        const long long t0 = clock64();
        if (imma_on)
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    if (k32)
                        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                                     : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
                                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
                    else
                        asm volatile("mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                                     : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
                                     : "r"(a0), "r"(a1), "r"(b0));
                }
            }
        const long long t1 = clock64();
        int s = 0;
        for (int ch = 0; ch < 4; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
        if (threadIdx.x == 0) imma_cycles[blockIdx.x] = t1 - t0;
    } else {
        uint32_t x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 747796405u + i;
        const long long t0 = clock64();
        for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = (x[k] ^ 0x9e3779b9u) & (x[(k + 1) & 7] | 0x55u);  // one LOP3 per chain step
        }
        const long long t1 = clock64();
        uint32_t s = 0;
        for (int k = 0; k < 8; ++k) s += x[k];
        out[blockIdx.x * blockDim.x + threadIdx.x] = int(s);
        if (threadIdx.x == 128) alu_cycles[blockIdx.x] = t1 - t0;
    }
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount, iters = 2048;
    int* out;
    long long *ac, *ic;
    cudaMalloc(&out, sizeof(int) * sms * 1024);
    cudaMallocManaged(&ac, sizeof(long long) * sms);
    cudaMallocManaged(&ic, sizeof(long long) * sms);
    for (int alu_warps : {4, 8, 16})
        for (int mode = 0; mode < 3; ++mode) {  // 0: IMMA warps idle, 1: IMMA.16816, 2: IMMA.16832
            for (int rep = 0; rep < 2; ++rep) {
                mix<<<sms, (4 + alu_warps) * 32>>>(iters, mode != 0, mode == 2, out, ac, ic);
                cudaDeviceSynchronize();
            }
            double am = 0, im = 0;
            for (int i = 0; i < sms; ++i) am += double(ac[i]) / sms, im += double(ic[i]) / sms;
            printf("{\"alu_warps_per_sm\": %d, \"imma\": \"%s\", \"alu_warp_inst_per_clk_per_sm\": %.3f, \"clk_per_imma_per_smsp\": %.2f}\n",
                   alu_warps, mode == 0 ? "off" : (mode == 1 ? "16816" : "16832"), double(iters) * 4 * 8 * alu_warps / am,
                   mode ? im / (double(iters) * 4) : 0.0);
        }
    return 0;
}
