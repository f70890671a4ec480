// imma_probe.cu — issue rate of the warp-level integer tensor-core instructions the match path uses
// (mma.sync m16n8k16 / m16n8k32 u8 -> IMMA.16816 / IMMA.16832) on every SM, 4 independent accumulator chains per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/imma_probe scripts/imma_probe.cu && /tmp/imma_probe
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int K32>
__global__ void probe(int iters, int* out, long long* cycles) {
    int c[4][4] = {};
    uint32_t a0 = threadIdx.x * 2654435761u, a1 = a0 ^ 0x5bd1e995u, a2 = a0 + 77u, a3 = a1 + 99u, b0 = a0 >> 3, b1 = a1 >> 5;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            if (K32)
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
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount, iters = 4096;
    int* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(int) * sms * 1024);
    cudaMallocManaged(&cyc, sizeof(long long) * sms);
    for (int k32 = 0; k32 < 2; ++k32)
        for (int warps : {1, 4, 8, 16, 32}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (k32) probe<1><<<sms, warps * 32>>>(iters, out, cyc);
                else probe<0><<<sms, warps * 32>>>(iters, out, cyc);
                cudaDeviceSynchronize();
            }
            double mean = 0;
            for (int i = 0; i < sms; ++i) mean += double(cyc[i]) / sms;
            const double per_sm = double(iters) * 4 * warps / mean;  // IMMA per clock per SM
            printf("{\"probe\": \"%s\", \"warps_per_sm\": %d, \"imma_per_clk_per_sm\": %.4f, \"clk_per_imma_per_smsp\": %.2f, \"mac_per_clk_per_sm\": %.0f}\n",
                   k32 ? "IMMA.16832.U8" : "IMMA.16816.U8", warps, per_sm, 4.0 / per_sm * (warps < 4 ? warps / 4.0 : 1.0),
                   per_sm * 16 * 8 * (k32 ? 32 : 16));
        }
    return 0;
}
