// onchip_probe.cu — measured on-chip peaks of the B200 for the resources the match kernel runs into:
//   POPC (XU pipe), plain integer ALU issue, VIADDMNMX-style min chains, LDS.128 shared-memory wavefronts.
// bench.py's roofline.on_chip uses these as denominators when profiles/onchip_peaks.json exists
// ("POPC issues at 16/clk/SM ... to be confirmed by micro-benchmark on sm_100").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/onchip_probe scripts/onchip_probe.cu && /tmp/onchip_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kThreads = 1024;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(kThreads) popc_kernel(uint32_t* out, uint32_t seed) {
    uint32_t x[8], acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
        acc[i] = 0;
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc[i] += __popc(x[i]);
            x[i] ^= acc[i];  // one LOP3 per POPC, as in the Hamming scan (xor, then popc)
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    out[blockIdx.x * kThreads + threadIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) alu_kernel(uint32_t* out, uint32_t seed) {
    uint32_t x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + 1) + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = (x[i] ^ seed) + (x[(i + 1) & 7] & 0xff);  // LOP3 + IADD3-class, independent chains
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * kThreads + threadIdx.x] = s;
}

__global__ void __launch_bounds__(kThreads) minchain_kernel(uint32_t* out, uint32_t seed) {
    uint32_t k[9], a = seed, b = seed ^ 0x5555u;
#pragma unroll
    for (int i = 0; i < 9; ++i) k[i] = seed * (threadIdx.x + 3) + i * 0x85ebca6bu;
    for (int it = 0; it < kIters; ++it) {
        const uint32_t nb = ~a;
        uint32_t acc = 0xffffffffu + nb, acc2 = k[0] + nb;
#pragma unroll
        for (int i = 1; i < 9; ++i) {
            if (i & 1) acc = min(acc, k[i] + nb);
            else acc2 = min(acc2, k[i] + nb);
        }
        a = min(acc, acc2) + b;
        b += 0x01000193u;
    }
    out[blockIdx.x * kThreads + threadIdx.x] = a;
}

__global__ void __launch_bounds__(kThreads) lds_kernel(uint32_t* out, uint32_t stride) {
    extern __shared__ uint4 s_codes[];  // 8,192 codes = 128 KiB, as the match kernel's train tile
    for (uint32_t i = threadIdx.x; i < 8192; i += kThreads) s_codes[i] = make_uint4(i, i * 3u, i * 5u, i * 7u);
    __syncthreads();
    uint32_t idx = (threadIdx.x * stride) & 8191u, acc = 0;
    for (int it = 0; it < kIters; ++it) {
        const uint4 v = s_codes[idx];
        acc += v.x ^ v.y ^ v.z ^ v.w;
        idx = (idx + 1024u * stride + (acc & 0u)) & 8191u;
    }
    out[blockIdx.x * kThreads + threadIdx.x] = acc;
}

template <class F>
static double time_ms(F&& launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

int main() {
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount, blocks = sms * 2;
    uint32_t* out;
    cudaMalloc(&out, size_t(blocks) * kThreads * 4);
    const double warps = double(blocks) * kThreads / 32;
    const double ms_popc = time_ms([&] { popc_kernel<<<blocks, kThreads>>>(out, 12345u); });
    const double ms_alu = time_ms([&] { alu_kernel<<<blocks, kThreads>>>(out, 12345u); });
    const double ms_min = time_ms([&] { minchain_kernel<<<blocks, kThreads>>>(out, 12345u); });
    cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    // stride 1: 32 consecutive codes per warp (4 wavefronts per LDS.128, conflict-free); stride 33: same, permuted
    const double ms_lds = time_ms([&] { lds_kernel<<<sms, kThreads, 131072>>>(out, 1u); });
    int clock_khz = 0;
    cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, 0);
    const double popc_s = warps * kIters * 8.0 * 32.0 / (ms_popc * 1e-3);             // thread-level POPC / s
    const double alu_winst_s = warps * kIters * 16.0 / (ms_alu * 1e-3);               // warp instructions / s (2 per chain step)
    const double min_iter_s = warps * kIters / (ms_min * 1e-3);                        // warp-level pull iterations / s (9 slots each)
    const double lds_wavefronts_s = double(sms) * kThreads / 32 * kIters * 4.0 / (ms_lds * 1e-3);
    std::printf("{\"device\": \"%s\", \"sm_count\": %d, \"clock_mhz_max\": %.0f, "
                "\"popc_per_s\": %.4e, \"popc_per_clk_per_sm_at_max_clock\": %.2f, "
                "\"alu_warp_inst_per_s\": %.4e, \"alu_warp_inst_per_clk_per_sm\": %.2f, "
                "\"pull_iterations_per_s\": %.4e, \"clk_per_pull_iteration_per_smsp\": %.2f, "
                "\"lds128_wavefronts_per_s\": %.4e, \"lds128_wavefronts_per_clk_per_sm\": %.2f, "
                "\"how\": \"scripts/onchip_probe.cu: 2 x 1024-thread CTAs per SM, %d iterations of 8 independent chains, best of 5, CUDA events\"}\n",
                prop.name, sms, clock_khz / 1e3, popc_s, popc_s / sms / (clock_khz * 1e3), alu_winst_s,
                alu_winst_s / sms / (clock_khz * 1e3), min_iter_s, 4.0 * sms * (clock_khz * 1e3) / min_iter_s, lds_wavefronts_s,
                lds_wavefronts_s / sms / (clock_khz * 1e3), kIters);
    return 0;
}
