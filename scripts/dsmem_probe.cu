// dsmem_probe.cu — how fast are random 16-byte gathers from a cluster peer's shared memory (ld.shared::cluster)?
// The match kernel gathers 128-bit codes by point id from a train image held in shared memory; images beyond one SM's
// capacity could be split over the CTAs of a cluster if remote gathers are fast enough.  Prints JSON lines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem_probe scripts/dsmem_probe.cu && /tmp/dsmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int kThreads = 896;
constexpr uint32_t kBytes = 128 * 1024;  // codes per CTA

template <int CLUSTER>
__global__ void __launch_bounds__(kThreads, 1) probe(uint32_t iters, uint32_t remote_of_16, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    for (uint32_t i = threadIdx.x; i < kBytes / 4; i += kThreads) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u + rank;
    cluster.sync();
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    uint32_t base[CLUSTER];
#pragma unroll
    for (int r = 0; r < CLUSTER; ++r)
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(base[r]) : "r"(local), "r"(r));
    uint32_t x = threadIdx.x * 747796405u + blockIdx.x, acc = 0;
    const long long t0 = clock64();
    for (uint32_t i = 0; i < iters; ++i) {
        x = x * 1664525u + 1013904223u;
        const uint32_t id = (x >> 8) & (kBytes / 16 - 1);
        // remote_of_16 of every 16 gathers go to a peer (chosen by the id), the rest stay local
        uint32_t r = rank;
        if (((x >> 4) & 15u) < remote_of_16) r = (rank + 1 + ((x >> 28) % (CLUSTER - 1 ? CLUSTER - 1 : 1))) % CLUSTER;
        uint32_t b = base[0];
#pragma unroll
        for (int k = 1; k < CLUSTER; ++k) b = r == uint32_t(k) ? base[k] : b;
        uint4 v;
        asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(b + id * 16u));
        acc += __popc(v.x ^ x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    const long long t1 = clock64();
    cluster.sync();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (acc == 0xffffffffu) *sink = acc;
}

template <int CLUSTER>
void run(uint32_t remote_of_16) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms / CLUSTER * CLUSTER;
    unsigned long long* d_out;
    uint32_t* d_sink;
    cudaMalloc(&d_out, grid * sizeof(unsigned long long));
    cudaMalloc(&d_sink, 4);
    cudaFuncSetAttribute(probe<CLUSTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBytes));
    if (CLUSTER > 8) cudaFuncSetAttribute(probe<CLUSTER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kBytes;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = CLUSTER;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    const uint32_t iters = 4000;
    for (int rep = 0; rep < 2; ++rep) {
        cudaError_t e = cudaLaunchKernelEx(&cfg, probe<CLUSTER>, iters, remote_of_16, d_out, d_sink);
        if (e != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
            printf("{\"cluster\": %d, \"error\": \"%s\"}\n", CLUSTER, cudaGetErrorString(e));
            return;
        }
    }
    unsigned long long h[256];
    cudaMemcpy(h, d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += double(h[i]);
    mean /= grid;
    const double gathers = double(iters) * kThreads;
    printf("{\"cluster\": %d, \"remote_of_16\": %u, \"ctas\": %d, \"clocks\": %.0f, \"gathers_per_clk_per_sm\": %.3f, \"bytes_per_clk_per_sm\": %.1f}\n",
           CLUSTER, remote_of_16, grid, mean, gathers / mean, 16.0 * gathers / mean);
    cudaFree(d_out);
    cudaFree(d_sink);
}

int main() {
    for (uint32_t r : {0u, 4u, 8u, 12u, 16u}) run<2>(r);
    for (uint32_t r : {8u, 12u, 16u}) run<4>(r);
    for (uint32_t r : {14u, 16u}) run<8>(r);
    return 0;
}
