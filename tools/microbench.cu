// microbench.cu -- B200 microbenchmarks that size the decoder design
// (DESIGN.md "Measured unit rates"):
//   1. MUFU ex2 / lg2 throughput per SM per clock (the SFU roofline);
//   2. random 4-byte gathers from local shared memory per SM per clock;
//   3. random 4-byte gathers through DSMEM (ld.shared::cluster) for cluster
//      sizes 2/4/8 and remote fractions 0..1.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

__global__ void mufu_kernel(float *out, int iters, int kind) {
    float a0 = threadIdx.x * 1e-3f + 0.5f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
    float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
    for (int i = 0; i < iters; ++i) {
        if (kind == 0) {
#define EX(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a))
            EX(a0); EX(a1); EX(a2); EX(a3); EX(a4); EX(a5); EX(a6); EX(a7);
        } else {
#define LG(a) asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(a))
            LG(a0); LG(a1); LG(a2); LG(a3); LG(a4); LG(a5); LG(a6); LG(a7);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

constexpr int kWords = 40960;   // 160 KB per CTA

template <int CL>
__global__ void dsmem_kernel(float *out, int iters, uint32_t remote_permille, unsigned long long *cycles) {
    extern __shared__ float sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned my = cluster.block_rank();
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = float(i);
    cluster.sync();
    float *base[CL];
#pragma unroll
    for (int r = 0; r < CL; ++r) base[r] = cluster.map_shared_rank(sm, r);
    float acc = 0.f;
    uint32_t s = hash32(threadIdx.x * 7919u + blockIdx.x * 104729u);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            s = hash32(s + q);
            const uint32_t off = s % kWords;
            const bool remote = (s >> 22) % 1000 < remote_permille;
            const unsigned r = remote ? (my + 1 + (s >> 8) % (CL > 1 ? CL - 1 : 1)) % CL : my;
            v[q] = base[r][off];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
    }
    unsigned long long t1 = clock64();
    cluster.sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CL>
int run_dsmem(int sms, float *d_out, unsigned long long *d_cyc, int permille) {
    const int threads = 1024, iters = 200;
    const int grid = (sms / CL) * CL;
    auto k = dsmem_kernel<CL>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4));
    if (CL > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = kWords * 4;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) CK(cudaLaunchKernelEx(&cfg, k, d_out, iters, (uint32_t)permille, d_cyc));
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> cyc(grid);
    CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost));
    double mean = 0;
    for (auto c : cyc) mean += double(c);
    mean /= grid;
    const double loads = double(threads) * iters * 8;
    printf("dsmem cluster=%d remote=%.2f : %.2f loads/clk/SM (%.0f cycles)\n", CL, permille / 1000.0,
           loads / mean, mean);
    return 0;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    printf("SMs=%d clock=%d kHz L2=%d bytes\n", sms, clk, l2);
    float *d_out;
    unsigned long long *d_cyc;
    CK(cudaMalloc(&d_out, sizeof(float) * 148 * 32 * 1024));
    CK(cudaMalloc(&d_cyc, sizeof(unsigned long long) * 4096));
    // MUFU
    for (int kind = 0; kind < 2; ++kind) {
        const int iters = 4096, threads = 1024, grid = sms * 2;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        mufu_kernel<<<grid, threads>>>(d_out, 16, kind);
        cudaEventRecord(a);
        mufu_kernel<<<grid, threads>>>(d_out, iters, kind);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = double(grid) * threads * iters * 8;
        printf("MUFU %s: %.3e ops/s = %.2f ops/clk/SM at %d MHz nominal\n", kind ? "lg2" : "ex2", ops / (ms * 1e-3),
               ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    run_dsmem<1>(sms, d_out, d_cyc, 0);
    for (int p : {0, 250, 500, 1000}) run_dsmem<2>(sms, d_out, d_cyc, p);
    for (int p : {0, 500, 1000}) run_dsmem<4>(sms, d_out, d_cyc, p);
    for (int p : {0, 500, 875, 1000}) run_dsmem<8>(sms, d_out, d_cyc, p);
    for (int p : {500, 1000}) run_dsmem<16>(sms, d_out, d_cyc, p);
    return 0;
}
