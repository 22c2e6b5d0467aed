// microbench_dsmem_stream.cu -- sustained DSMEM bandwidth of the exchange
// pattern of the C5 decoder (spa_cluster.cu xband2_kernel): every CTA of a
// C-CTA cluster streams segments of `seg` bytes to every other CTA of its
// cluster with cp.async.bulk shared::cta -> shared::cluster (complete_tx on
// the receiver's mbarrier), `rounds` rounds back to back with no handshake in
// between (the bandwidth ceiling, not one exchange's latency).  One CTA per
// SM (200 KB of shared memory), as many clusters as fit.  Prints bytes sent
// per clock per SM (each SM also receives as many).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_dsmem_stream tools/microbench_dsmem_stream.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t saddr(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

// issuers: lanes that issue copies (1: one lane round-robins over the peers,
// as the decoder's producer warp does per chunk; C - 1: one lane per peer)
__global__ void kern(int seg, int rounds, int issuers, unsigned long long *cycles) {
    extern __shared__ __align__(128) char smem[];
    const int tt = threadIdx.x;
    const uint32_t q = ctarank(), C = nctarank();
    char *send = smem;                                   // 64 KB source
    char *recv = smem + 65536;                           // 128 KB receive area
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536 + 131072);
    const uint32_t send_s = saddr(send), recv_s = saddr(recv), bar_s = saddr(bar);
    for (int i = tt; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(send)[i] = float(i);
    const uint32_t incoming = uint32_t(rounds) * (C - 1) * uint32_t(seg);
    if (tt == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(incoming) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    cluster_sync_all();
    const unsigned long long t0 = clock64();
    if (tt < issuers) {
        for (int r = 0; r < rounds; ++r) {
            for (uint32_t k = 1 + uint32_t(tt); k < C; k += uint32_t(issuers)) {
                const uint32_t d = (q + k) % C;
                const uint32_t slot = ((q * 7u + uint32_t(r)) % 64u) * 2048u % (131072u - uint32_t(seg));
                const uint32_t dst = mapa_u32(recv_s + (slot & ~15u), d);
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                    "r"(send_s + ((uint32_t(r) * 4096u) % (65536u - uint32_t(seg)) & ~15u)), "r"(uint32_t(seg)),
                    "r"(mapa_u32(bar_s, d))
                    : "memory");
            }
        }
    }
    mbar_wait(bar_s, 0);
    const unsigned long long t1 = clock64();
    cluster_sync_all();
    if (tt == 0) cycles[blockIdx.x] = t1 - t0;
}

void run(int C, int seg, int rounds, int issuers, int sms, unsigned long long *d_cyc) {
    const int smem = 65536 + 131072 + 64;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    const int grid = ncl * C;
    cfg.gridDim = dim3(grid);
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, kern, seg, rounds, issuers, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("C=%d error %s\n", C, cudaGetErrorString(e));
        return;
    }
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    const double mx = double(*std::max_element(cyc.begin(), cyc.end()));
    const double bytes = double(rounds) * (C - 1) * seg;
    printf("C=%2d clusters=%2d (%3d SMs) seg=%5d B rounds=%3d issuers=%2d : %8.0f clk  %6.2f B/clk/SM out (+ as much in)\n",
           C, ncl, grid, seg, rounds, issuers, mx, bytes / mx);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d_cyc;
    cudaMalloc(&d_cyc, sizeof(unsigned long long) * 4096);
    for (int C : {16, 8, 4, 2})
        for (int seg : {1024, 2048, 8192})
            for (int iss : {1, 32}) run(C, seg, std::max(4, (900 * 1024) / ((C - 1) * seg)), std::min(iss, C - 1), sms, d_cyc);
    return 0;
}
