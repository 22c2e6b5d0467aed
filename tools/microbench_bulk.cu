// microbench_bulk.cu -- cost of one all-to-all message-segment exchange inside
// a thread-block cluster, the communication step of the exchange cluster
// decoder (spa_cluster.cu).  Every CTA sends `bytes` in C equal segments, one
// to each CTA of its cluster (itself included), then waits until its own
// segments from every CTA have landed.  Modes:
//   bulk  : C threads issue cp.async.bulk shared::cta -> shared::cluster with
//           complete_tx on the receiver's mbarrier; free-barrier handshake
//           (the decoder's protocol, no compute in between);
//   st.v4 : all threads store 16-byte vectors to the remote CTAs
//           (st.shared::cluster.v4), then a cluster barrier;
//   l2.v4 : all threads store the send buffer to a global slot (L2-resident,
//           16-byte vectors), cluster barrier, then load their segments from
//           every CTA's slot (ld.global.cg.v4) into shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_bulk microbench_bulk.cu
#include <cuda_runtime.h>

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

template <int C, int MODE>
__global__ void kern(int bytes, int reps, unsigned long long *cycles, float4 *gbuf) {
    extern __shared__ __align__(128) char smem[];
    const int tt = threadIdx.x, T = blockDim.x;
    const uint32_t q = ctarank();
    char *send = smem, *recv = smem + bytes * 2;     // recv[2] at bytes*2 .. bytes*4 (double buffered)
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 4 * bytes);
    const uint32_t send_s = saddr(send), recv_s = saddr(recv), bar_s = saddr(bars), free_s = bar_s + 16;
    const int seg = bytes / C;
    for (int i = tt; i < bytes / 4; i += T) reinterpret_cast<float *>(send)[i] = float(i);
    if (tt == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(free_s), "r"(C) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(bytes) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s + 8), "r"(bytes) : "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    cluster_sync_all();
    unsigned long long t0 = clock64();
    for (int h = 0; h < reps; ++h) {
        const uint32_t x = h & 1;
        if (MODE == 0) {
            if (h > 0) mbar_wait(free_s, (h - 1) & 1);
            __syncthreads();
            if (tt < C) {
                const uint32_t dst = mapa_u32(recv_s + x * bytes + q * seg, tt);
                const uint32_t bar = mapa_u32(bar_s + 8 * x, tt);
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(dst), "r"(send_s + tt * seg), "r"(seg), "r"(bar) : "memory");
            }
            mbar_wait(bar_s + 8 * x, (h >> 1) & 1);
            if (tt == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s + 8 * x), "r"(bytes)
                             : "memory");
            if (tt < C)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_u32(free_s, tt))
                             : "memory");
        } else if (MODE == 2) {
            float4 *mine = gbuf + size_t(blockIdx.x) * (bytes / 16);
            for (int i = tt; i < bytes / 16; i += T) mine[i] = reinterpret_cast<const float4 *>(send)[i];
            cluster_sync_all();
            const int vec_per_seg = seg / 16;
            const size_t cl0 = size_t(blockIdx.x - q);
            for (int i = tt; i < bytes / 16; i += T) {
                const int s = i / vec_per_seg, o = i - s * vec_per_seg;
                const float4 v = __ldcg(gbuf + (cl0 + s) * (bytes / 16) + q * vec_per_seg + o);
                reinterpret_cast<float4 *>(recv + x * bytes)[i] = v;
            }
            __syncthreads();
        } else {
            // every thread stores 16-byte vectors: destination d = i / (seg/16)
            const int vec_per_seg = seg / 16;
            for (int i = tt; i < bytes / 16; i += T) {
                const int d = i / vec_per_seg, o = i - d * vec_per_seg;
                const float4 v = reinterpret_cast<const float4 *>(send)[i];
                const uint32_t dst = mapa_u32(recv_s + x * bytes + q * seg + o * 16, d);
                asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "f"(v.x), "f"(v.y),
                             "f"(v.z), "f"(v.w)
                             : "memory");
            }
            cluster_sync_all();
        }
    }
    unsigned long long t1 = clock64();
    cluster_sync_all();
    if (tt == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int C, int MODE>
void run(int sms, unsigned long long *d_cyc, int bytes, int threads) {
    const int reps = 200;
    int grid = (sms / C) * C;
    auto k = kern<C, MODE>;
    const int smem = 4 * bytes + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    grid = std::min(grid, ncl * C);
    cfg.gridDim = dim3(grid);
    float4 *gbuf = nullptr;
    cudaMalloc(&gbuf, size_t(grid) * bytes);
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, bytes, reps, d_cyc, gbuf);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return;
    }
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    cudaFree(gbuf);
    double mean = 0;
    for (auto c : cyc) mean += double(c);
    mean /= grid;
    const double per = mean / reps;
    printf("%-5s C=%2d clusters=%3d threads=%4d bytes/CTA=%6d : %8.0f clk/exchange  %6.1f B/clk/SM out\n",
           MODE == 0 ? "bulk" : (MODE == 1 ? "st.v4" : "l2.v4"), C, grid / C, threads, bytes, per, bytes / per);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d_cyc;
    cudaMalloc(&d_cyc, sizeof(unsigned long long) * 4096);
    for (int bytes : {2048, 16384, 49152}) {
        run<8, 0>(sms, d_cyc, bytes, 1024);
        run<8, 1>(sms, d_cyc, bytes, 1024);
        run<8, 2>(sms, d_cyc, bytes, 1024);
        run<4, 2>(sms, d_cyc, bytes, 1024);
        run<2, 2>(sms, d_cyc, bytes, 1024);
        run<1, 2>(sms, d_cyc, bytes, 1024);
        run<4, 0>(sms, d_cyc, bytes, 1024);
        run<4, 1>(sms, d_cyc, bytes, 1024);
        run<16, 0>(sms, d_cyc, bytes / 2, 1024);
        run<2, 0>(sms, d_cyc, bytes, 1024);
    }
    return 0;
}
