// microbench_dsmem.cu -- DSMEM random 4-byte gathers and scatters with explicit
// mapa + ld/st.shared::cluster (no pointer arrays), vs local shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_dsmem microbench_dsmem.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;
constexpr int kWords = 32768;   // 128 KB per CTA

template <int CL, bool STORE>
__global__ void kern(float *out, int iters, int remote_shift, unsigned long long *cycles) {
    extern __shared__ float sm[];
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t my = cluster.block_rank();
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = float(i);
    cluster.sync();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 40503u + 12345u;
    float acc = 0.f;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            s = s * 1664525u + 1013904223u;
            const uint32_t off = (s >> 17) << 2;                         // 0 .. 128 KB
            // remote_shift: 32 -> all local; 0 -> rank uniform over the cluster
            const uint32_t r = (remote_shift >= 32) ? my : ((s >> remote_shift) % CL);
            uint32_t addr;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(base + off), "r"(r));
            if (STORE) {
                asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(acc) : "memory");
                acc += 1.0f;
            } else {
                float v;
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
                acc += v;
            }
        }
    }
    unsigned long long t1 = clock64();
    cluster.sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CL, bool STORE>
void run(int sms, float *d_out, unsigned long long *d_cyc, int remote_shift, const char *label) {
    const int threads = 1024, iters = 256;
    const int grid = (sms / CL) * CL;
    auto k = kern<CL, STORE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
    if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
    for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k, d_out, iters, remote_shift, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
    std::vector<unsigned long long> cyc(grid);
    cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto c : cyc) mean += double(c);
    mean /= grid;
    printf("%-6s cluster=%2d %-22s: %.2f ops/clk/SM\n", STORE ? "store" : "load", CL, label,
           double(threads) * iters * 8 / mean);
}

// Random 4-byte gathers from an L2-resident global buffer (words = 2^log2w).
__global__ void l2_gather(const float *__restrict__ buf, int log2w, int iters, float *out,
                          unsigned long long *cycles) {
    uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 40503u + 12345u;
    float acc = 0.f;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            s = s * 1664525u + 1013904223u;
            v[q] = __ldcg(buf + (s >> (32 - log2w)));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

void run_l2(int sms, float *d_out, unsigned long long *d_cyc, int log2w) {
    float *buf;
    cudaMalloc(&buf, sizeof(float) << log2w);
    cudaMemset(buf, 0, sizeof(float) << log2w);
    const int threads = 1024, iters = 128;
    for (int rep = 0; rep < 2; ++rep) l2_gather<<<sms, threads>>>(buf, log2w, iters, d_out, d_cyc);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> cyc(sms);
    cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (auto c : cyc) mean += double(c);
    mean /= sms;
    printf("global random gather, %6.1f MB buffer: %.2f loads/clk/SM\n", (4.0 * (1 << log2w)) / 1e6,
           double(threads) * iters * 8 / mean);
    cudaFree(buf);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *d_out;
    unsigned long long *d_cyc;
    cudaMalloc(&d_out, sizeof(float) * 148 * 1024);
    cudaMalloc(&d_cyc, sizeof(unsigned long long) * 4096);
    run<2, false>(sms, d_out, d_cyc, 32, "local only");
    run<2, false>(sms, d_out, d_cyc, 3, "uniform rank (1/2 rem)");
    run<4, false>(sms, d_out, d_cyc, 3, "uniform rank (3/4 rem)");
    run<8, false>(sms, d_out, d_cyc, 3, "uniform rank (7/8 rem)");
    run<2, true>(sms, d_out, d_cyc, 32, "local only");
    run<2, true>(sms, d_out, d_cyc, 3, "uniform rank (1/2 rem)");
    run<4, true>(sms, d_out, d_cyc, 3, "uniform rank (3/4 rem)");
    run<8, true>(sms, d_out, d_cyc, 3, "uniform rank (7/8 rem)");
    for (int lw : {18, 22, 24, 25}) run_l2(sms, d_out, d_cyc, lw);
    return 0;
}
