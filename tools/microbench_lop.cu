// microbench_lop.cu -- the encoder's roofline (DESIGN.md §6 "encode"): the
// GF(2) product M.P runs as `acc ^= m & p` (one LOP3 per 32 bit-MACs) plus one
// POPC per output bit, both on the INT/ALU side.  Measures, per SM per clock:
//   1. LOP3 (3-input logic, acc = acc ^ (m & p)), 8 independent chains/thread;
//   2. POPC;
//   3. the encoder's inner mix: 32 LOP3 : 1 POPC (k = 32 words per output bit).
// Timed with clock64 inside each CTA (cycles of the slowest warp), 16 warps
// per SM, every SM busy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_lop tools/microbench_lop.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t lop_xa(uint32_t acc, uint32_t m, uint32_t p) {
    uint32_t d;
    // 0x6A = a ^ (b & c)
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(acc), "r"(m), "r"(p));
    return d;
}
__device__ __forceinline__ uint32_t popc(uint32_t x) {
    uint32_t d;
    asm volatile("popc.b32 %0, %1;" : "=r"(d) : "r"(x));
    return d;
}

__global__ void lop_kernel(uint32_t *out, int iters, int kind, unsigned long long *cyc) {
    uint32_t a[8], m = threadIdx.x * 2654435761u, p = blockIdx.x * 40503u + 17u;
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = m ^ (i * 0x9e3779b9u);
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (kind == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = lop_xa(a[i], m, p + i);
            p = p * 3u + 1u;        // 1 IMAD (fma pipe) per 8 LOP3
        }
    } else if (kind == 1) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = popc(a[i] ^ p) + a[i];
            p = p * 3u + 1u;
        }
    } else {
        // 32 LOP3 then 1 POPC per chain: one output bit of a k = 1024 code
        uint32_t s = 0;
        for (int it = 0; it < iters; it += 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = lop_xa(a[i], m + r, p + i);
            p = p * 3u + 1u;
            if ((it & 31) == 28) {
#pragma unroll
                for (int i = 0; i < 8; ++i) s += popc(a[i]);
            }
        }
        a[0] ^= s;
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x % 32 == 0) atomicMax(cyc + blockIdx.x, t1 - t0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, per_sm = 1, blocks = sms * per_sm;    // 16 warps per SM
    uint32_t *out;
    unsigned long long *cyc;
    cudaMalloc(&out, size_t(blocks) * threads * 4);
    cudaMalloc(&cyc, size_t(blocks) * 8);
    const char *names[] = {"LOP3 (acc ^= m & p)", "POPC", "encoder mix 32 LOP3 : 1 POPC"};
    const int iters = 1 << 16;
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(cyc, 0, size_t(blocks) * 8);
            lop_kernel<<<blocks, threads>>>(out, iters, kind, cyc);
            cudaDeviceSynchronize();
        }
        std::vector<unsigned long long> h(blocks);
        cudaMemcpy(h.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (auto c : h) mx = c > mx ? c : mx;
        // ops per thread: kind 0: 8 LOP3 per iter; kind 1: 8 POPC per iter;
        // kind 2: 8 LOP3 per iter + 8 POPC per 32 iters
        const double thr_per_sm = double(threads) * per_sm;
        const double ops = double(iters) * 8.0 * thr_per_sm;
        printf("%-30s %7.2f ops/clk/SM (%llu cycles, %d warps/SM)\n", names[kind], ops / double(mx), mx,
               threads * per_sm / 32);
        if (kind == 2)
            printf("%-30s %7.2f POPC/clk/SM alongside\n", "", ops / 32.0 / double(mx));
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
