// microbench_ffma2.cu -- packed fp32x2 arithmetic on sm_100a (FFMA2 / FADD2 /
// FMUL2, PTX fma/add/mul.rn.f32x2) against scalar FFMA: issue slots and
// throughput per SM per clock, 8 independent chains per thread, 16 warps per
// SM.  Sizes the psi evaluation: the decoders are issue-bound,
// and a packed op does two lanes' worth of fp32 work in one issue slot.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_ffma2 tools/microbench_ffma2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float fma1(float a, float b, float c) {
    float d;
    asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ u64 pk(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__global__ void k(float *out, int iters, int kind, unsigned long long *cyc) {
    const float x = threadIdx.x * 1e-7f + 0.999f;
    __syncthreads();
    const unsigned long long t0 = clock64();
    float r = 0.f;
    if (kind == 0) {
        float a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = x + i;
        const float m = 0.9999f, c = 1e-3f;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma1(a[i], m, c);
#pragma unroll
        for (int i = 0; i < 8; ++i) r += a[i];
    } else if (kind == 1) {
        // the same 16 fp32 FMAs per iteration as 8 packed ops
        u64 a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = pk(x + i, x - i);
        const u64 m = pk(0.9999f, 0.9998f), c = pk(1e-3f, 2e-3f);
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma2(a[i], m, c);
#pragma unroll
        for (int i = 0; i < 8; ++i) r += __uint_as_float(unsigned(a[i])) + __uint_as_float(unsigned(a[i] >> 32));
    } else {
        // scalar FFMA with 3 register operands (all varying)
        float a[8], m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = x + i;
            m[i] = 0.9999f - i * 1e-6f;
        }
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = fma1(a[i], m[i], m[(i + 1) & 7]);
#pragma unroll
        for (int i = 0; i < 8; ++i) r += a[i];
    }
    const unsigned long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x % 32 == 0) atomicMax(cyc + blockIdx.x, t1 - t0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 512, blocks = sms;
    float *out;
    unsigned long long *cyc;
    cudaMalloc(&out, size_t(blocks) * threads * 4);
    cudaMalloc(&cyc, size_t(blocks) * 8);
    const char *names[] = {"FFMA (imm/const operands)", "FFMA2 (fma.rn.f32x2)", "FFMA (3 register operands)"};
    const int iters = 1 << 15;
    for (int kind = 0; kind < 3; ++kind) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(cyc, 0, size_t(blocks) * 8);
            k<<<blocks, threads>>>(out, iters, kind, cyc);
            cudaDeviceSynchronize();
        }
        std::vector<unsigned long long> h(blocks);
        cudaMemcpy(h.data(), cyc, blocks * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (auto c : h) mx = c > mx ? c : mx;
        const double instr = double(iters) * 8.0 * threads / 32.0;     // warp instructions per SM
        const double flops = double(iters) * 8.0 * threads * (kind == 1 ? 2 : 1);
        printf("%-28s %6.3f warp-instr/clk/SM  %7.2f fp32 FMA/clk/SM  (%llu cycles)\n", names[kind],
               instr / double(mx), flops / double(mx), mx);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
