// codec_kernels.cu -- the encoder (Eq. 3 in standard form) and the harness
// kernels around the decoder: info-bit generator, BPSK/AWGN channel with the
// LLR of Eq. 4, and the error counters.  All sm_100a, no tensor cores.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ldpc_internal.h"

namespace ldpc {
namespace {

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): the counter-based generator the
// workload recipe fixes.
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// ---------------------------------------------------------------------------
// Encoder, Eq. 3 with G in standard form.  One CTA per tile
// of FT frames:
//   1. stage the FT messages (kw words each) in shared memory;
//   2. parity bit b of frame f = parity(popc(XOR_w m_f[w] & P_b[w])): one warp
//      per parity column b, lanes stride the kw words (the P column is read
//      coalesced from L2 once per tile), XOR-accumulate per frame, then one
//      redux.sync.xor and a popcount per (frame, b) -- 1 LOP3 per 32 GF(2) MACs;
//   3. the permuted codeword [m | mP] is gathered to H column order with the
//      inverse permutation and packed by ballot.
constexpr int kEncFT = 8;

__global__ void __launch_bounds__(512) encode_kernel(const DeviceCode code, const uint32_t *__restrict__ info,
                                                     uint32_t *__restrict__ cw, int64_t frames) {
    extern __shared__ __align__(16) uint32_t esm[];
    const int kw = code.kw, nw = code.nw, k = code.k, n = code.n;
    const int npar = n - k;
    const int pw = (n + 31) / 32;              // words of the permuted codeword
    uint32_t *msg = esm;                       // [FT][kw]
    uint32_t *cperm = esm + kEncFT * kw;       // [FT][pw]
    const int64_t f0 = int64_t(blockIdx.x) * kEncFT;
    const int nf = int(std::min<int64_t>(kEncFT, frames - f0));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;

    for (int i = threadIdx.x; i < kEncFT * kw; i += blockDim.x) {
        const int f = i / kw, w = i - f * kw;
        uint32_t x = 0;
        if (f < nf) {
            x = __ldg(info + (f0 + f) * int64_t(kw) + w);
            if (w == kw - 1 && (k & 31)) x &= (1u << (k & 31)) - 1u;
        }
        msg[i] = x;
    }
    for (int i = threadIdx.x; i < kEncFT * pw; i += blockDim.x) cperm[i] = 0;
    __syncthreads();
    // systematic part: bits [0, k) of [m | mP] are m
    for (int i = threadIdx.x; i < kEncFT * kw; i += blockDim.x) {
        const int f = i / kw, w = i - f * kw;
        cperm[f * pw + w] = msg[i];
    }
    __syncthreads();
    for (int b = warp; b < npar; b += nwarps) {
        const uint32_t *col = code.pcols + int64_t(b) * kw;
        uint32_t acc[kEncFT];
#pragma unroll
        for (int f = 0; f < kEncFT; ++f) acc[f] = 0;
        for (int w = lane; w < kw; w += 32) {
            const uint32_t p = __ldg(col + w);
#pragma unroll
            for (int f = 0; f < kEncFT; ++f) acc[f] ^= msg[f * kw + w] & p;
        }
#pragma unroll
        for (int f = 0; f < kEncFT; ++f) {
            const uint32_t x = __reduce_xor_sync(0xffffffffu, acc[f]);
            if (lane == f && (__popc(x) & 1)) {
                const int pos = k + b;
                atomicOr(&cperm[f * pw + (pos >> 5)], 1u << (pos & 31));
            }
        }
    }
    __syncthreads();
    // scatter to H column order: c[v] = cperm[pinv[v]]
    for (int f = 0; f < nf; ++f) {
        uint32_t *out = cw + (f0 + f) * int64_t(nw);
        for (int v = threadIdx.x; v < nw * 32; v += blockDim.x) {
            bool bit = false;
            if (v < n) {
                const int t = __ldg(code.pinv + v);
                bit = (cperm[f * pw + (t >> 5)] >> (t & 31)) & 1u;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, bit);
            if (lane == 0) out[v >> 5] = word;
        }
    }
}

// ---------------------------------------------------------------------------
// Info bits: one thread per 4 words = one Philox block (counter (w/4, f, 0)).
__global__ void gen_info_kernel(uint64_t seed, int64_t frame0, int64_t frames, int k, uint32_t *out) {
    const int kw = (k + 31) / 32;
    const int blocks = (kw + 3) / 4;
    const int64_t total = frames * blocks;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = i / blocks;
        const int j = int(i - f * blocks);
        const uint64_t fr = uint64_t(frame0 + f);
        U4 r = philox(U4{uint32_t(j), uint32_t(fr), uint32_t(fr >> 32), 0u}, uint32_t(seed), uint32_t(seed >> 32));
        const uint32_t v[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int w = 4 * j + q;
            if (w < kw) {
                uint32_t x = v[q];
                if (w == kw - 1 && (k & 31)) x &= (1u << (k & 31)) - 1u;
                out[f * kw + w] = x;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Channel: BPSK + AWGN + LLR (Eq. 4).  One thread per 4
// variables = one Philox block (counter (v/4, f, 1)); Box-Muller in fp64.
__global__ void channel_kernel(uint64_t seed, int64_t frame0, int64_t frames, int n, const uint32_t *cw, double sigma,
                               float *llr) {
    const int nw = (n + 31) / 32;
    const int groups = (n + 3) / 4;
    const int64_t total = frames * groups;
    const double two_pi = 6.283185307179586476925286766559;
    const double inv32 = 1.0 / 4294967296.0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = i / groups;
        const int j = int(i - f * groups);
        const uint64_t fr = uint64_t(frame0 + f);
        U4 r = philox(U4{uint32_t(j), uint32_t(fr), uint32_t(fr >> 32), 1u}, uint32_t(seed), uint32_t(seed >> 32));
        double z[4];
        {
            const double rad = sqrt(-2.0 * log((double(r.x) + 1.0) * inv32));
            double sn, cs;
            sincos(two_pi * (double(r.y) * inv32), &sn, &cs);
            z[0] = rad * cs;
            z[1] = rad * sn;
        }
        {
            const double rad = sqrt(-2.0 * log((double(r.z) + 1.0) * inv32));
            double sn, cs;
            sincos(two_pi * (double(r.w) * inv32), &sn, &cs);
            z[2] = rad * cs;
            z[3] = rad * sn;
        }
        const uint32_t *c = cw + f * nw;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int v = 4 * j + q;
            if (v < n) {
                const double x = ((__ldg(c + (v >> 5)) >> (v & 31)) & 1u) ? 1.0 : -1.0;
                // y = x + sigma z, R = 2y / sigma^2, with no FMA contraction so the
                // fp64 roundings are those of the plain formula
                const double y = __dadd_rn(x, __dmul_rn(sigma, z[q]));
                double l = __ddiv_rn(__dmul_rn(2.0, y), __dmul_rn(sigma, sigma));
                l = fmin(fmax(l, -30.0), 30.0);
                llr[f * n + v] = float(l);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Error counters: one warp per frame; block partial sums, one atomic each.
__global__ void count_kernel(const DeviceCode code, const uint32_t *info, const uint32_t *bits, const uint32_t *cw,
                             const uint8_t *syn, const int32_t *iters, int64_t frames,
                             unsigned long long *counters) {
    __shared__ unsigned long long part[6];
    if (threadIdx.x < 6) part[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp_global = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
    const int k = code.k, kw = code.kw, nw = code.nw;
    for (int64_t f = warp_global; f < frames; f += nwarps) {
        const uint32_t *b = bits + f * nw;
        const uint32_t *m = info + f * kw;
        int ie = 0;
        for (int t0 = 0; t0 < kw * 32; t0 += 32) {
            const int t = t0 + lane;
            bool err = false;
            if (t < k) {
                const int v = __ldg(code.perm + t);
                const uint32_t zb = (__ldg(b + (v >> 5)) >> (v & 31)) & 1u;
                const uint32_t mb = (__ldg(m + (t >> 5)) >> (t & 31)) & 1u;
                err = zb != mb;
            }
            ie += __popc(__ballot_sync(0xffffffffu, err));
        }
        int ce = 0;
        for (int w = lane; w < nw; w += 32) {
            uint32_t x = __ldg(b + w) ^ __ldg(cw + f * nw + w);
            if (w == nw - 1 && (code.n & 31)) x &= (1u << (code.n & 31)) - 1u;
            ce += __popc(x);
        }
        ce = __reduce_add_sync(0xffffffffu, ce);
        if (lane == 0) {
            c0 += ie;
            c1 += ce;
            c2 += ie > 0;
            c3 += (syn[f] && ce > 0);
            c4 += iters[f];
            c5 += 1;
        }
    }
    if (lane == 0) {
        atomicAdd(&part[0], c0);
        atomicAdd(&part[1], c1);
        atomicAdd(&part[2], c2);
        atomicAdd(&part[3], c3);
        atomicAdd(&part[4], c4);
        atomicAdd(&part[5], c5);
    }
    __syncthreads();
    if (threadIdx.x < 6 && part[threadIdx.x]) atomicAdd(&counters[threadIdx.x], part[threadIdx.x]);
}

int sm_count() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return std::max(sms, 1);
}

}  // namespace
}  // namespace ldpc

extern "C" {

ldpc_status ldpc_encode(const ldpc_code *code, const uint32_t *d_info, uint32_t *d_cw, int64_t frames, void *stream) {
    if (!code || frames < 0) return LDPC_ERR_ARG;
    if (!code->has_G || !code->bound_G || !code->d_buf) return LDPC_ERR_STATE;
    if (frames == 0) return LDPC_OK;
    if (!d_info || !d_cw) return LDPC_ERR_ARG;
    const ldpc::DeviceCode &D = code->dev;
    const int pw = (D.n + 31) / 32;
    const size_t smem = sizeof(uint32_t) * size_t(ldpc::kEncFT) * size_t(D.kw + pw);
    if (smem > 200 * 1024) return LDPC_ERR_UNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(ldpc::encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
            cudaSuccess)
        return LDPC_ERR_CUDA;
    const int64_t grid = (frames + ldpc::kEncFT - 1) / ldpc::kEncFT;
    ldpc::encode_kernel<<<dim3(unsigned(grid)), 512, smem, static_cast<cudaStream_t>(stream)>>>(D, d_info, d_cw,
                                                                                               frames);
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

ldpc_status ldpc_gen_info(uint64_t seed, int64_t frame0, int64_t frames, int32_t k, uint32_t *d_info, void *stream) {
    if (k <= 0 || frames < 0 || frame0 < 0) return LDPC_ERR_ARG;
    if (frames == 0) return LDPC_OK;
    if (!d_info) return LDPC_ERR_ARG;
    const int64_t work = frames * ((int64_t(k) + 127) / 128);
    const int grid = int(std::min<int64_t>((work + 255) / 256, int64_t(ldpc::sm_count()) * 16));
    ldpc::gen_info_kernel<<<dim3(unsigned(std::max(grid, 1))), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        seed, frame0, frames, k, d_info);
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

ldpc_status ldpc_channel(const ldpc_code *code, uint64_t seed, int64_t frame0, int64_t frames, const uint32_t *d_cw,
                         double sigma, float *d_llr, void *stream) {
    if (!code || frames < 0 || frame0 < 0 || !(sigma > 0.0)) return LDPC_ERR_ARG;
    if (frames == 0) return LDPC_OK;
    if (!d_cw || !d_llr) return LDPC_ERR_ARG;
    const int64_t work = frames * ((int64_t(code->n) + 3) / 4);
    const int grid = int(std::min<int64_t>((work + 255) / 256, int64_t(ldpc::sm_count()) * 16));
    ldpc::channel_kernel<<<dim3(unsigned(std::max(grid, 1))), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        seed, frame0, frames, code->n, d_cw, sigma, d_llr);
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

ldpc_status ldpc_count_errors(const ldpc_code *code, const uint32_t *d_info, const uint32_t *d_bits,
                              const uint32_t *d_cw, const uint8_t *d_syndrome_ok, const int32_t *d_iters,
                              int64_t frames, int64_t *d_counters6, void *stream) {
    if (!code || frames < 0) return LDPC_ERR_ARG;
    if (!code->has_G || !code->bound_G || !code->d_buf) return LDPC_ERR_STATE;
    if (frames == 0) return LDPC_OK;
    if (!d_info || !d_bits || !d_cw || !d_syndrome_ok || !d_iters || !d_counters6) return LDPC_ERR_ARG;
    const int grid = int(std::min<int64_t>((frames + 7) / 8, int64_t(ldpc::sm_count()) * 8));
    ldpc::count_kernel<<<dim3(unsigned(std::max(grid, 1))), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        code->dev, d_info, d_bits, d_cw, d_syndrome_ok, d_iters, frames,
        reinterpret_cast<unsigned long long *>(d_counters6));
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // extern "C"
