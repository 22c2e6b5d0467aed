// codec_kernels.cu -- the encoder (Eq. 3 in standard form) and the harness
// kernels around the decoder: info-bit generator, BPSK/AWGN channel with the
// LLR of Eq. 4, and the error counters.  All sm_100a; the tensor-core form
// of the parity product is encode_mma.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "channel_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {

// ---------------------------------------------------------------------------
// Encoder, Eq. 3 with G in standard form: the parity bits
// are the GF(2) product M P (frames x k times k x (n-k)), bit-packed along k.
// Kernel 1 (parity) is a register-tiled binary "GEMM" on the INT pipe: a CTA
// owns 64 frames x 128 parity columns; k is streamed in chunks of 32 words
// through shared memory (messages as [frame][word], P pre-transposed at bind
// time as [word][column] so both loads are coalesced); every thread keeps
// 4 frames x 8 columns of XOR accumulators, acc ^= m & p -- one LOP3 per 32
// GF(2) multiply-adds -- and the parity of each accumulator is one popc.
// Parity words are parked in the tail of the frame's output row.  Kernel 2
// (assemble) scatters [m | m P] to H column order with the inverse
// permutation, one CTA per frame row, packing 32 bits per ballot.
constexpr int kEncTF = 64;    // frames per CTA tile
constexpr int kEncKC = 32;    // message words per k chunk

__global__ void __launch_bounds__(256) encode_parity_kernel(const DeviceCode code, const uint32_t *__restrict__ info,
                                                            uint32_t *__restrict__ cw, int64_t frames) {
    // message rows padded to 36 words: 16-byte aligned for the 4-word vector
    // loads, and the two frames a warp reads (4 rows apart) on disjoint banks
    constexpr int MS = kEncKC + 4;
    __shared__ __align__(16) uint32_t ms[kEncTF][MS];
    __shared__ __align__(16) uint32_t ps[kEncKC][kEncColTile];
    __shared__ uint8_t pnib[kEncTF][kEncColTile / 4];
    const int kw = code.kw, npp = code.npar_pad, nw = code.nw;
    const int npw = (code.n - code.k + 31) / 32;
    const int b0 = blockIdx.x * kEncColTile;
    const int64_t f0 = int64_t(blockIdx.y) * kEncTF;
    // thread (tf, tb): frames tf*4 .. tf*4+3, parity columns tb*4 .. tb*4+3 and
    // 64 + tb*4 .. 64 + tb*4+3 -- the 16 lanes of a half-warp read 256
    // contiguous bytes of a P row per vector load (2 wavefronts)
    const int tid = threadIdx.x, tf = tid >> 4, tb = tid & 15;
    uint32_t acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0u;

    for (int w0 = 0; w0 < kw; w0 += kEncKC) {
        for (int i = tid; i < kEncTF * kEncKC; i += 256) {
            const int f = i >> 5, w = i & 31;
            uint32_t x = 0u;
            if (f0 + f < frames && w0 + w < kw) x = __ldg(info + (f0 + f) * int64_t(kw) + w0 + w);
            ms[f][w] = x;      // bits beyond k meet zero rows of P: no mask needed
        }
        for (int i = tid; i < kEncKC * (kEncColTile / 4); i += 256) {
            const int w = i >> 5, c4 = i & 31;
            uint4 x = make_uint4(0u, 0u, 0u, 0u);
            if (w0 + w < kw) x = __ldg(reinterpret_cast<const uint4 *>(code.pt + size_t(w0 + w) * npp + b0) + c4);
            *reinterpret_cast<uint4 *>(&ps[w][4 * c4]) = x;
        }
        __syncthreads();
        // the last chunk's words beyond kw are zero: skip them (Table I: kw
        // = 9..25 in one 32-word chunk)
        const int wend = min(kEncKC, (kw - w0 + 3) & ~3);
#pragma unroll 2
        for (int w = 0; w < wend; w += 4) {
            uint4 m4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) m4[i] = *reinterpret_cast<const uint4 *>(&ms[tf * 4 + i][w]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint4 pa = *reinterpret_cast<const uint4 *>(&ps[w + u][tb * 4]);
                const uint4 pb = *reinterpret_cast<const uint4 *>(&ps[w + u][64 + tb * 4]);
                const uint32_t p[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t m = u == 0 ? m4[i].x : u == 1 ? m4[i].y : u == 2 ? m4[i].z : m4[i].w;
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] ^= m & p[j];
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t lo = 0u, hi = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            lo |= (uint32_t(__popc(acc[i][j])) & 1u) << j;
            hi |= (uint32_t(__popc(acc[i][4 + j])) & 1u) << j;
        }
        pnib[tf * 4 + i][tb] = uint8_t(lo);          // columns tb*4 .. tb*4+3
        pnib[tf * 4 + i][16 + tb] = uint8_t(hi);     // columns 64 + tb*4 ..
    }
    __syncthreads();
    // parity word q of this tile -> word (b0/32 + q) of the parity area, which
    // is parked in the last npw words of the frame's output row
    for (int i = tid; i < kEncTF * (kEncColTile / 32); i += 256) {
        const int f = i >> 2, q = i & 3;
        const int pwi = b0 / 32 + q;
        if (f0 + f < frames && pwi < npw) {
            const uint8_t *nb = &pnib[f][8 * q];
            uint32_t word = 0u;
#pragma unroll
            for (int t = 0; t < 8; ++t) word |= uint32_t(nb[t]) << (4 * t);
            cw[(f0 + f) * int64_t(nw) + (nw - npw) + pwi] = word;
        }
    }
}

__global__ void __launch_bounds__(256) encode_assemble_kernel(const DeviceCode code, const uint32_t *__restrict__ info,
                                                              uint32_t *__restrict__ cw, int64_t frames) {
    extern __shared__ uint32_t asm_buf[];
    const int kw = code.kw, nw = code.nw, k = code.k, n = code.n;
    const int npw = (n - k + 31) / 32;
    uint32_t *mrow = asm_buf, *prow = asm_buf + kw;
    for (int64_t f = blockIdx.x; f < frames; f += gridDim.x) {
        uint32_t *row = cw + f * int64_t(nw);
        for (int i = threadIdx.x; i < kw; i += blockDim.x) mrow[i] = __ldg(info + f * int64_t(kw) + i);
        for (int i = threadIdx.x; i < npw; i += blockDim.x) prow[i] = row[nw - npw + i];
        __syncthreads();
        for (int v = threadIdx.x; v < nw * 32; v += blockDim.x) {
            uint32_t bit = 0u;
            if (v < n) {
                const int t = __ldg(code.pinv + v);
                bit = t < k ? (mrow[t >> 5] >> (t & 31)) & 1u : (prow[(t - k) >> 5] >> ((t - k) & 31)) & 1u;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, bit != 0u);
            if ((threadIdx.x & 31) == 0) row[v >> 5] = word;
        }
        __syncthreads();
    }
}

// Assemble by deposits, warp per frame: codeword word j is the next message
// bits deposited into its info mask OR the next parity bits deposited into
// its parity mask (both halves of perm ascend; host_code.cpp
// assemble_table).  Lane l builds words l, l + 32, ...: two 32-bit windows
// of the staged message / parity rows (funnel shifts), two five-step
// expands, one coalesced store -- instead of one ballot per 32 bits with a
// pinv gather per bit (encode_assemble_kernel).  Same output bits.
constexpr int kAsmWarps = 8;
__device__ __forceinline__ uint32_t expand32(uint32_t x, const uint32_t *mv, uint32_t m) {
#pragma unroll
    for (int i = 4; i >= 0; --i) {
        const uint32_t t = x << (1 << i);
        x = (x & ~mv[i]) | (t & mv[i]);
    }
    return x & m;
}
__global__ void __launch_bounds__(kAsmWarps * 32) encode_assemble_dep_kernel(const DeviceCode code,
                                                                             const uint32_t *__restrict__ info,
                                                                             uint32_t *__restrict__ cw,
                                                                             int64_t frames) {
    extern __shared__ __align__(16) uint32_t asm_smem[];
    const int kw = code.kw, nw = code.nw, k = code.k, n = code.n;
    const int npw = (n - k + 31) / 32;
    const int rw = kw + npw + 2;                 // one zero word behind each row (funnel shifts)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *mrow = asm_smem + size_t(warp) * rw, *prow = mrow + kw + 1;
    const int64_t gw = int64_t(blockIdx.x) * kAsmWarps + warp, nwarps = int64_t(gridDim.x) * kAsmWarps;
    const uint4 *tab = reinterpret_cast<const uint4 *>(code.asmtab);
    for (int64_t f = gw; f < frames; f += nwarps) {
        uint32_t *row = cw + f * int64_t(nw);
        for (int i = lane; i < kw; i += 32) mrow[i] = __ldg(info + f * int64_t(kw) + i);
        for (int i = lane; i < npw; i += 32) prow[i] = row[nw - npw + i];
        if (lane == 0) {
            mrow[kw] = 0u;
            prow[npw] = 0u;
        }
        __syncwarp();
        for (int j = lane; j < nw; j += 32) {
            const uint4 h = __ldg(tab + 4 * j), u = __ldg(tab + 4 * j + 1), v = __ldg(tab + 4 * j + 2),
                        w = __ldg(tab + 4 * j + 3);
            const uint32_t mi = h.x, mp = h.y, a = h.z, b = 32u * uint32_t(j) - a;
            const uint32_t mvi[5] = {u.x, u.y, u.z, u.w, v.x}, mvp[5] = {v.y, v.z, v.w, w.x, w.y};
            uint32_t x = 0u, y = 0u;
            if (mi) x = __funnelshift_r(mrow[a >> 5], mrow[(a >> 5) + 1], a & 31u);
            if (mp) y = __funnelshift_r(prow[b >> 5], prow[(b >> 5) + 1], b & 31u);
            row[j] = expand32(x, mvi, mi) | expand32(y, mvp, mp);
        }
        __syncwarp();
    }
}

// Small codes (k <= 128 bits) in small batches: the tiled kernel's 64-frame
// x 128-column tiles and 32-word k chunks are mostly padding there (C1: k =
// 48, two words), so one kernel does both steps, one warp per frame: lane i
// holds message word i, and each output bit v (H column order) is either a
// message bit or parity column c = pinv[v] - k, the GF(2) dot product of the
// message with column c of P (popc of kw ANDed words); bits are packed by
// ballot.  Same result as parity + assemble (tests/test_gpu_parity.py).
__global__ void __launch_bounds__(256) encode_small_kernel(const DeviceCode code, const uint32_t *__restrict__ info,
                                                           uint32_t *__restrict__ cw, int64_t frames) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int kw = code.kw, nw = code.nw, k = code.k, n = code.n, npp = code.npar_pad;
    for (int64_t f = wg; f < frames; f += nwarps) {
        const uint32_t mine = lane < kw ? __ldg(info + f * int64_t(kw) + lane) : 0u;
        uint32_t *row = cw + f * int64_t(nw);
        for (int v0 = 0; v0 < nw * 32; v0 += 32) {
            const int v = v0 + lane;
            const int t = v < n ? __ldg(code.pinv + v) : -1;
            // parity column t - k: every lane takes part in the shuffles
            uint32_t acc = 0u;
            for (int w = 0; w < kw; ++w) {
                const uint32_t mw = __shfl_sync(0xffffffffu, mine, w);
                if (t >= k) acc ^= mw & __ldg(code.pt + size_t(w) * npp + (t - k));
            }
            uint32_t bit = uint32_t(__popc(acc)) & 1u;
            // message bits: word t >> 5 from its lane (every lane takes part)
            const uint32_t mw = __shfl_sync(0xffffffffu, mine, t >= 0 && t < k ? (t >> 5) : 0);
            if (t >= 0 && t < k) bit = (mw >> (t & 31)) & 1u;
            const uint32_t word = __ballot_sync(0xffffffffu, bit != 0u);
            if (lane == 0) row[v0 >> 5] = word;
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
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t f = i / groups;
        const int j = int(i - f * groups);
        const uint64_t fr = uint64_t(frame0 + f);
        double z[4];
        channel_normals(seed, fr, j, z);
        const uint32_t *c = cw + f * nw;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int v = 4 * j + q;
            if (v < n) {
                const bool one = (__ldg(c + (v >> 5)) >> (v & 31)) & 1u;
                const float l = channel_llr(one, sigma, z[q]);
                llr[f * n + v] = l;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Error counters: a group of TPF threads per frame (a warp at
// large batches; up to the whole 256-thread CTA when there are few frames, so
// a small batch still spreads its bits over every SM); block partial sums,
// one atomic each.  Each thread counts its own info-bit and codeword-bit
// errors without a per-chunk ballot, so the loads of successive chunks are
// independent (a cold small batch was a chain of 2 x kw/32 dependent HBM
// loads per warp: 10 us for 1000 Table I frames); the group's sums meet in
// shared memory before the per-frame flags (frame error, undetected) are set.
__global__ void __launch_bounds__(256) count_kernel(const DeviceCode code, const uint32_t *info, const uint32_t *bits,
                                                    const uint32_t *cw, const uint8_t *syn, const int32_t *iters,
                                                    int64_t frames, int tpf, const uint32_t *asmtab,
                                                    unsigned long long *counters) {
    __shared__ unsigned long long part[6];
    __shared__ int fr_ie[8], fr_ce[8];
    constexpr int kStageW = 64;
    __shared__ uint32_t s_b[8][kStageW];
    if (threadIdx.x < 6) part[threadIdx.x] = 0;
    const int fpb = blockDim.x / tpf;                  // frames per block pass
    const int slot = threadIdx.x / tpf, g = threadIdx.x - slot * tpf;
    const int lane = threadIdx.x & 31;
    unsigned long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
    const int k = code.k, kw = code.kw, nw = code.nw;
    const uint32_t tail = (code.n & 31) ? (1u << (code.n & 31)) - 1u : 0xffffffffu;
    const bool stage = nw <= kStageW;
    const uint4 *tab = reinterpret_cast<const uint4 *>(asmtab);     // null: per-bit gathers
    // uniform trip count over the block (every thread meets the barriers)
    for (int64_t fb = int64_t(blockIdx.x) * fpb; fb < frames; fb += int64_t(gridDim.x) * fpb) {
        const int64_t f = fb + slot;
        int ie = 0, ce = 0;
        const uint32_t *b = bits + f * nw;
        const uint32_t *m = info + f * kw;
        // codeword-bit errors, word-wise.  Info-bit errors (decoded bit at H
        // column perm[t] against message bit t): with the encoder's deposit
        // table (both halves of perm ascend, every make_G here) also
        // word-wise -- the message bits that land in word j, deposited into
        // its info mask as the encoder does, against the decoded word under
        // that mask -- instead of a scattered gather per bit (C4: 2.0 ms for
        // 200k frames); without it, a gather per bit from the decoded row,
        // staged in shared memory when short (n <= 2048)
        if (f < frames) {
            const uint32_t *c = cw + f * nw;
#pragma unroll 2
            for (int w = g; w < nw; w += tpf) {
                const uint32_t bw = __ldg(b + w);
                uint32_t x = bw ^ __ldg(c + w);
                if (w == nw - 1) x &= tail;
                ce += __popc(x);
                if (tab) {
                    const uint4 h = __ldg(tab + 4 * w), u = __ldg(tab + 4 * w + 1), v4 = __ldg(tab + 4 * w + 2);
                    const uint32_t mi = h.x, sa = h.z;
                    uint32_t mw = 0u;
                    if (mi) {
                        const int w0 = int(sa >> 5);
                        const uint32_t lo = __ldg(m + w0), hi = w0 + 1 < kw ? __ldg(m + w0 + 1) : 0u;
                        mw = __funnelshift_r(lo, hi, sa & 31u);
                    }
                    const uint32_t mv[5] = {u.x, u.y, u.z, u.w, v4.x};
                    ie += __popc((bw ^ expand32(mw, mv, mi)) & mi);
                } else if (stage) {
                    s_b[slot][w] = bw;
                }
            }
        }
        if (!tab) {
            if (stage) {
                if (tpf == 32) __syncwarp();
                else __syncthreads();
            }
            if (f < frames) {
#pragma unroll 4
                for (int t = g; t < k; t += tpf) {
                    const int v = __ldg(code.perm + t);
                    const uint32_t zw = stage ? s_b[slot][v >> 5] : __ldg(b + (v >> 5));
                    ie += int(((zw >> (v & 31)) ^ (__ldg(m + (t >> 5)) >> (t & 31))) & 1u);
                }
            }
        }
        ie = __reduce_add_sync(0xffffffffu, ie);
        ce = __reduce_add_sync(0xffffffffu, ce);
        if (tpf > 32) {
            if (g == 0) fr_ie[slot] = 0, fr_ce[slot] = 0;
            __syncthreads();
            if (lane == 0) atomicAdd(&fr_ie[slot], ie), atomicAdd(&fr_ce[slot], ce);
            __syncthreads();
            ie = fr_ie[slot];
            ce = fr_ce[slot];
            __syncthreads();                           // read before the next pass resets them
        }
        if (g == 0 && f < frames) {
            c0 += ie;
            c1 += ce;
            c2 += ie > 0;
            c3 += (syn[f] && ce > 0);
            c4 += iters[f];
            c5 += 1;
        }
    }
    __syncthreads();
    if (g == 0 && (c5 | c4)) {
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
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // measured: C1 (kw = 2) 11.4 -> 6 us cold; at kw = 9..25 (Table I) the
    // per-lane scattered P loads made it 10x slower than the tiled path
    if (D.kw <= 4 && frames * int64_t(D.n) * D.kw <= (int64_t(1) << 26)) {
        const int grid = int(std::min<int64_t>((frames + 7) / 8, int64_t(ldpc::sm_count()) * 16));
        ldpc::encode_small_kernel<<<dim3(unsigned(std::max(grid, 1))), 256, 0, s>>>(D, d_info, d_cw, frames);
        return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
    }
    // parity words: on the tensor cores (encode_mma.cu) for long messages in
    // large batches, else the INT-pipe binary GEMM; identical bits
    cudaError_t merr = cudaSuccess;
    const bool mma = ldpc::encode_parity_mma(D, d_info, d_cw, frames, s, &merr);
    if (merr != cudaSuccess) return LDPC_ERR_CUDA;
    const unsigned col_tiles = mma ? 0u : unsigned(D.npar_pad / ldpc::kEncColTile);
    const int64_t max_chunk = int64_t(65535) * ldpc::kEncTF;      // gridDim.y limit
    for (int64_t f0 = 0; f0 < frames && col_tiles > 0; f0 += max_chunk) {
        const int64_t nf = std::min<int64_t>(max_chunk, frames - f0);
        const dim3 grid(col_tiles, unsigned((nf + ldpc::kEncTF - 1) / ldpc::kEncTF));
        ldpc::encode_parity_kernel<<<grid, 256, 0, s>>>(D, d_info + f0 * D.kw, d_cw + f0 * D.nw, nf);
    }
    const size_t smemw = sizeof(uint32_t) * size_t(ldpc::kAsmWarps) * size_t(D.kw + (D.n - D.k + 31) / 32 + 2);
    const char *aenv = std::getenv("LDPC_ASM_WARP");
    if (D.asmtab && smemw <= 200 * 1024 && !(aenv && std::atoi(aenv) == 0)) {
        if (smemw > 48 * 1024 &&
            !ldpc::ensure_smem_attribute(reinterpret_cast<const void *>(&ldpc::encode_assemble_dep_kernel), smemw))
            return LDPC_ERR_CUDA;
        // as many CTAs per SM as shared memory holds (C4: 4, i.e. 32 warps)
        const int per_sm = int(std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (smemw + 1024))));
        const int grid = int(std::min<int64_t>((frames + ldpc::kAsmWarps - 1) / ldpc::kAsmWarps,
                                               int64_t(ldpc::sm_count()) * per_sm));
        ldpc::encode_assemble_dep_kernel<<<std::max(grid, 1), ldpc::kAsmWarps * 32, smemw, s>>>(D, d_info, d_cw,
                                                                                             frames);
        return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
    }
    const size_t smem = sizeof(uint32_t) * size_t(D.kw + (D.n - D.k + 31) / 32);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(ldpc::encode_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) !=
            cudaSuccess)
        return LDPC_ERR_CUDA;
    const int grid2 = int(std::min<int64_t>(frames, int64_t(ldpc::sm_count()) * 8));
    ldpc::encode_assemble_kernel<<<grid2, 256, smem, s>>>(D, d_info, d_cw, frames);
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
    // threads per frame: a warp once the batch fills 8 warps on every SM,
    // else up to 256 so a small batch is spread over the whole GPU
    const int64_t sms = ldpc::sm_count();
    int tpf = 32;
    while (tpf < 256 && frames * int64_t(tpf) * 2 <= sms * 256 * 8) tpf *= 2;
    const int fpb = 256 / tpf;
    const int grid = int(std::min<int64_t>((frames + fpb - 1) / fpb, sms * 8));
    // the encoder's deposit table (LDPC_ASM_WARP=0 turns it off here too:
    // the per-bit gather path, A/B and tests)
    const char *aenv = std::getenv("LDPC_ASM_WARP");
    const uint32_t *tab = (aenv && std::atoi(aenv) == 0) ? nullptr : code->dev.asmtab;
    ldpc::count_kernel<<<dim3(unsigned(std::max(grid, 1))), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        code->dev, d_info, d_bits, d_cw, d_syndrome_ok, d_iters, frames, tpf, tab,
        reinterpret_cast<unsigned long long *>(d_counters6));
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // extern "C"
