// encode_mma.cu -- the parity half of the encoder (Eq. 3, G in
// standard form) on the 5th-generation tensor cores.
//
// The parity bits of a batch are the GF(2) product M P: M the frames' message
// bits (frames x k), P the standard form's parity block (k x (n - k)).  That
// is a dense contraction, so it runs as an integer matrix product on
// tcgen05: each bit becomes an unsigned 8-bit 0/1 operand, the tensor cores
// accumulate exact int32 dot products (at most k <= 32400 << 2^31), and the
// parity bit is the accumulator's least significant bit -- the same GF(2)
// sum the INT-pipe kernel (codec_kernels.cu encode_parity_kernel) forms with
// AND/XOR and popc, so the two give identical bits (tests).
//
// CTA tile: 256 frames x 256 parity columns, as two M = 128 accumulators of
// N = 256 int32 columns in Tensor Memory (all 512 columns).  k is streamed in
// stages of 128 bits through shared memory, three stages deep:
//   * warps 0-7 (producers) read the stage's message words (L2-resident rows
//     of the info array) and the stage's words of 256 P columns (the
//     encoder's bind-time transposed P, `pt`), expand every bit to a byte
//     (one IMAD per nibble: nibble * 0x204081 & 0x01010101) and store the
//     bytes in the UMMA K-major no-swizzle layout -- core matrices of 8 rows
//     x 16 bytes, [16-byte K chunk][8-row group][row][16 B];
//   * warp 8, one elected lane, issues 8 tcgen05.mma.kind::i8 (M 128, N 256,
//     K 32) per stage and commits them to the stage's "empty" barrier;
//   * after the last stage, warps 0-3 read the accumulators back
//     (tcgen05.ld 32x32b: warp w <-> TMEM lanes 32 w ..), pack the LSBs of 32
//     columns per word and write the parity words into the tail of the
//     frame's codeword row, where encode_assemble_kernel expects them.
// Expanding bits in shared memory keeps the operands' global traffic at one
// bit per element (P of C5 is 131 MB as bits, 1 GB as bytes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ldpc_internal.h"

namespace ldpc {
namespace {

constexpr int kMmaTileM = 256;          // frames per CTA (two M = 128 accumulators)
constexpr int kMmaTileN = 256;          // parity columns per CTA
constexpr int kMmaStageW = 4;           // message words (128 bits of k) per stage
constexpr int kMmaStages = 3;
constexpr int kMmaProducers = 256;      // warps 0-7
constexpr int kMmaThreads = kMmaProducers + 32;
constexpr uint32_t kOpBytes = 256u * kMmaStageW * 32u;          // one operand stage: 256 rows x 128 bytes
constexpr uint32_t kStageBytes = 2u * kOpBytes;                  // A + B
constexpr size_t kMmaSmem = size_t(kMmaStages) * kStageBytes + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows
// x 16 bytes; lbo = byte distance between the two 16-byte K chunks of one
// MMA, sbo = between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3fffu);
    d |= uint64_t((lbo >> 4) & 0x3fffu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3fffu) << 32;
    d |= uint64_t(1) << 46;
    return d;
}
// instruction descriptor: D s32 (c_format 2), A/B unsigned 8-bit, both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t kIdesc = (2u << 4) | (uint32_t(kMmaTileN >> 3) << 17) | (uint32_t(128 >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// 32 bits -> 32 bytes of 0/1 (byte j <-> bit j), as two 16-byte K chunks
__device__ __forceinline__ void expand_bits(uint32_t x, uint4 &lo, uint4 &hi) {
    auto nib = [&](int q) { return ((x >> (4 * q)) & 0xfu) * 0x00204081u & 0x01010101u; };
    lo = make_uint4(nib(0), nib(1), nib(2), nib(3));
    hi = make_uint4(nib(4), nib(5), nib(6), nib(7));
}

__global__ void __launch_bounds__(kMmaThreads, 1)
    encode_mma_kernel(const DeviceCode code, const uint32_t *__restrict__ info, uint32_t *__restrict__ cw,
                      int64_t frames) {
    extern __shared__ __align__(1024) char smem_raw[];
    // 1024-byte aligned operand area, barriers behind it
    char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bars[2 * kMmaStages + 1];
    __shared__ uint32_t s_tmem;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kw = code.kw, npp = code.npar_pad, nw = code.nw;
    const int npw = (code.n - code.k + 31) / 32;
    const int n0 = blockIdx.x * kMmaTileN;
    const int64_t f0 = int64_t(blockIdx.y) * kMmaTileM;
    const int nstages = (kw + kMmaStageW - 1) / kMmaStageW;
    const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[kMmaStages]),
                   done = smem_u32(&bars[2 * kMmaStages]);
    const uint32_t op0 = smem_u32(smem);
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kMmaStages; ++s) {
            mbar_init(full0 + 8u * s, kMmaProducers / 32);
            mbar_init(empty0 + 8u * s, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;

    if (warp < 8) {
        // ---- producers: stage j's bits -> bytes in the K-major core-matrix layout
        const int r = tid;                                  // operand row 0..255
        const bool frow = f0 + r < frames;
        const uint32_t *irow = info + (f0 + r) * int64_t(kw);
        const bool prow = n0 + r < npp;
        // row r of either operand: core matrix (chunk c, group r / 8), row r % 8
        const uint32_t rbyte = uint32_t(r >> 3) * 128u + uint32_t(r & 7) * 16u;
        for (int j = 0; j < nstages; ++j) {
            const int s = j % kMmaStages;
            if (j >= kMmaStages) mbar_wait(empty0 + 8u * s, uint32_t((j / kMmaStages - 1) & 1));
            char *A = smem + size_t(s) * kStageBytes, *B = A + kOpBytes;
            const int w0 = j * kMmaStageW;
#pragma unroll
            for (int wi = 0; wi < kMmaStageW; ++wi) {
                const int w = w0 + wi;
                const uint32_t xa = (frow && w < kw) ? __ldg(irow + w) : 0u;
                const uint32_t xb = (prow && w < kw) ? __ldg(code.pt + size_t(w) * npp + n0 + r) : 0u;
                uint4 lo, hi;
                const uint32_t c0 = uint32_t(2 * wi) * 4096u + rbyte;     // 16-byte K chunk 2 wi, 32 groups x 128 B
                expand_bits(xa, lo, hi);
                *reinterpret_cast<uint4 *>(A + c0) = lo;
                *reinterpret_cast<uint4 *>(A + c0 + 4096u) = hi;
                expand_bits(xb, lo, hi);
                *reinterpret_cast<uint4 *>(B + c0) = lo;
                *reinterpret_cast<uint4 *>(B + c0 + 4096u) = hi;
            }
            // generic-proxy stores -> visible to the tensor core's async proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(full0 + 8u * s);
        }
        // ---- epilogue (warps 0-3): accumulator LSBs -> parity words
        if (warp < 4) {
            mbar_wait(done, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int h = 0; h < 2; ++h) {
                const int64_t f = f0 + 128 * h + 32 * warp + lane;
                for (int c = 0; c < kMmaTileN / 32; ++c) {
                    uint32_t v[32];
                    const uint32_t ta = tmem + (uint32_t(32 * warp) << 16) + uint32_t(h * kMmaTileN + 32 * c);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
                        "%30, %31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(ta)
                        : "memory");
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    uint32_t word = 0u;
#pragma unroll
                    for (int i = 0; i < 32; ++i) word |= (v[i] & 1u) << i;
                    const int pwi = n0 / 32 + c;
                    if (f < frames && pwi < npw) cw[f * int64_t(nw) + (nw - npw) + pwi] = word;
                }
            }
        }
    } else {
        // ---- MMA issuer: one elected lane of warp 8
        for (int j = 0; j < nstages; ++j) {
            const int s = j % kMmaStages;
            mbar_wait(full0 + 8u * s, uint32_t((j / kMmaStages) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                const uint32_t A = op0 + uint32_t(s) * kStageBytes, B = A + kOpBytes;
#pragma unroll
                for (int ks = 0; ks < kMmaStageW; ++ks) {       // K 32 per MMA: chunks 2 ks, 2 ks + 1
                    const uint64_t bd = umma_desc(B + uint32_t(2 * ks) * 4096u, 4096u, 128u);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint64_t ad = umma_desc(A + uint32_t(2 * ks) * 4096u + uint32_t(h) * 2048u, 4096u, 128u);
                        umma_i8(tmem + uint32_t(h * kMmaTileN), ad, bd, (j > 0 || ks > 0) ? 1u : 0u);
                    }
                }
                umma_commit(empty0 + 8u * s);
                if (j == nstages - 1) umma_commit(done);
            }
            __syncwarp();
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 8) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace

// Parity words of frames [0, frames) on the tensor cores (see the top of this
// file); false when the code or the batch does not take this path.
bool encode_parity_mma(const DeviceCode &D, const uint32_t *d_info, uint32_t *d_cw, int64_t frames,
                       cudaStream_t s, cudaError_t *err) {
    *err = cudaSuccess;
    const char *env = std::getenv("LDPC_ENC_MMA");
    if (env && std::atoi(env) == 0) return false;
    const bool force = env && std::atoi(env) == 1;
    // the INT-pipe kernel is as fast on short messages, and faster where the
    // 256 x 256 tiles would not fill the GPU (Table I at 1000 frames: 8 tiles,
    // measured 3.38 -> 3.23 Gbit/s on the MMA path)
    const int64_t tiles = (frames + kMmaTileM - 1) / kMmaTileM * ((D.npar_pad + kMmaTileN - 1) / kMmaTileN);
    if (!force && (D.kw < 16 || tiles < int64_t(device_attribute(cudaDevAttrMultiProcessorCount)))) return false;
    // per-device, thread-safe attribute cache (host_code.cpp)
    if (!ensure_smem_attribute(reinterpret_cast<const void *>(&encode_mma_kernel), kMmaSmem)) return false;
    const unsigned ntiles = unsigned((D.npar_pad + kMmaTileN - 1) / kMmaTileN);
    const int64_t max_chunk = int64_t(65535) * kMmaTileM;      // gridDim.y limit
    for (int64_t f0 = 0; f0 < frames; f0 += max_chunk) {
        const int64_t nf = std::min<int64_t>(max_chunk, frames - f0);
        const dim3 grid(ntiles, unsigned((nf + kMmaTileM - 1) / kMmaTileM));
        encode_mma_kernel<<<grid, kMmaThreads, kMmaSmem, s>>>(D, d_info + f0 * D.kw, d_cw + f0 * D.nw, nf);
    }
    *err = cudaGetLastError();
    return true;
}

}  // namespace ldpc
