// spa_band.cu -- the Sum-Product decoder specialised for regular Gallager
// codes built by ldpc_make_H (band construction S:52): the hot path of
// every BASELINE.json config.  Same algorithm and schedule as spa_decode.cu
// (Eqs. 4-8; flooding, Alg. 1); the structure of H is
// used to cut instructions and shared-memory traffic:
//
//  * Band 0 row r holds variables [r wr, (r+1) wr): the thread that owns
//    band-0 row r keeps that row's E_cv in REGISTERS across iterations, reads
//    the row's L_v as contiguous vectors, and performs the variable-node update
//    (Eq. 7) for exactly those wr variables.  Only the E of bands 1..wc-1 and
//    L (and R when it fits) live in shared memory -- which is what lets an
//    n = 16200 frame decode inside one SM (2n + n floats = 194 KB).
//  * Graph indices are pre-scaled byte offsets into the frame's shared-memory
//    image (DeviceLayout::band_lidx / band_vpos), read with vector loads.
//  * All LLRs are carried in log2 units (L' = L log2 e): phi becomes
//    psi(y) = log2(e) phi(y ln 2), still self-inverse, and e^-x becomes a bare
//    ex2 on the SFU.  R is scaled on ingest, posteriors rescaled on output.
//  * One CTA decodes one frame at a time (persistent grid); frames are taken
//    from a global atomic counter, so early-terminating frames free their CTA
//    immediately.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {
using namespace band;

#include "channel_common.cuh"
#include "band_kernel.cuh"

template <int WR, int WC, int B0>
void *pick_et(bool et, int mode) {
    if (mode == 2)
        return et ? reinterpret_cast<void *>(&band_kernel<WR, WC, B0, true, 2>)
                  : reinterpret_cast<void *>(&band_kernel<WR, WC, B0, false, 2>);
    if (mode == 1)
        return et ? reinterpret_cast<void *>(&band_kernel<WR, WC, B0, true, 1>)
                  : reinterpret_cast<void *>(&band_kernel<WR, WC, B0, false, 1>);
    return et ? reinterpret_cast<void *>(&band_kernel<WR, WC, B0, true, 0>)
              : reinterpret_cast<void *>(&band_kernel<WR, WC, B0, false, 0>);
}

template <int WR, int WC>
void *pick_b0(int b0, bool et, int vm) {
    switch (b0) {
        case 1: return pick_et<WR, WC, 1>(et, vm);
        case 2: return pick_et<WR, WC, 2>(et, vm);
        case 3: return pick_et<WR, WC, 3>(et, vm);
        case 4: return pick_et<WR, WC, 4>(et, vm);
    }
    return nullptr;
}

template <int WR, int WC>
void *pick_b0_small(int b0, bool et, int vm) {
    switch (b0) {
        case 1: return pick_et<WR, WC, 1>(et, vm);
        case 2: return pick_et<WR, WC, 2>(et, vm);
    }
    return nullptr;
}

// (wc, wr) instantiated: the BASELINE.json configs ((3, 4), (3, 6), (3, 12))
// and the paper's Table I (wr = 12 with wc = 9, 6, 3).
void *pick_band_kernel(int wr, int wc, int b0, bool et, int vm) {
    if (wc == 3) {
        switch (wr) {
            case 4: return pick_b0<4, 3>(b0, et, vm);
            case 6: return pick_b0<6, 3>(b0, et, vm);
            case 12: return pick_b0<12, 3>(b0, et, vm);
        }
    } else if (wr == 12 && wc == 6) {
        return pick_b0_small<12, 6>(b0, et, vm);
    } else if (wr == 12 && wc == 9) {
        return pick_b0_small<12, 9>(b0, et, vm);
    }
    return nullptr;
}

// ---------------------------------------------------------------------------
// Cluster band kernel: frames too large for one SM (C5: n = 64800, 1.04 MB of
// message state).  A cluster of C CTAs decodes one frame; CTA q owns rows
// [q mbq, (q+1) mbq) of every band and the variables of its band-0 rows, and
// keeps their E (band 0 in registers, bands >= 1 in shared memory) and L in
// shared memory.  Values owned by another CTA of the cluster are read from
// the frame's global copies Lg / Eg (L2-resident; random DSMEM access was
// measured 10-20x slower, profiles/r01_microbench.txt), which every CTA
// refreshes with coalesced stores after each phase; a cluster barrier
// (release/acquire) separates the phases.  Fixed-iteration mode only.
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ float ld_l_or_g(const char *smem, const float *g, int32_t idx) {
    return idx >= 0 ? *reinterpret_cast<const float *>(smem + idx) : __ldcg(g + ~idx);
}

struct ClusterArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
    float *gstate;          // per cluster slot: Lg[n] | Eg[(wc-1) n] | Rg[n] | flags[16]
    int64_t slot_floats;
};

// ET: early termination (reading Q11).  The syndrome of z^{t-1} is computed in
// check phase t from the L values the rows read anyway; each CTA ORs its rows
// into iflags[q] before the cluster barrier that ends the check phase, and
// every CTA reads all C flags after it, so the stop decision is uniform over
// the cluster (the flags are rewritten only after the next barrier).
template <int WR, int WC, int B0, int C, bool ET>
__global__ void __launch_bounds__(1024, 1) band_cluster_kernel(const ClusterArgs a) {
    extern __shared__ __align__(16) char smem[];
    const DeviceCode &code = a.code;
    const int n = code.n, mb = code.mb;
    const int mbq = mb / C, nq = n / C;
    const int T = blockDim.x, tt = threadIdx.x;
    constexpr int NB = WC - 1;
    constexpr int B1 = NB * B0;
    const int q = int(blockIdx.x % C);
    const int64_t cid = blockIdx.x / C, nclusters = gridDim.x / C;
    const uint32_t lbase = uint32_t(NB) * uint32_t(mbq) * WR * 4u;      // own L after own E_hi
    float *Ls = reinterpret_cast<float *>(smem + lbase);
    float *Lg = a.gstate + cid * a.slot_floats;
    float *Eg = Lg + n;
    float *Rg = Eg + int64_t(NB) * n;
    int *flags = reinterpret_cast<int *>(Rg + n);
    int *iflags = flags + 32;                      // per-iteration syndrome flags (ET)
    const int32_t *lidx = code.cband_lidx;
    const int32_t *vpos = code.cband_vpos;

    for (int64_t f = cid; f < a.frames; f += nclusters) {
        // ingest own variables: R (log2 units) to Rg, L = R to Ls and Lg; E = 0
        const float *src = a.llr + f * int64_t(n) + int64_t(q) * nq;
        for (int v4 = tt; v4 < (nq >> 2); v4 += T) {
            float4 r = __ldg(reinterpret_cast<const float4 *>(src) + v4);
            r.x = fminf(fmaxf(r.x, -30.0f), 30.0f) * kL2E;
            r.y = fminf(fmaxf(r.y, -30.0f), 30.0f) * kL2E;
            r.z = fminf(fmaxf(r.z, -30.0f), 30.0f) * kL2E;
            r.w = fminf(fmaxf(r.w, -30.0f), 30.0f) * kL2E;
            reinterpret_cast<float4 *>(Ls)[v4] = r;
            reinterpret_cast<float4 *>(Lg + int64_t(q) * nq)[v4] = r;
            reinterpret_cast<float4 *>(Rg + int64_t(q) * nq)[v4] = r;
        }
        for (int i = tt; i < int(lbase >> 4); i += T) reinterpret_cast<float4 *>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        float e0[B0][WR];
#pragma unroll
        for (int k = 0; k < B0; ++k)
#pragma unroll
            for (int j = 0; j < WR; ++j) e0[k][j] = 0.0f;
        cluster_sync_all();

        int32_t iters = a.max_iter;
        bool stopped = false;
        for (int t = 1; t <= a.max_iter; ++t) {
            // check phase over own rows (and the syndrome of z^{t-1} when ET)
            uint32_t synd = 0;
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = tt + k * T;
                if (r < mbq) {
                    float lv[WR], x[WR];
                    lds_row<WR>(reinterpret_cast<const char *>(Ls), uint32_t(r) * WR * 4u, lv);
                    uint32_t rp = 0;
#pragma unroll
                    for (int j = 0; j < WR; ++j) {
                        x[j] = lv[j] - e0[k][j];
                        if (ET) rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
                    }
                    synd |= rp;
                    check_row<WR, !ET>(x, e0[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < B1; ++k) {
                const int r = tt + k * T;                 // local row over bands >= 1
                if (r < NB * mbq) {
                    const int b = r / mbq, lr = r - b * mbq;
                    const int64_t gpos = int64_t(b) * n + int64_t(q * mbq + lr) * WR;   // Eg / lidx position
                    int32_t li[WR];
                    float e[WR], x[WR];
                    ldg_idx<WR>(lidx + gpos, li);
                    lds_row<WR>(smem, uint32_t(r) * WR * 4u, e);
                    uint32_t rp = 0;
#pragma unroll
                    for (int j = 0; j < WR; ++j) {
                        const float lv = ld_l_or_g(smem, Lg, li[j]);
                        x[j] = lv - e[j];
                        if (ET) rp ^= (lv >= 0.0f) ? 1u : 0u;
                    }
                    synd |= rp;
                    check_row<WR, !ET>(x, e);
                    sts_row<WR>(smem, uint32_t(r) * WR * 4u, e);
                    sts_row<WR>(reinterpret_cast<char *>(Eg + gpos), 0u, e);
                }
            }
            if (ET) {
                const int any = __syncthreads_or(synd != 0);
                if (tt == 0) iflags[q] = any;
            }
            cluster_sync_all();
            if (ET && t > 1) {
                int any = 0;
                for (int i = 0; i < C; ++i) any |= __ldcg(iflags + i);
                if (!any) {                        // z^{t-1} has zero syndrome: stop (reading c6)
                    iters = t - 1;
                    stopped = true;
                    break;
                }
            }
            // variable phase over own variables
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = tt + k * T;
                if (r < mbq) {
                    const int64_t v0 = int64_t(q * mbq + r) * WR;
                    float rv[WR], lv[WR];
                    int32_t vp[WR * NB];
                    lds_row<WR>(reinterpret_cast<const char *>(Rg + v0), 0u, rv);
                    ldg_idx<WR * NB>(vpos + v0 * NB, vp);
#pragma unroll
                    for (int j = 0; j < WR; ++j) {
                        float s = rv[j] + e0[k][j];
#pragma unroll
                        for (int b = 0; b < NB; ++b) s += ld_l_or_g(smem, Eg, vp[j * NB + b]);
                        lv[j] = s;
                    }
                    sts_row<WR>(reinterpret_cast<char *>(Ls), uint32_t(r) * WR * 4u, lv);
                    sts_row<WR>(reinterpret_cast<char *>(Lg + v0), 0u, lv);
                }
            }
            cluster_sync_all();
        }
        // syndrome of z = [L >= 0] over own rows, OR-ed across the cluster
        uint32_t synd = 0;
        for (int r = tt; r < mbq; r += T) {
            uint32_t rp = 0;
            for (int j = 0; j < WR; ++j) rp ^= (Ls[r * WR + j] >= 0.0f) ? 1u : 0u;
            synd |= rp;
        }
        for (int r = tt; r < NB * mbq; r += T) {
            const int b = r / mbq, lr = r - b * mbq;
            const int64_t gpos = int64_t(b) * n + int64_t(q * mbq + lr) * WR;
            uint32_t rp = 0;
            for (int j = 0; j < WR; ++j) rp ^= (ld_l_or_g(smem, Lg, __ldg(lidx + gpos + j)) >= 0.0f) ? 1u : 0u;
            synd |= rp;
        }
        const int any = __syncthreads_or(synd != 0);
        if (tt == 0) flags[q] = any;
        cluster_sync_all();
        // outputs: CTA q writes a word-aligned slice of the frame's bits
        const int nw = code.nw;
        const int wper = (nw + C - 1) / C;
        const int w0 = q * wper, w1 = min(nw, w0 + wper);
        uint32_t *bits = a.bits + f * int64_t(nw);
        for (int v = w0 * 32 + tt; v < w1 * 32; v += T) {
            const bool z = (v < n) ? (__ldcg(Lg + v) >= 0.0f) : false;
            const uint32_t word = __ballot_sync(0xffffffffu, z);
            if ((tt & 31) == 0) bits[v >> 5] = word;
        }
        if (a.posterior) {
            float *dst = a.posterior + f * int64_t(n) + int64_t(q) * nq;
            for (int v = tt; v < nq; v += T) dst[v] = Ls[v] * kLn2;
        }
        if (q == 0 && tt == 0) {
            int ok = 1;
            for (int i = 0; i < C; ++i) ok &= (__ldcg(flags + i) == 0);
            a.syn_ok[f] = uint8_t(ok || stopped);
            a.iters[f] = iters;
        }
        cluster_sync_all();     // Lg / flags are reused by the next frame
    }
}

template <int WR, int B0, bool ET>
void *pick_cluster_c(int C) {
    switch (C) {
        case 2: return reinterpret_cast<void *>(&band_cluster_kernel<WR, 3, B0, 2, ET>);
        case 4: return reinterpret_cast<void *>(&band_cluster_kernel<WR, 3, B0, 4, ET>);
        case 8: return reinterpret_cast<void *>(&band_cluster_kernel<WR, 3, B0, 8, ET>);
    }
    return nullptr;
}

void *pick_cluster_kernel(int wr, int wc, int b0, int C, bool et) {
    if (wc != 3 || wr != 6) return nullptr;
    switch (b0) {
        case 1: return et ? pick_cluster_c<6, 1, true>(C) : pick_cluster_c<6, 1, false>(C);
        case 2: return et ? pick_cluster_c<6, 2, true>(C) : pick_cluster_c<6, 2, false>(C);
        case 3: return et ? pick_cluster_c<6, 3, true>(C) : pick_cluster_c<6, 3, false>(C);
    }
    return nullptr;
}

}  // namespace

bool cluster_plan(const ldpc_code &c, int64_t frames, bool et, ClusterPlan &p) {
    if (!c.gallager || !c.regular_col || (c.n & 3)) return false;
    const int C = band_cluster_size(c.n, c.wc, c.wr);
    if (C == 0) return false;
    const int mbq = c.n / c.wr / C, nq = c.n / C;
    if (nq & 3) return false;
    const int b0 = std::max(1, (mbq + 1023) / 1024);
    void *k = pick_cluster_kernel(c.wr, c.wc, b0, C, et);
    if (!k) return false;
    p.kernel = k;
    p.cluster = C;
    p.threads = ((mbq + b0 - 1) / b0 + 31) / 32 * 32;
    p.smem = size_t(c.wc) * size_t(nq) * 4;
    if (!ensure_smem_attribute(k, p.smem, C > 8)) return false;
    int nclusters = occupancy_clusters(k, p.threads, p.smem, C);
    if (nclusters < 1) return false;
    nclusters = int(std::min<int64_t>(nclusters, std::max<int64_t>(frames, 1)));
    p.grid = nclusters * C;
    p.slot_floats = (int64_t(c.wc + 1) * c.n + 64 + 63) & ~int64_t(63);     // + flags[32], iflags[32]
    p.ws_bytes = size_t(nclusters) * size_t(p.slot_floats) * 4;
    return true;
}

ldpc_status cluster_launch(const ldpc_code &c, const ClusterPlan &p, const float *llr, int64_t frames,
                           const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                           void *ws, size_t ws_bytes, void *stream) {
    if (!ws || ws_bytes < p.ws_bytes) return LDPC_ERR_ARG;
    ClusterArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.bits = bits;
    a.syn_ok = syn;
    a.iters = iters;
    a.posterior = post;
    a.gstate = static_cast<float *>(ws);
    a.slot_floats = p.slot_floats;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(p.cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(p.grid));
    cfg.blockDim = dim3(unsigned(p.threads));
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {&a};
    cudaError_t e = cudaLaunchKernelExC(&cfg, p.kernel, args);
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

bool band_plan(const ldpc_code &c, int64_t frames, bool et, int variant, BandPlan &p, int max_iter, bool lane_pairs) {
    if (!c.gallager || !c.regular_col || (c.n & 3)) return false;
    const int mb = c.n / c.wr;
    const int sms = device_attribute(cudaDevAttrMultiProcessorCount);
    const int optin = device_attribute(cudaDevAttrMaxSharedMemoryPerBlockOptin);
    if (sms < 1 || optin < 1) return false;
    int b0 = std::max(1, (mb + 1023) / 1024);
    const int fb0 = band_fixed_b0(c.n, c.wr, c.wc, frames, sms);
    if (!std::getenv("LDPC_NO_NFIX") && fb0 > b0) b0 = fb0;
    if (b0 > 4) return false;
    p.b0 = b0;
    const size_t base = size_t(c.wc) * size_t(c.n) * 4;          // E_hi + L
    const size_t with_r = base + size_t(c.n) * 4;
    const size_t reserve = 1024;                                  // static smem + driver
    if (base + reserve > size_t(optin)) return false;
    p.r_in_smem = with_r + reserve <= size_t(optin);
    // Variable-major E (variant 4) drops the variable phase's index loads and
    // gathers; it pays off when the indices no longer fit in L1 (large n).
    p.vm = variant == 4 || variant == 6 ||
           (variant == 0 && (!p.r_in_smem || c.wc > 3 ||
                             (!std::getenv("LDPC_NO_NFIX") && band_fixed_vm(c.n, c.wr, c.wc))));
    // 16-bit offsets (variant 6, auto with VM when n <= 16383): +2% on C4
    p.mode = p.vm ? (((variant == 6 || variant == 0) && c.n <= 16383) ? 2 : 1) : 0;
    p.threads = ((mb + b0 - 1) / b0 + 31) / 32 * 32;
    // Codes with long per-thread chains (wc x wr >= 64 edges per thread and
    // iteration: Table I R1/4, R1/2) split every check row over a lane pair
    // (LPR = 2): twice the warps per frame, half the chain per thread, more
    // warps per SM where shared memory caps the CTAs; without psi votes bit
    // for bit the same results.  Measured (SFU roofline): T1-R1/4 29 -> 40%
    // at 1000 frames, 39 -> 47% at 100k; T1-R1/2 33 -> 42%, 39 -> 52%.
    p.lpr = 1;
    void *k = nullptr;
    const bool nfix = !std::getenv("LDPC_NO_NFIX");
    if (lane_pairs && nfix && !std::getenv("LDPC_NO_LPR2") && (c.wc * c.wr >= 64 || std::getenv("LDPC_LPR2_ALL"))) {
        k = pick_band_kernel_fixed(c.n, c.wr, c.wc, b0, et, p.mode, max_iter, 2);
        if (k) {
            p.lpr = 2;
            p.threads *= 2;
        }
    }
    if (!k && nfix) k = pick_band_kernel_fixed(c.n, c.wr, c.wc, b0, et, p.mode, max_iter);
    if (!k) k = pick_band_kernel(c.wr, c.wc, b0, et, p.mode);
    if (!k) return false;
    p.smem = p.r_in_smem ? with_r : base;
    if (p.threads > (c.wc > 3 ? 256 * p.lpr : 1024)) return false;    // the kernel's launch bound
    p.kernel = k;
    if (!ensure_smem_attribute(k, p.smem)) return false;
    const int per_sm = occupancy_blocks(k, p.threads, p.smem);
    if (per_sm < 1) return false;
    p.capacity = int64_t(sms) * per_sm;
    p.grid = int(std::max<int64_t>(1, std::min<int64_t>(frames, p.capacity)));
    p.ws_bytes = 256 + (p.r_in_smem ? 0 : size_t(p.grid) * size_t(c.n) * 4);
    return true;
}

ldpc_status band_launch(const ldpc_code &c, const BandPlan &p, const float *llr, int64_t frames,
                        const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                        void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ws || ws_bytes < p.ws_bytes) return LDPC_ERR_ARG;
    BandArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.early_term = o.early_term ? 1 : 0;
    a.bits = bits;
    a.syn_ok = syn;
    a.iters = iters;
    a.posterior = post;
    // one frame per CTA (the grid holds the batch): no counter to zero
    const bool stat = int64_t(p.grid) >= frames;
    a.frame_counter = stat ? nullptr : static_cast<unsigned long long *>(ws);
    a.r_global = p.r_in_smem ? nullptr : reinterpret_cast<float *>(static_cast<char *>(ws) + 256);
    a.r_in_smem = p.r_in_smem ? 1 : 0;
    // Row stride = block size.  (A stride of exactly ceil(mb / B0), which gives
    // every thread the same row count, measured 1.7 points slower on C4.)
    a.row_stride = p.threads / p.lpr;
    if (!stat && cudaMemsetAsync(ws, 0, 8, s) != cudaSuccess) return LDPC_ERR_CUDA;
    void *args[] = {&a};
    cudaError_t e = cudaLaunchKernel(p.kernel, dim3(unsigned(p.grid)), dim3(unsigned(p.threads)), args, p.smem, s);
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // namespace ldpc
