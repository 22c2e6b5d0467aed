// spa_cluster.cu -- Sum-Product decoding of Gallager frames too large for one
// SM (C5: n = 64800, 1.04 MB of message state) by a thread-block cluster that
// exchanges whole message SEGMENTS between its CTAs with bulk DSMEM copies.
//
// Same algorithm and schedule as spa_band.cu (Eqs. 4-8; flooding,
// Alg. 1).  It is the on-chip analogue of the paper's stream mode
// (Alg. 1: interleaved node ownership, Send/Recv of L_vc and E_cv every
// half-iteration): CTA q of a C-CTA cluster owns
//   * band-0 rows [q mbq, (q+1) mbq) and their variables [q nq, (q+1) nq)
//     (band 0 is contiguous): their E lives in registers and the
//     variable update (Eq. 6/7) and band-0 check update run thread-locally;
//   * band-b >= 1 rows [q mbq, (q+1) mbq) (check-node update, Eq. 5).
// Each half-iteration, every CTA writes the messages it produces into a local
// SEND buffer laid out by destination CTA (random local shared-memory stores
// at precomputed 16-bit slots), then C threads each push one contiguous
// segment to one destination CTA with cp.async.bulk shared::cta ->
// shared::cluster, completing on the destination's mbarrier (complete_tx).
// Random remote 4-byte DSMEM accesses run at ~0.4/clk/SM
// (profiles/r01_microbench.txt); the segment exchange turns them into local
// random accesses plus bulk transfers.
//
// Buffers (floats, per CTA): SEND[cap], RECV[2][cap] (double-buffered by
// exchange parity).  Exchange h carries L_vc (variable -> check) or E_cv
// (check -> variable); one edge uses the same slot for both directions, so a
// phase reads RECV at slot s and writes SEND at the same slot s.
// Synchronisation per exchange h (x = h & 1):
//   1. writers: fence.proxy.async; __syncthreads
//   2. thread d < C: bulk copy of segment (q -> d) into d's RECV[x],
//      complete_tx on d's recv_bar[x]
//   3. all: wait recv_bar[x] (phase h >> 1)
//   4. thread 0 re-arms recv_bar[x] (expect_tx of exchange h + 2);
//      thread s < C arrives on CTA s's free_bar (its segment to us landed)
//   5. the next phase waits free_bar (exchange h) before writing SEND.
// A remote RECV[x] is free when we write it at exchange h + 2: that needs
// free_bar(h + 1) of ours, i.e. every destination passed step 1 of exchange
// h + 1, i.e. finished reading RECV[x] in its phase.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace cg = cooperative_groups;

namespace ldpc {
namespace {
using namespace band;

__device__ __forceinline__ uint32_t saddr(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// Default .acquire.cta scope: the awaited data is shared memory written by the
// async proxy (complete_tx), or nothing at all (free_bar).  A .cluster-scope
// acquire makes every poll invalidate L1 (CCTL.IVALL: 46% of stall samples in
// the first ncu capture) and evicts the cached slot tables.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_cluster),
                 "r"(src_cta), "r"(bytes), "r"(bar_cluster)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int D>
__device__ __forceinline__ void ld_u16_row(const uint16_t *p, uint32_t (&o)[D]) {
    // D 16-bit slots; p is 4-byte aligned when D is even
    if constexpr (D % 2 == 0) {
        const uint32_t *p32 = reinterpret_cast<const uint32_t *>(p);
#pragma unroll
        for (int w = 0; w < D / 2; ++w) {
            const uint32_t x = __ldg(p32 + w);
            o[2 * w] = x & 0xffffu;
            o[2 * w + 1] = x >> 16;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) o[j] = __ldg(p + j);
    }
}

struct XArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
};

// Shared memory: SEND | RECV0 | RECV1 (cap floats each) | recv_bar[2] | free_bar | flags[C]
template <int WR, int WC, int B0, int C>
__global__ void __launch_bounds__(1024, 1) xband_kernel(const XArgs a) {
    extern __shared__ __align__(128) char smem[];
    constexpr int NB = WC - 1;
    constexpr int B1 = NB * B0;
    const DeviceCode &code = a.code;
    const int n = code.n, mb = code.mb, mbq = mb / C, nq = n / C;
    const int T = blockDim.x, tt = threadIdx.x;
    const uint32_t cap_b = uint32_t(code.xcap) * 4u;
    const uint32_t q = cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    char *send = smem;
    char *recv0 = smem + cap_b;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 3 * cap_b);
    int *flags = reinterpret_cast<int *>(bars + 4);
    const uint32_t send_s = saddr(send), recv_s = saddr(recv0), bar_s = saddr(bars);
    const uint32_t free_s = bar_s + 16;
    const int32_t *sOff = code.xband_seg, *rOff = code.xband_seg + C * C, *sbytes = code.xband_seg + 2 * C * C;

    // bytes CTA q receives in an L exchange (from every variable owner s) and
    // in an E exchange (from every row owner d)
    uint32_t rx_l = 0, rx_e = 0;
#pragma unroll
    for (int s = 0; s < C; ++s) {
        rx_l += uint32_t(__ldg(sbytes + s * C + q));
        rx_e += uint32_t(__ldg(sbytes + q * C + s));
    }
    // exchange j of a frame (0..2T): even j carries L (to row owners), odd j E
    const int per_frame = 2 * a.max_iter + 1;
    if (tt == 0) {
        mbar_init(bar_s, 1);
        mbar_init(bar_s + 8, 1);
        mbar_init(free_s, C);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arm(bar_s, rx_l);                             // exchange 0: L
        mbar_arm(bar_s + 8, per_frame > 1 ? rx_e : rx_l);  // exchange 1
    }
    cluster_sync_all();

    uint32_t h = 0;      // exchanges completed by this CTA (over all frames)
    // Exchange h: SEND -> RECV[h & 1] of every CTA of the cluster.  type_l:
    // an L exchange (segment (q, d) from the send layout) or an E exchange
    // (segment (d, q) from the receive layout).
    auto exchange = [&](bool type_l, int j) {
        fence_proxy_async_smem();
        __syncthreads();
        const uint32_t x = h & 1u;
        if (tt < C) {
            const int d = tt;
            const uint32_t src = type_l ? uint32_t(__ldg(sOff + q * C + d)) : uint32_t(__ldg(rOff + d * C + q));
            const uint32_t dst = type_l ? uint32_t(__ldg(rOff + q * C + d)) : uint32_t(__ldg(sOff + d * C + q));
            const uint32_t nbytes = uint32_t(__ldg(sbytes + (type_l ? q * C + d : d * C + q)));
            if (nbytes)
                bulk_s2c(mapa_u32(recv_s + x * cap_b + dst, uint32_t(d)), send_s + src, nbytes,
                         mapa_u32(bar_s + 8u * x, uint32_t(d)));
        }
        mbar_wait(bar_s + 8u * x, (h >> 1) & 1u);
        if (tt == 0) {
            int jn = j + 2;
            if (jn >= per_frame) jn -= per_frame;
            mbar_arm(bar_s + 8u * x, (jn & 1) ? rx_e : rx_l);
        }
        if (tt < C) mbar_arrive_remote(mapa_u32(free_s, uint32_t(tt)));
        ++h;
    };
    // SEND may be rewritten once every destination holds exchange h - 1.
    auto send_free = [&]() {
        if (h > 0) mbar_wait(free_s, (h - 1) & 1u);
    };

    const uint16_t *ridx = code.xband_ridx, *sidx = code.xband_sidx;
    for (int64_t f = cid; f < a.frames; f += ncl) {
        const float *llr = a.llr + f * int64_t(n);
        float e0[B0][WR];
        uint32_t synd = 0;
        // ---- V-phase 0 (a1/a2): L = R, E = 0; send L_vc = R; band-0 check of t = 1
        send_free();
#pragma unroll
        for (int k = 0; k < B0; ++k) {
            const int r = tt + k * T;
            if (r < mbq) {
                const int v0 = (int(q) * mbq + r) * WR;
                float lv[WR];
                lds_row<WR>(reinterpret_cast<const char *>(llr), uint32_t(v0) * 4u, lv);   // global, 8B aligned rows
#pragma unroll
                for (int j = 0; j < WR; ++j) lv[j] = fminf(fmaxf(lv[j], -30.0f), 30.0f) * kL2E;
                uint32_t sl[WR * NB];
                ld_u16_row<WR * NB>(sidx + size_t(v0) * NB, sl);
#pragma unroll
                for (int j = 0; j < WR; ++j)
#pragma unroll
                    for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(send + sl[j * NB + b]) = lv[j];
                check_row<WR, true>(lv, e0[k]);
            }
        }
        exchange(true, 0);
        for (int t = 1; t <= a.max_iter; ++t) {
            const char *rin = recv0 + ((h - 1) & 1u) * cap_b;
            // ---- C-phase t (a3): rows of bands >= 1 owned by q
            send_free();
#pragma unroll
            for (int k = 0; k < B1; ++k) {
                const int r = tt + k * T;
                if (r < NB * mbq) {
                    const int b = r / mbq, lr = r - b * mbq;
                    uint32_t sl[WR];
                    ld_u16_row<WR>(ridx + size_t(b) * n + size_t(int(q) * mbq + lr) * WR, sl);
                    float x[WR], e[WR];
#pragma unroll
                    for (int j = 0; j < WR; ++j) x[j] = *reinterpret_cast<const float *>(rin + sl[j]);
                    check_row<WR, true>(x, e);
#pragma unroll
                    for (int j = 0; j < WR; ++j) *reinterpret_cast<float *>(send + sl[j]) = e[j];
                }
            }
            exchange(false, 2 * t - 1);
            // ---- V-phase t (a4/a5): L = R + sum E; send L_vc (L itself at t = T)
            const bool last = t == a.max_iter;
            rin = recv0 + ((h - 1) & 1u) * cap_b;
            send_free();
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = tt + k * T;
                if (r < mbq) {
                    const int v0 = (int(q) * mbq + r) * WR;
                    float lv[WR];
                    lds_row<WR>(reinterpret_cast<const char *>(llr), uint32_t(v0) * 4u, lv);
                    uint32_t sl[WR * NB];
                    ld_u16_row<WR * NB>(sidx + size_t(v0) * NB, sl);
                    float eb[WR * NB];
#pragma unroll
                    for (int j = 0; j < WR; ++j) {
                        lv[j] = fminf(fmaxf(lv[j], -30.0f), 30.0f) * kL2E + e0[k][j];
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            eb[j * NB + b] = *reinterpret_cast<const float *>(rin + sl[j * NB + b]);
                            lv[j] += eb[j * NB + b];
                        }
                    }
                    if (last) {
                        uint32_t rp = 0;      // band-0 row syndrome bit (Eq. 1)
#pragma unroll
                        for (int j = 0; j < WR; ++j) {
                            rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
#pragma unroll
                            for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(send + sl[j * NB + b]) = lv[j];
                        }
                        synd |= rp;
                    } else {
                        float x[WR];
#pragma unroll
                        for (int j = 0; j < WR; ++j) {
#pragma unroll
                            for (int b = 0; b < NB; ++b)
                                *reinterpret_cast<float *>(send + sl[j * NB + b]) = lv[j] - eb[j * NB + b];
                            x[j] = lv[j] - e0[k][j];
                        }
                        check_row<WR, true>(x, e0[k]);
                    }
                }
            }
            exchange(true, 2 * t);
        }
        // ---- a7: syndrome of z = [L >= 0]; rows of bands >= 1 see L at their slots
        const char *lin = recv0 + ((h - 1) & 1u) * cap_b;
        for (int r = tt; r < NB * mbq; r += T) {
            const int b = r / mbq, lr = r - b * mbq;
            uint32_t sl[WR];
            ld_u16_row<WR>(ridx + size_t(b) * n + size_t(int(q) * mbq + lr) * WR, sl);
            uint32_t rp = 0;
#pragma unroll
            for (int j = 0; j < WR; ++j) rp ^= (*reinterpret_cast<const float *>(lin + sl[j]) >= 0.0f) ? 1u : 0u;
            synd |= rp;
        }
        const int any = __syncthreads_or(synd != 0);
        // final L in variable order, into the idle receive buffer (its last
        // readers passed the barrier of exchange h - 1)
        float *lfin = reinterpret_cast<float *>(recv0 + (h & 1u) * cap_b);
        for (int i = tt; i < nq; i += T) {
            const uint32_t s0 = __ldg(sidx + (size_t(q) * nq + i) * NB);
            lfin[i] = *reinterpret_cast<const float *>(send + s0);
        }
        if (tt == 0) {
            int *f0 = cg::this_cluster().map_shared_rank(flags, 0);
            f0[q] = any;
        }
        cluster_sync_all();
        // ---- a6/a8: bits (words starting in q's variable range), posteriors, flags
        {
            const int nw = code.nw;
            const int w_lo = (int(q) * nq + 31) / 32;
            const int w_hi = (int(q) == C - 1) ? nw : ((int(q) + 1) * nq + 31) / 32;
            const float *lnext = (int(q) + 1 < C) ? cg::this_cluster().map_shared_rank(lfin, int(q) + 1) : lfin;
            uint32_t *bits = a.bits + f * int64_t(nw);
            // T is a multiple of 32: each warp covers whole words
            for (int base = w_lo * 32; base < w_hi * 32; base += T) {
                const int v = base + tt;
                if (v >= w_hi * 32) break;          // warp-uniform
                bool z = false;
                if (v < n) {
                    const int i = v - int(q) * nq;
                    z = (i < nq ? lfin[i] : lnext[i - nq]) >= 0.0f;
                }
                const uint32_t word = __ballot_sync(0xffffffffu, z);
                if ((tt & 31) == 0) bits[v >> 5] = word;
            }
            if (a.posterior) {
                float *dst = a.posterior + f * int64_t(n) + int64_t(q) * nq;
                for (int i = tt; i < nq; i += T) dst[i] = lfin[i] * kLn2;
            }
            if (q == 0 && tt == 0) {
                int ok = 1;
                for (int i = 0; i < C; ++i) ok &= (flags[i] == 0);
                a.syn_ok[f] = uint8_t(ok);
                a.iters[f] = a.max_iter;
            }
        }
        cluster_sync_all();     // lfin / flags are reused by the next frame
    }
}

template <int WR, int B0>
void *pick_x_c(int C) {
    switch (C) {
        case 4: return reinterpret_cast<void *>(&xband_kernel<WR, 3, B0, 4>);
        case 8: return reinterpret_cast<void *>(&xband_kernel<WR, 3, B0, 8>);
        case 16: return reinterpret_cast<void *>(&xband_kernel<WR, 3, B0, 16>);
    }
    return nullptr;
}

void *pick_xband_kernel(int wr, int wc, int b0, int C) {
    if (wc != 3 || wr != 6) return nullptr;
    switch (b0) {
        case 1: return pick_x_c<6, 1>(C);
        case 2: return pick_x_c<6, 2>(C);
        case 4: return pick_x_c<6, 4>(C);
    }
    return nullptr;
}

}  // namespace

bool xcluster_plan(const ldpc_code &c, int64_t frames, bool et, XClusterPlan &p) {
    if (et || !c.gallager || !c.regular_col || !c.dev.xcluster) return false;
    const int C = c.dev.xcluster;
    const int mbq = c.n / c.wr / C;
    int b0 = std::max(1, (mbq + 1023) / 1024);
    if (b0 == 3) b0 = 4;
    void *k = pick_xband_kernel(c.wr, c.wc, b0, C);
    if (!k) return false;
    p.kernel = k;
    p.cluster = C;
    p.threads = ((mbq + b0 - 1) / b0 + 31) / 32 * 32;
    if (p.threads * b0 * (c.wc - 1) < mbq * (c.wc - 1)) return false;
    p.smem = 3 * size_t(c.dev.xcap) * 4 + 32 + 4 * size_t(C);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem)) != cudaSuccess) return false;
    if (C > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return false;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(C));
    cfg.blockDim = dim3(unsigned(p.threads));
    cfg.dynamicSmemBytes = p.smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    const cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
    if (oe != cudaSuccess || nclusters < 1) {
        if (std::getenv("LDPC_DEBUG"))
            std::fprintf(stderr, "ldpc xcluster_plan: occupancy query: %s, clusters %d (C=%d, threads %d, smem %zu)\n",
                         cudaGetErrorString(oe), nclusters, C, p.threads, p.smem);
        cudaGetLastError();
        return false;
    }
    nclusters = int(std::min<int64_t>(nclusters, std::max<int64_t>(frames, 1)));
    p.grid = nclusters * C;
    p.ws_bytes = 0;
    return true;
}

ldpc_status xcluster_launch(const ldpc_code &c, const XClusterPlan &p, const float *llr, int64_t frames,
                            const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                            void *stream) {
    XArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.bits = bits;
    a.syn_ok = syn;
    a.iters = iters;
    a.posterior = post;
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

}  // namespace ldpc
