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
// Message state lives IN PLACE in two shared-memory regions per CTA: every
// band-b >= 1 edge has one slot in its variable owner's VAR region and one in
// its row owner's ROW region (host_code.cpp xband_tables).
//   C-phase: read L_vc from the ROW slot, write E_cv over it; after each
//            chunk (band, row step) ship its segments (one per (variable
//            owner, V chunk)) to the owners' VAR regions.
//   V-phase: read E_cv from the VAR slots, write L_vc over them; after each
//            row chunk h, ship its segments (one per (row owner, C chunk)) to
//            the owners' ROW regions.
// Shipping = cp.async.bulk shared::cta -> shared::cluster, complete_tx on the
// receiver's region barrier, issued by a producer warp as soon as the compute
// warps have arrived on the chunk's barrier: early chunks travel while later
// chunks compute, and no CTA-wide barrier sits inside the iteration loop.
// Random remote 4-byte DSMEM accesses run at ~0.4/clk/SM and bulk segment
// exchange at ~12 B/clk/SM (profiles/r01_microbench*.txt), hence the segments
// and the overlap.  The two slot tables of the CTA are copied to shared memory
// once per launch.
//
// Why no region is overwritten while still needed: a CTA writes its VAR
// region only after its VAR barrier completed (every row owner shipped every
// band, i.e. finished its C-phase), and its outgoing copies from that region
// (previous V-phase) were complete before any row owner could start the
// C-phase whose results just arrived; the ROW region symmetrically.  A CTA
// ships into a peer's region only after having received that peer's whole
// previous exchange, which the peer issues after its last read of the region.
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

template <int D>
__device__ __forceinline__ void ld_u32_row(const uint32_t *p, uint32_t (&o)[D]) {
    // D 32-bit slots from shared memory; p is 16-byte aligned for D % 4 == 0, 8-byte for D even
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int w = 0; w < D / 4; ++w) {
            const uint4 x = reinterpret_cast<const uint4 *>(p)[w];
            o[4 * w] = x.x; o[4 * w + 1] = x.y; o[4 * w + 2] = x.z; o[4 * w + 3] = x.w;
        }
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int w = 0; w < D / 2; ++w) {
            const uint2 x = reinterpret_cast<const uint2 *>(p)[w];
            o[2 * w] = x.x; o[2 * w + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) o[j] = p[j];
    }
}

struct XArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    int32_t adapt_votes;    // xband2: psi votes only after a hit (or every 4th iteration)
    float *rws;             // xband2: R' = clamp(R) log2(e) per (cluster, slot, variable), written at V-phase 0
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
};

__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Shared memory: VAR region | ROW region (cap floats each) | var slot table
// u16 [nq][NB] | row slot table u16 [NB][mbq][WR] | barriers | flags[C].
// Barriers: var_bar, row_bar (incoming E / L exchange, complete_tx),
// vchunk[H], cchunk[NB H] (compute warps finished a chunk).
// Warps: TW / 32 compute warps, then one producer warp that ships each chunk
// as soon as every compute warp arrived on its chunk barrier -- no CTA-wide
// barrier inside the iteration loop.
// MAXT: launch bound (768 lets a 736-thread C5 block keep 85 registers).
// NFIX: 0, or the code length compiled in (C5's n = 64800, the DVB-S2 normal
// frame): sizes and loop bounds become immediates.
template <int WR, int WC, int H, int C, int MAXT, int NFIX = 0>
__global__ void __launch_bounds__(MAXT, 1) xband_kernel(const XArgs a) {
    extern __shared__ __align__(128) char smem[];
    constexpr int NB = WC - 1;
    const DeviceCode &code = a.code;
    const int n = NFIX ? NFIX : code.n, mb = NFIX ? NFIX / WR : code.mb, mbq = mb / C, nq = n / C;
    const int TW = NFIX ? xband_threads(NFIX / WR / C) : int(blockDim.x) - 32, tt = threadIdx.x, lane = tt & 31;
    const bool producer = tt >= TW;
    const uint32_t cap_b = uint32_t(code.xcap) * 4u;
    const uint32_t q = cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    char *varr = smem;
    char *rowr = smem + cap_b;
    uint16_t *vtab = reinterpret_cast<uint16_t *>(smem + 2 * cap_b);
    uint16_t *rtab = vtab + size_t(nq) * NB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + ((2 * cap_b + 4u * uint32_t(NB * nq) + 15u) & ~15u));
    constexpr int NC = NB * H;      // C-phase chunks: (band, row step)
    int *flags = reinterpret_cast<int *>(bars + 2 + H + NC);
    const uint32_t var_s = saddr(varr), row_s = saddr(rowr), vbar = saddr(bars), rbar = vbar + 8;
    const uint32_t vchunk = vbar + 16, cchunk = vchunk + 8 * H;
    const int nkey = C * C * H * NC;
    const int32_t *varOff = code.xband_seg, *rowOff = code.xband_seg + nkey, *sbytes = code.xband_seg + 2 * nkey;
    auto key = [](int s, int d, int h, int c) { return ((s * C + d) * H + h) * NC + c; };

    // slot tables of CTA q -> shared memory (once)
    {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(code.xband_sidx + size_t(q) * nq * NB);
        uint32_t *dst = reinterpret_cast<uint32_t *>(vtab);
        for (int i = tt; i < nq * NB / 2; i += blockDim.x) dst[i] = __ldg(src + i);
        for (int b = 0; b < NB; ++b) {
            const uint32_t *rs = reinterpret_cast<const uint32_t *>(code.xband_ridx + size_t(b) * n + size_t(q) * mbq * WR);
            uint32_t *rd = reinterpret_cast<uint32_t *>(rtab + size_t(b) * mbq * WR);
            for (int i = tt; i < mbq * WR / 2; i += blockDim.x) rd[i] = __ldg(rs + i);
        }
    }
    // bytes arriving in an L exchange (ROW region) and an E exchange (VAR region)
    uint32_t rx_l = 0, rx_e = 0;
    for (int s = 0; s < C; ++s)
        for (int h = 0; h < H; ++h)
            for (int c = 0; c < NC; ++c) {
                rx_l += uint32_t(__ldg(sbytes + key(s, q, h, c)));
                rx_e += uint32_t(__ldg(sbytes + key(q, s, h, c)));
            }
    if (tt == 0) {
        mbar_init(vbar, 1);
        mbar_init(rbar, 1);
        for (int i = 0; i < H + NC; ++i) mbar_init(vchunk + 8 * i, uint32_t(TW / 32));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_arm(vbar, rx_e);
        mbar_arm(rbar, rx_l);
    }
    cluster_sync_all();

    // compute warps: one arrival per warp on a chunk barrier, after making the
    // lanes' shared-memory writes visible to the async (bulk-copy) proxy
    auto chunk_done = [&](uint32_t bar) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar);
    };
    uint32_t nv = 0, nc = 0;    // V / C phases shipped (producer: chunk barrier phases)
    // producer: ship V chunk h (segments (q, d, h, c): VAR region -> ROW region of d)
    auto ship_l = [&](int h) {
        mbar_wait(vchunk + 8 * h, nv & 1u);
        for (int i = lane; i < C * NC; i += 32) {
            const int d = i / NC, c = i - d * NC;
            const int k = key(int(q), d, h, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(row_s + uint32_t(__ldg(rowOff + k)), uint32_t(d)), var_s + uint32_t(__ldg(varOff + k)),
                         nbytes, mapa_u32(rbar, uint32_t(d)));
        }
    };
    // producer: ship C chunk c (segments (s, q, h, c): ROW region -> VAR region of s)
    auto ship_e = [&](int c) {
        mbar_wait(cchunk + 8 * c, nc & 1u);
        if (lane < C * H) {
            const int s = lane / H, h = lane - s * H;
            const int k = key(s, int(q), h, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(var_s + uint32_t(__ldg(varOff + k)), uint32_t(s)), row_s + uint32_t(__ldg(rowOff + k)),
                         nbytes, mapa_u32(vbar, uint32_t(s)));
        }
    };
    uint32_t nl = 0, ne = 0;    // compute warps: L / E exchanges received
    auto wait_row = [&]() {
        mbar_wait(rbar, nl & 1u);
        if (tt == 0) mbar_arm(rbar, rx_l);
        ++nl;
    };
    auto wait_var = [&]() {
        mbar_wait(vbar, ne & 1u);
        if (tt == 0) mbar_arm(vbar, rx_e);
        ++ne;
    };

    for (int64_t f = cid; f < a.frames; f += ncl) {
        const float *llr = a.llr + f * int64_t(n);
        float e0[H][WR];
        uint32_t synd = 0;
        if (producer) {
            // the producer's view of the frame: V0, then (C, V) x max_iter
#pragma unroll
            for (int h = 0; h < H; ++h) ship_l(h);
            ++nv;
            for (int t = 1; t <= a.max_iter; ++t) {
#pragma unroll
                for (int c = 0; c < NC; ++c) ship_e(c);
                ++nc;
#pragma unroll
                for (int h = 0; h < H; ++h) ship_l(h);
                ++nv;
            }
        } else {
            // ---- V-phase 0 (a1/a2): L = R, E = 0; L_vc = R; band-0 check of t = 1
            //      (after both chunks are handed to the producer, as below)
            float lv[H][WR];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const int r = tt + h * TW;
                if (r < mbq) {
                    const int v0 = (int(q) * mbq + r) * WR;
                    lds_row<WR>(reinterpret_cast<const char *>(llr), uint32_t(v0) * 4u, lv[h]);   // global, 8B-aligned rows
#pragma unroll
                    for (int j = 0; j < WR; ++j) lv[h][j] = fminf(fmaxf(lv[h][j], -30.0f), 30.0f) * kL2E;
                    const uint16_t *vt = vtab + size_t(r) * WR * NB;
#pragma unroll
                    for (int j = 0; j < WR; ++j)
#pragma unroll
                        for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr + vt[j * NB + b]) = lv[h][j];
                }
                chunk_done(vchunk + 8 * h);
            }
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (tt + h * TW < mbq) check_row<WR, true>(lv[h], e0[h]);
            for (int t = 1; t <= a.max_iter; ++t) {
                // ---- C-phase t (a3): rows of bands >= 1 owned by q, band by band
                wait_row();
#pragma unroll
                for (int b = 0; b < NB; ++b) {
#pragma unroll
                    for (int k = 0; k < H; ++k) {
                        const int lr = tt + k * TW;
                        if (lr < mbq) {
                            const uint16_t *rt = rtab + (size_t(b) * mbq + lr) * WR;
                            uint32_t sl[WR];
#pragma unroll
                            for (int j = 0; j < WR; ++j) sl[j] = rt[j];
                            float x[WR], e[WR];
#pragma unroll
                            for (int j = 0; j < WR; ++j) x[j] = *reinterpret_cast<const float *>(rowr + sl[j]);
                            check_row<WR, true>(x, e);
#pragma unroll
                            for (int j = 0; j < WR; ++j) *reinterpret_cast<float *>(rowr + sl[j]) = e[j];
                        }
                        chunk_done(cchunk + 8 * (b * H + k));
                    }
                }
                // ---- V-phase t (a4/a5): L = R + sum E; L_vc over the E slots (L itself at t = T)
                const bool last = t == a.max_iter;
                // R does not depend on the exchange: its (L2) loads are issued
                // before waiting for the E segments
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const int r = tt + h * TW;
                    if (r < mbq)
                        lds_row<WR>(reinterpret_cast<const char *>(llr), uint32_t((int(q) * mbq + r) * WR) * 4u, lv[h]);
                }
                wait_var();
                // Each chunk's L_vc go to the producer first; the band-0 checks
                // (thread-local, x = L - E0) run afterwards, overlapping the transfer.
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const int r = tt + h * TW;
                    if (r < mbq) {
                        const uint16_t *vt = vtab + size_t(r) * WR * NB;
                        uint32_t sl[WR * NB];
#pragma unroll
                        for (int i = 0; i < WR * NB; ++i) sl[i] = vt[i];
                        float eb[WR * NB];
#pragma unroll
                        for (int j = 0; j < WR; ++j) {
                            lv[h][j] = fminf(fmaxf(lv[h][j], -30.0f), 30.0f) * kL2E + e0[h][j];
#pragma unroll
                            for (int b = 0; b < NB; ++b) {
                                eb[j * NB + b] = *reinterpret_cast<const float *>(varr + sl[j * NB + b]);
                                lv[h][j] += eb[j * NB + b];
                            }
                        }
                        if (last) {
                            uint32_t rp = 0;      // band-0 row syndrome bit (Eq. 1)
#pragma unroll
                            for (int j = 0; j < WR; ++j) {
                                rp ^= (lv[h][j] >= 0.0f) ? 1u : 0u;
#pragma unroll
                                for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr + sl[j * NB + b]) = lv[h][j];
                            }
                            synd |= rp;
                        } else {
#pragma unroll
                            for (int j = 0; j < WR; ++j) {
#pragma unroll
                                for (int b = 0; b < NB; ++b)
                                    *reinterpret_cast<float *>(varr + sl[j * NB + b]) = lv[h][j] - eb[j * NB + b];
                                lv[h][j] -= e0[h][j];
                            }
                        }
                    }
                    chunk_done(vchunk + 8 * h);
                }
                if (!last) {
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        if (tt + h * TW < mbq) check_row<WR, true>(lv[h], e0[h]);
                }
            }
            // ---- a7: syndrome of z = [L >= 0]: ROW slots now hold L (bands >= 1)
            wait_row();
            for (int r = tt; r < NB * mbq; r += TW) {
                const uint16_t *rt = rtab + size_t(r) * WR;
                uint32_t rp = 0;
#pragma unroll
                for (int j = 0; j < WR; ++j) rp ^= (*reinterpret_cast<const float *>(rowr + rt[j]) >= 0.0f) ? 1u : 0u;
                synd |= rp;
            }
        }
        const int any = __syncthreads_or(synd != 0);
        if (tt == 0) {
            int *f0 = cg::this_cluster().map_shared_rank(flags, 0);
            f0[q] = any;
        }
        cluster_sync_all();
        // ---- a6/a8: bits (words starting in q's variable range), posteriors, flags.
        // L_v sits in the VAR slot of (v, band 1) of its owner.
        if (!producer) {
            const int nw = code.nw;
            const int w_lo = (int(q) * nq + 31) / 32;
            const int w_hi = (int(q) == C - 1) ? nw : ((int(q) + 1) * nq + 31) / 32;
            const int qn = (int(q) + 1 < C) ? int(q) + 1 : int(q);
            const char *vnext = cg::this_cluster().map_shared_rank(varr, qn);
            const uint16_t *tnext = cg::this_cluster().map_shared_rank(vtab, qn);
            uint32_t *bits = a.bits + f * int64_t(nw);
            // TW is a multiple of 32: each warp covers whole words
            for (int base = w_lo * 32; base < w_hi * 32; base += TW) {
                const int v = base + tt;
                if (v >= w_hi * 32) break;          // warp-uniform
                bool z = false;
                if (v < n) {
                    const int i = v - int(q) * nq;
                    const float lv = i < nq ? *reinterpret_cast<const float *>(varr + vtab[size_t(i) * NB])
                                            : *reinterpret_cast<const float *>(vnext + tnext[size_t(i - nq) * NB]);
                    z = lv >= 0.0f;
                }
                const uint32_t word = __ballot_sync(0xffffffffu, z);
                if (lane == 0) bits[v >> 5] = word;
            }
            if (a.posterior) {
                float *dst = a.posterior + f * int64_t(n) + int64_t(q) * nq;
                for (int i = tt; i < nq; i += TW) dst[i] = *reinterpret_cast<const float *>(varr + vtab[size_t(i) * NB]) * kLn2;
            }
            if (q == 0 && tt == 0) {
                int ok = 1;
                for (int i = 0; i < C; ++i) ok &= (flags[i] == 0);
                a.syn_ok[f] = uint8_t(ok);
                a.iters[f] = a.max_iter;
            }
        }
        cluster_sync_all();     // VAR regions / flags are reused by the next frame
    }
}

// Tensor Memory helpers (32x32b shapes: each lane of the warp its own TMEM lane)
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void tm_ld2(uint32_t a, uint32_t &v0, uint32_t &v1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v0), "=r"(v1) : "r"(a) : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_st4(uint32_t a, uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v0), "r"(v1), "r"(v2),
                 "r"(v3)
                 : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t a, uint32_t v0, uint32_t v1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(v0), "r"(v1) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 6 words (WR = 6): x4 + x2
__device__ __forceinline__ void tm_ld6(uint32_t a, uint32_t (&v)[6]) {
    uint32_t t[4];
    tm_ld4(a, t);
    tm_ld2(a + 4, v[4], v[5]);
    tm_wait_ld();
    v[0] = t[0]; v[1] = t[1]; v[2] = t[2]; v[3] = t[3];
}
__device__ __forceinline__ void tm_st6(uint32_t a, const uint32_t (&v)[6]) {
    tm_st4(a, v[0], v[1], v[2], v[3]);
    tm_st2(a + 4, v[4], v[5]);
}

// ---------------------------------------------------------------------------
// Two frames in flight per cluster (slots 0 and 1; H = 1, e.g. 16-CTA
// clusters on C5).  Each slot has its own VAR / ROW regions and barriers; the
// slot tables are shared.  The compute warps alternate the slots' phases --
// C(0), C(1), V(0), V(1) -- so one slot's segment exchange travels while the
// other slot computes, hiding the exchange's fixed latency; the producer warp
// ships the chunks in the same order.  Per slot the protocol and the safety
// argument are those of xband_kernel.  Frames 2p and 2p+1 of cluster pair
// index p run together; a lone last frame runs in slot 0 only.
template <int WR, int WC, int C, int MAXT, int NFIX = 0>
__global__ void __launch_bounds__(MAXT, 1) xband2_kernel(const XArgs a) {
    extern __shared__ __align__(128) char smem[];
    constexpr int NB = WC - 1, H = 1, NC = NB;
    const DeviceCode &code = a.code;
    const int n = NFIX ? NFIX : code.n, mb = NFIX ? NFIX / WR : code.mb, mbq = mb / C, nq = n / C;
    const int TW = NFIX ? xband_threads(NFIX / WR / C) : int(blockDim.x) - 32, tt = threadIdx.x, lane = tt & 31;
    const bool producer = tt >= TW;
    const uint32_t cap_b = uint32_t(code.xcap) * 4u;
    const uint32_t q = cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    // every CTA of this grid is resident (one wave of clusters): let a
    // dependent launch (the global-exchange tail on the SMs 16-CTA clusters
    // leave idle, xcluster_launch) start now instead of after this grid
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    char *varr[2] = {smem, smem + 2 * cap_b};
    char *rowr[2] = {smem + cap_b, smem + 3 * cap_b};
    // slot tables widened to 32-bit byte offsets in shared memory (vector
    // loads, no unpacking in the phases)
    uint32_t *vtab = reinterpret_cast<uint32_t *>(smem + 4 * cap_b);
    uint32_t *rtab = vtab + size_t(nq) * NB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + ((4 * cap_b + 8u * uint32_t(NB * nq) + 15u) & ~15u));
    constexpr int NBAR = 2 + H + NC;                 // per slot: var, row, vchunk, cchunk[NC]
    int *flags = reinterpret_cast<int *>(bars + 2 * NBAR);   // [2][C]
    const uint32_t bar0 = saddr(bars);
    auto vbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR); };
    auto rbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 1); };
    auto vchunk = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 2); };
    auto cchunk = [&](int sl, int c) { return bar0 + 8u * uint32_t(sl * NBAR + 3 + c); };
    const int nkey = C * C * H * NC;
    const int32_t *varOff = code.xband_seg, *rowOff = code.xband_seg + nkey, *sbytes = code.xband_seg + 2 * nkey;
    auto key = [](int s, int d, int h, int c) { return ((s * C + d) * H + h) * NC + c; };
    // R' (clamped, log2-scaled R) of the thread's band-0 row, per slot, in
    // Tensor Memory (otherwise idle here): compute warp w owns lanes
    // 32 (w % 4) .. + 31, columns 16 (w / 4) + 6 sl .. + 5; written at
    // V-phase 0, read by every V-phase (it was an L2-resident slot)
    __shared__ uint32_t s_tmem;
    {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(code.xband_sidx + size_t(q) * nq * NB);
        for (int i = tt; i < nq * NB / 2; i += blockDim.x) {
            const uint32_t x = __ldg(src + i);
            reinterpret_cast<uint2 *>(vtab)[i] = make_uint2(x & 0xffffu, x >> 16);
        }
        for (int b = 0; b < NB; ++b) {
            const uint32_t *rs = reinterpret_cast<const uint32_t *>(code.xband_ridx + size_t(b) * n + size_t(q) * mbq * WR);
            uint2 *rd = reinterpret_cast<uint2 *>(rtab + size_t(b) * mbq * WR);
            for (int i = tt; i < mbq * WR / 2; i += blockDim.x) {
                const uint32_t x = __ldg(rs + i);
                rd[i] = make_uint2(x & 0xffffu, x >> 16);
            }
        }
    }
    const uint32_t warp = uint32_t(tt) >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm_r = s_tmem + ((32u * (warp & 3u)) << 16) + 16u * (warp >> 2);
    uint32_t rx_l = 0, rx_e = 0;
    for (int s = 0; s < C; ++s)
        for (int c = 0; c < NC; ++c) {
            rx_l += uint32_t(__ldg(sbytes + key(s, q, 0, c)));
            rx_e += uint32_t(__ldg(sbytes + key(q, s, 0, c)));
        }
    if (tt == 0) {
        for (int sl = 0; sl < 2; ++sl) {
            mbar_init(vbar(sl), 1);
            mbar_init(rbar(sl), 1);
            mbar_init(vchunk(sl), uint32_t(TW / 32));
            for (int c = 0; c < NC; ++c) mbar_init(cchunk(sl, c), uint32_t(TW / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int sl = 0; sl < 2; ++sl) {
            mbar_arm(vbar(sl), rx_e);
            mbar_arm(rbar(sl), rx_l);
        }
    }
    cluster_sync_all();

    auto chunk_done = [&](uint32_t bar) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar);
    };
    uint32_t nv[2] = {0, 0}, nc[2] = {0, 0};        // producer: chunk barrier phases per slot
    uint32_t nl[2] = {0, 0}, ne[2] = {0, 0};        // compute: exchanges received per slot
    auto ship_l = [&](int sl) {
        mbar_wait(vchunk(sl), nv[sl] & 1u);
        const uint32_t vs = saddr(varr[sl]), rs = saddr(rowr[sl]);
        for (int i = lane; i < C * NC; i += 32) {
            const int d = i / NC, c = i - d * NC;
            const int k = key(int(q), d, 0, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(rs + uint32_t(__ldg(rowOff + k)), uint32_t(d)), vs + uint32_t(__ldg(varOff + k)), nbytes,
                         mapa_u32(rbar(sl), uint32_t(d)));
        }
        ++nv[sl];
    };
    auto ship_e = [&](int sl, int c) {
        mbar_wait(cchunk(sl, c), nc[sl] & 1u);
        const uint32_t vs = saddr(varr[sl]), rs = saddr(rowr[sl]);
        if (lane < C) {
            const int s = lane;
            const int k = key(s, int(q), 0, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(vs + uint32_t(__ldg(varOff + k)), uint32_t(s)), rs + uint32_t(__ldg(rowOff + k)), nbytes,
                         mapa_u32(vbar(sl), uint32_t(s)));
        }
        if (c == NC - 1) ++nc[sl];
    };
    auto wait_row = [&](int sl) {
        mbar_wait(rbar(sl), nl[sl] & 1u);
        if (tt == 0) mbar_arm(rbar(sl), rx_l);
        ++nl[sl];
    };
    auto wait_var = [&](int sl) {
        mbar_wait(vbar(sl), ne[sl] & 1u);
        if (tt == 0) mbar_arm(vbar(sl), rx_e);
        ++ne[sl];
    };

    const int r = tt;                 // H = 1: this thread's band-0 row (if r < mbq)
    const bool own = !producer && r < mbq;
    const int64_t npairs = (a.frames + 1) / 2;
    for (int64_t pi = cid; pi < npairs; pi += ncl) {
        int64_t fs[2] = {2 * pi, 2 * pi + 1};
        const int ns = fs[1] < a.frames ? 2 : 1;    // cluster-uniform
        float e0[2][WR];
        uint32_t synd[2] = {0, 0};
        // adaptive psi votes (warp-uniform): vote in iteration t only if a
        // vote hit in iteration t - 1 or t = 1 mod 4
        bool vote_on[2] = {true, true}, hit[2] = {false, false};
        if (producer) {
            for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            for (int t = 1; t <= a.max_iter; ++t) {
                for (int sl = 0; sl < ns; ++sl)
#pragma unroll
                    for (int c = 0; c < NC; ++c) ship_e(sl, c);
                for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            }
        } else {
            // ---- V-phase 0 of both slots: L = R, E = 0; band-0 check of t = 1
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
                if (sl < ns) {
                    float lv[WR] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                    if (own) {
                        const int v0 = (int(q) * mbq + r) * WR;
                        lds_row<WR>(reinterpret_cast<const char *>(a.llr + fs[sl] * int64_t(n)), uint32_t(v0) * 4u, lv);
#pragma unroll
                        for (int j = 0; j < WR; ++j) lv[j] = fminf(fmaxf(lv[j], -30.0f), 30.0f) * kL2E;
                        const uint32_t *vt = vtab + size_t(r) * WR * NB;
#pragma unroll
                        for (int j = 0; j < WR; ++j)
#pragma unroll
                            for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr[sl] + vt[j * NB + b]) = lv[j];
                    }
                    // R' of the slot's frame, reread by every V-phase (TMEM; all lanes)
                    {
                        const uint32_t u[6] = {__float_as_uint(lv[0]), __float_as_uint(lv[1]), __float_as_uint(lv[2]),
                                               __float_as_uint(lv[3]), __float_as_uint(lv[4]), __float_as_uint(lv[5])};
                        tm_st6(tm_r + 6u * uint32_t(sl), u);
                    }
                    chunk_done(vchunk(sl));
                    if (own) check_row<WR, true>(lv, e0[sl]);
                }
            }
            tm_wait_st();
            for (int t = 1; t <= a.max_iter; ++t) {
                // ---- C-phases (a3)
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    if (sl < ns) {
                        if (a.adapt_votes) {
                            vote_on[sl] = hit[sl] || (t & 3) == 1;
                            hit[sl] = false;
                        }
                        wait_row(sl);
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            if (r < mbq) {
                                uint32_t s_[WR];
                                ld_u32_row<WR>(rtab + (size_t(b) * mbq + r) * WR, s_);
                                float x[WR], e[WR];
#pragma unroll
                                for (int j = 0; j < WR; ++j) x[j] = *reinterpret_cast<const float *>(rowr[sl] + s_[j]);
                                hit[sl] |= check_row_gated<WR>(x, e, vote_on[sl]);
#pragma unroll
                                for (int j = 0; j < WR; ++j) *reinterpret_cast<float *>(rowr[sl] + s_[j]) = e[j];
                            }
                            chunk_done(cchunk(sl, b));
                        }
                    }
                }
                // ---- V-phases (a4/a5)
                const bool last = t == a.max_iter;
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    if (sl < ns) {
                        float lv[WR];
                        {
                            uint32_t u[6];
                            tm_ld6(tm_r + 6u * uint32_t(sl), u);
#pragma unroll
                            for (int j = 0; j < WR; ++j) lv[j] = __uint_as_float(u[j]);
                        }
                        wait_var(sl);
                        if (own) {
                            uint32_t s_[WR * NB];
                            ld_u32_row<WR * NB>(vtab + size_t(r) * WR * NB, s_);
                            float eb[WR * NB];
#pragma unroll
                            for (int j = 0; j < WR; ++j) {
                                lv[j] += e0[sl][j];
#pragma unroll
                                for (int b = 0; b < NB; ++b) {
                                    eb[j * NB + b] = *reinterpret_cast<const float *>(varr[sl] + s_[j * NB + b]);
                                    lv[j] += eb[j * NB + b];
                                }
                            }
                            if (last) {
                                uint32_t rp = 0;
#pragma unroll
                                for (int j = 0; j < WR; ++j) {
                                    rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
#pragma unroll
                                    for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr[sl] + s_[j * NB + b]) = lv[j];
                                }
                                synd[sl] |= rp;
                            } else {
#pragma unroll
                                for (int j = 0; j < WR; ++j) {
#pragma unroll
                                    for (int b = 0; b < NB; ++b)
                                        *reinterpret_cast<float *>(varr[sl] + s_[j * NB + b]) = lv[j] - eb[j * NB + b];
                                    lv[j] -= e0[sl][j];
                                }
                            }
                        }
                        chunk_done(vchunk(sl));
                        if (own && !last) hit[sl] |= check_row_gated<WR>(lv, e0[sl], vote_on[sl]);
                    }
                }
            }
            // ---- a7: syndrome (ROW slots hold L of bands >= 1)
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
                if (sl < ns) {
                    wait_row(sl);
                    for (int rr = tt; rr < NB * mbq; rr += TW) {
                        const uint32_t *rt = rtab + size_t(rr) * WR;
                        uint32_t rp = 0;
#pragma unroll
                        for (int j = 0; j < WR; ++j) rp ^= (*reinterpret_cast<const float *>(rowr[sl] + rt[j]) >= 0.0f) ? 1u : 0u;
                        synd[sl] |= rp;
                    }
                }
            }
        }
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
            const int any = __syncthreads_or(synd[sl] != 0);
            if (tt == 0) {
                int *f0 = cg::this_cluster().map_shared_rank(flags, 0);
                f0[sl * C + int(q)] = any;
            }
        }
        cluster_sync_all();
        if (!producer) {
            const int nw = code.nw;
            const int w_lo = (int(q) * nq + 31) / 32;
            const int w_hi = (int(q) == C - 1) ? nw : ((int(q) + 1) * nq + 31) / 32;
            const int qn = (int(q) + 1 < C) ? int(q) + 1 : int(q);
            const uint32_t *tnext = cg::this_cluster().map_shared_rank(vtab, qn);
            for (int sl = 0; sl < ns; ++sl) {
                const char *vnext = cg::this_cluster().map_shared_rank(varr[sl], qn);
                uint32_t *bits = a.bits + fs[sl] * int64_t(nw);
                for (int base = w_lo * 32; base < w_hi * 32; base += TW) {
                    const int v = base + tt;
                    if (v >= w_hi * 32) break;
                    bool z = false;
                    if (v < n) {
                        const int i = v - int(q) * nq;
                        const float lv = i < nq ? *reinterpret_cast<const float *>(varr[sl] + vtab[size_t(i) * NB])
                                                : *reinterpret_cast<const float *>(vnext + tnext[size_t(i - nq) * NB]);
                        z = lv >= 0.0f;
                    }
                    const uint32_t word = __ballot_sync(0xffffffffu, z);
                    if (lane == 0) bits[v >> 5] = word;
                }
                if (a.posterior) {
                    float *dst = a.posterior + fs[sl] * int64_t(n) + int64_t(q) * nq;
                    for (int i = tt; i < nq; i += TW)
                        dst[i] = *reinterpret_cast<const float *>(varr[sl] + vtab[size_t(i) * NB]) * kLn2;
                }
                if (q == 0 && tt == 0) {
                    int ok = 1;
                    for (int i = 0; i < C; ++i) ok &= (flags[sl * C + i] == 0);
                    a.syn_ok[fs[sl]] = uint8_t(ok);
                    a.iters[fs[sl]] = a.max_iter;
                }
            }
        }
        cluster_sync_all();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(s_tmem) : "memory");
}

// ---------------------------------------------------------------------------
// NS frames in flight per 16-CTA cluster with the per-thread constant state in
// Tensor Memory (xbandt_kernel; C5 batches).  Same ownership, protocol,
// arithmetic and adaptive votes as xband2_kernel; what moves:
//   * the CTA's slot tables leave shared memory: compute thread r keeps its
//     own rows -- the VAR slots of its band-0 row's WR x NB edges and the ROW
//     slots of its band-b rows -- in TMEM columns of its warp (tcgen05.ld per
//     phase, 12-cycle latency), which frees 32 KB of shared memory for a
//     third slot (6 regions of ~33 KB);
//   * the band-0 E of every slot also lives in TMEM (loaded for the slot's
//     variable phase, stored after its band-0 check) instead of NS x WR
//     registers, which spilled when a third slot was held in registers.
// A third frame in flight gives every segment exchange two other slots'
// phases of cover instead of one (the exchange is latency-, not
// bandwidth-bound: DESIGN.md xband2_kernel).
// TMEM layout (512 columns, one CTA per SM): compute warp w owns lanes
// 32 (w % 4) .. + 31 and columns 64 (w / 4) .. + 63: [0, 12) VAR slots of the
// band-0 row's edges (j NB + b), [12, 12 + WR NB) ROW slots of the band-b rows
// (b WR + j), [24, 24 + WR NS) band-0 E of the slots.
// Hard decisions go through a CTA byte array in shared memory (the words
// that straddle two CTAs read the neighbour's through DSMEM).
template <int WR, int WC, int C, int MAXT, int NFIX = 0, int NS = 3>
__global__ void __launch_bounds__(MAXT, 1) xbandt_kernel(const XArgs a) {
    static_assert(WR == 6 && WC == 3, "xbandt: the (3,6) layout of its TMEM columns");
    extern __shared__ __align__(128) char smem[];
    constexpr int NB = WC - 1, H = 1, NC = NB;
    const DeviceCode &code = a.code;
    const int n = NFIX ? NFIX : code.n, mb = NFIX ? NFIX / WR : code.mb, mbq = mb / C, nq = n / C;
    const int TW = NFIX ? xband_threads(NFIX / WR / C) : int(blockDim.x) - 32, tt = threadIdx.x, lane = tt & 31;
    const bool producer = tt >= TW;
    const uint32_t cap_b = uint32_t(code.xcap) * 4u;
    const uint32_t q = cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = ncluster_x();
    // slot regions by offset (no per-slot pointer registers)
    auto varr = [&](int sl) { return smem + 2u * uint32_t(sl) * cap_b; };
    auto rowr = [&](int sl) { return smem + (2u * uint32_t(sl) + 1u) * cap_b; };
    uint8_t *zscr = reinterpret_cast<uint8_t *>(smem + 2 * NS * cap_b);        // nq hard-decision bytes
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + ((2 * NS * cap_b + uint32_t(nq) + 15u) & ~15u));
    constexpr int NBAR = 2 + H + NC;
    int *flags = reinterpret_cast<int *>(bars + NS * NBAR);   // [NS][C]
    __shared__ uint32_t s_tmem;
    const uint32_t bar0 = saddr(bars);
    auto vbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR); };
    auto rbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 1); };
    auto vchunk = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 2); };
    auto cchunk = [&](int sl, int c) { return bar0 + 8u * uint32_t(sl * NBAR + 3 + c); };
    const int nkey = C * C * H * NC;
    const int32_t *varOff = code.xband_seg, *rowOff = code.xband_seg + nkey, *sbytes = code.xband_seg + 2 * nkey;
    auto key = [](int s, int d, int h, int c) { return ((s * C + d) * H + h) * NC + c; };
    auto rslot = [&](int sl) { return a.rws + (size_t(cid) * NS + size_t(sl)) * size_t(n); };
    const int r = tt;                 // H = 1: this thread's band-0 row (if r < mbq)
    const bool own = !producer && r < mbq;

    // ---- TMEM: allocate, then every compute thread parks its table rows
    const uint32_t warp = uint32_t(tt) >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&s_tmem)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = s_tmem + ((32u * (warp & 3u)) << 16) + 64u * (warp >> 2);
    const uint32_t tm_vt = tm, tm_rt = tm + 12, tm_e0 = tm + 24;
    if (!producer) {
        uint32_t v[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, w[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (r < mbq) {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(code.xband_sidx + (size_t(q) * nq + size_t(r) * WR) * NB);
#pragma unroll
            for (int i = 0; i < WR * NB / 2; ++i) {
                const uint32_t x = __ldg(src + i);
                v[2 * i] = x & 0xffffu;
                v[2 * i + 1] = x >> 16;
            }
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const uint32_t *rs =
                    reinterpret_cast<const uint32_t *>(code.xband_ridx + size_t(b) * n + (size_t(q) * mbq + r) * WR);
#pragma unroll
                for (int i = 0; i < WR / 2; ++i) {
                    const uint32_t x = __ldg(rs + i);
                    w[b * WR + 2 * i] = x & 0xffffu;
                    w[b * WR + 2 * i + 1] = x >> 16;
                }
            }
        }
        tm_st4(tm_vt, v[0], v[1], v[2], v[3]);
        tm_st4(tm_vt + 4, v[4], v[5], v[6], v[7]);
        tm_st4(tm_vt + 8, v[8], v[9], v[10], v[11]);
        tm_st4(tm_rt, w[0], w[1], w[2], w[3]);
        tm_st4(tm_rt + 4, w[4], w[5], w[6], w[7]);
        tm_st4(tm_rt + 8, w[8], w[9], w[10], w[11]);
        tm_wait_st();
    }
    uint32_t rx_l = 0, rx_e = 0;
    for (int s = 0; s < C; ++s)
        for (int c = 0; c < NC; ++c) {
            rx_l += uint32_t(__ldg(sbytes + key(s, q, 0, c)));
            rx_e += uint32_t(__ldg(sbytes + key(q, s, 0, c)));
        }
    if (tt == 0) {
        for (int sl = 0; sl < NS; ++sl) {
            mbar_init(vbar(sl), 1);
            mbar_init(rbar(sl), 1);
            mbar_init(vchunk(sl), uint32_t(TW / 32));
            for (int c = 0; c < NC; ++c) mbar_init(cchunk(sl, c), uint32_t(TW / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int sl = 0; sl < NS; ++sl) {
            mbar_arm(vbar(sl), rx_e);
            mbar_arm(rbar(sl), rx_l);
        }
    }
    cluster_sync_all();

    auto chunk_done = [&](uint32_t bar) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar);
    };
    // barrier phase parities, one bit per slot
    uint32_t nv = 0, nc = 0, nl = 0, ne = 0;
    auto ship_l = [&](int sl) {
        mbar_wait(vchunk(sl), (nv >> sl) & 1u);
        const uint32_t vs = saddr(varr(sl)), rs = saddr(rowr(sl));
        for (int i = lane; i < C * NC; i += 32) {
            const int d = i / NC, c = i - d * NC;
            const int k = key(int(q), d, 0, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(rs + uint32_t(__ldg(rowOff + k)), uint32_t(d)), vs + uint32_t(__ldg(varOff + k)), nbytes,
                         mapa_u32(rbar(sl), uint32_t(d)));
        }
        nv ^= 1u << sl;
    };
    auto ship_e = [&](int sl, int c) {
        mbar_wait(cchunk(sl, c), (nc >> sl) & 1u);
        const uint32_t vs = saddr(varr(sl)), rs = saddr(rowr(sl));
        if (lane < C) {
            const int s = lane;
            const int k = key(s, int(q), 0, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes)
                bulk_s2c(mapa_u32(vs + uint32_t(__ldg(varOff + k)), uint32_t(s)), rs + uint32_t(__ldg(rowOff + k)), nbytes,
                         mapa_u32(vbar(sl), uint32_t(s)));
        }
        if (c == NC - 1) nc ^= 1u << sl;
    };
    auto wait_row = [&](int sl) {
        mbar_wait(rbar(sl), (nl >> sl) & 1u);
        if (tt == 0) mbar_arm(rbar(sl), rx_l);
        nl ^= 1u << sl;
    };
    auto wait_var = [&](int sl) {
        mbar_wait(vbar(sl), (ne >> sl) & 1u);
        if (tt == 0) mbar_arm(vbar(sl), rx_e);
        ne ^= 1u << sl;
    };
    auto e0_store = [&](int sl, const float (&e)[WR]) {
        const uint32_t u[6] = {__float_as_uint(e[0]), __float_as_uint(e[1]), __float_as_uint(e[2]),
                               __float_as_uint(e[3]), __float_as_uint(e[4]), __float_as_uint(e[5])};
        tm_st6(tm_e0 + uint32_t(WR * sl), u);
    };

    const int64_t ngroups = (a.frames + NS - 1) / NS;
    for (int64_t pi = cid; pi < ngroups; pi += ncl) {
        auto fs = [&](int sl) { return int64_t(NS) * pi + sl; };
        // per-slot bits: syndrome of the slot's frame, votes on, a vote hit
        uint32_t synd = 0, vote_on = (1u << NS) - 1u, hit = 0;
        const int ns = int(std::min<int64_t>(NS, a.frames - int64_t(NS) * pi));    // cluster-uniform
        if (producer) {
            for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            for (int t = 1; t <= a.max_iter; ++t) {
                for (int sl = 0; sl < ns; ++sl)
#pragma unroll
                    for (int c = 0; c < NC; ++c) ship_e(sl, c);
                for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            }
        } else {
            // ---- V-phase 0 of every slot: L = R, E = 0; band-0 check of t = 1
#pragma unroll
            for (int sl = 0; sl < NS; ++sl) {
                if (sl < ns) {
                    uint32_t vt[12];
                    tm_ld8(tm_vt, *reinterpret_cast<uint32_t(*)[8]>(vt));
                    tm_ld4(tm_vt + 8, *reinterpret_cast<uint32_t(*)[4]>(vt + 8));
                    tm_wait_ld();
                    float lv[WR], e0n[WR];
                    if (own) {
                        const int v0 = (int(q) * mbq + r) * WR;
                        lds_row<WR>(reinterpret_cast<const char *>(a.llr + fs(sl) * int64_t(n)), uint32_t(v0) * 4u, lv);
#pragma unroll
                        for (int j = 0; j < WR; ++j) lv[j] = fminf(fmaxf(lv[j], -30.0f), 30.0f) * kL2E;
                        sts_row<WR>(reinterpret_cast<char *>(rslot(sl)), uint32_t(v0) * 4u, lv);
#pragma unroll
                        for (int j = 0; j < WR; ++j)
#pragma unroll
                            for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr(sl) + vt[j * NB + b]) = lv[j];
                    }
                    chunk_done(vchunk(sl));
                    if (own) check_row<WR, true>(lv, e0n);
                    e0_store(sl, e0n);
                }
            }
            tm_wait_st();
            for (int t = 1; t <= a.max_iter; ++t) {
                // ---- C-phases (a3)
#pragma unroll
                for (int sl = 0; sl < NS; ++sl) {
                    if (sl < ns) {
                        if (a.adapt_votes) {
                            const bool on = ((hit >> sl) & 1u) || (t & 3) == 1;
                            vote_on = (vote_on & ~(1u << sl)) | (uint32_t(on) << sl);
                            hit &= ~(1u << sl);
                        }
                        wait_row(sl);
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            uint32_t s_[WR];
                            tm_ld6(tm_rt + uint32_t(b * WR), s_);
                            if (r < mbq) {
                                float x[WR], e[WR];
#pragma unroll
                                for (int j = 0; j < WR; ++j) x[j] = *reinterpret_cast<const float *>(rowr(sl) + s_[j]);
                                hit |= uint32_t(check_row_gated<WR>(x, e, (vote_on >> sl) & 1u)) << sl;
#pragma unroll
                                for (int j = 0; j < WR; ++j) *reinterpret_cast<float *>(rowr(sl) + s_[j]) = e[j];
                            }
                            chunk_done(cchunk(sl, b));
                        }
                    }
                }
                // ---- V-phases (a4/a5)
                const bool last = t == a.max_iter;
#pragma unroll
                for (int sl = 0; sl < NS; ++sl) {
                    if (sl < ns) {
                        float lv[WR], e0c[WR];
                        if (own)
                            lds_row<WR>(reinterpret_cast<const char *>(rslot(sl)), uint32_t((int(q) * mbq + r) * WR) * 4u, lv);
                        uint32_t s_[WR * NB];
                        {
                            uint32_t eu[6];
                            tm_ld8(tm_vt, *reinterpret_cast<uint32_t(*)[8]>(s_));
                            tm_ld4(tm_vt + 8, *reinterpret_cast<uint32_t(*)[4]>(s_ + 8));
                            tm_ld4(tm_e0 + uint32_t(WR * sl), *reinterpret_cast<uint32_t(*)[4]>(eu));
                            tm_ld2(tm_e0 + uint32_t(WR * sl) + 4, eu[4], eu[5]);
                            tm_wait_ld();
#pragma unroll
                            for (int j = 0; j < WR; ++j) e0c[j] = __uint_as_float(eu[j]);
                        }
                        wait_var(sl);
                        if (own) {
                            float eb[WR * NB];
#pragma unroll
                            for (int j = 0; j < WR; ++j) {
                                lv[j] += e0c[j];
#pragma unroll
                                for (int b = 0; b < NB; ++b) {
                                    eb[j * NB + b] = *reinterpret_cast<const float *>(varr(sl) + s_[j * NB + b]);
                                    lv[j] += eb[j * NB + b];
                                }
                            }
                            if (last) {
                                uint32_t rp = 0;
#pragma unroll
                                for (int j = 0; j < WR; ++j) {
                                    rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
#pragma unroll
                                    for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr(sl) + s_[j * NB + b]) = lv[j];
                                }
                                synd |= (rp & 1u) << sl;
                            } else {
#pragma unroll
                                for (int j = 0; j < WR; ++j) {
#pragma unroll
                                    for (int b = 0; b < NB; ++b)
                                        *reinterpret_cast<float *>(varr(sl) + s_[j * NB + b]) = lv[j] - eb[j * NB + b];
                                    lv[j] -= e0c[j];
                                }
                            }
                        }
                        chunk_done(vchunk(sl));
                        if (!last) {
                            if (own) hit |= uint32_t(check_row_gated<WR>(lv, e0c, (vote_on >> sl) & 1u)) << sl;
                            e0_store(sl, e0c);
                        }
                    }
                }
                tm_wait_st();
            }
            // ---- a7: syndrome of the CTA's rows (ROW slots hold L of bands >= 1)
#pragma unroll
            for (int sl = 0; sl < NS; ++sl) {
                if (sl < ns) {
                    wait_row(sl);
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        uint32_t s_[WR];
                        tm_ld6(tm_rt + uint32_t(b * WR), s_);
                        if (r < mbq) {
                            uint32_t rp = 0;
#pragma unroll
                            for (int j = 0; j < WR; ++j) rp ^= (*reinterpret_cast<const float *>(rowr(sl) + s_[j]) >= 0.0f) ? 1u : 0u;
                            synd |= (rp & 1u) << sl;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int sl = 0; sl < NS; ++sl) {
            const int any = __syncthreads_or(((synd >> sl) & 1u) != 0);
            if (tt == 0) {
                int *f0 = cg::this_cluster().map_shared_rank(flags, 0);
                f0[sl * C + int(q)] = any;
            }
        }
        cluster_sync_all();
        // ---- a6/a8, slot by slot: L_v sits in the VAR slot of (v, band 1);
        // each thread writes its own row's posteriors and hard-decision bytes,
        // then whole words are packed (the word straddling into the next CTA
        // reads its bytes through DSMEM)
        const int nw = code.nw;
        const int w_lo = (int(q) * nq + 31) / 32;
        const int w_hi = (int(q) == C - 1) ? nw : ((int(q) + 1) * nq + 31) / 32;
        const int qn = (int(q) + 1 < C) ? int(q) + 1 : int(q);
        const uint8_t *znext = cg::this_cluster().map_shared_rank(zscr, qn);
        for (int sl = 0; sl < ns; ++sl) {
            if (!producer) {
                uint32_t vt[12];
                tm_ld8(tm_vt, *reinterpret_cast<uint32_t(*)[8]>(vt));
                tm_ld4(tm_vt + 8, *reinterpret_cast<uint32_t(*)[4]>(vt + 8));
                tm_wait_ld();
                if (own) {
#pragma unroll
                    for (int j = 0; j < WR; ++j) {
                        const float lv = *reinterpret_cast<const float *>(varr(sl) + vt[j * NB]);
                        zscr[r * WR + j] = lv >= 0.0f ? 1 : 0;
                        if (a.posterior) a.posterior[fs(sl) * int64_t(n) + int64_t(q) * nq + r * WR + j] = lv * kLn2;
                    }
                }
            }
            cluster_sync_all();             // every CTA's bytes are written
            if (!producer) {
                uint32_t *bits = a.bits + fs(sl) * int64_t(nw);
                for (int base = w_lo * 32; base < w_hi * 32; base += TW) {
                    const int v = base + tt;
                    if (v >= w_hi * 32) break;
                    bool z = false;
                    if (v < n) {
                        const int i = v - int(q) * nq;
                        z = (i < nq ? zscr[i] : znext[i - nq]) != 0;
                    }
                    const uint32_t word = __ballot_sync(0xffffffffu, z);
                    if (lane == 0) bits[v >> 5] = word;
                }
                if (q == 0 && tt == 0) {
                    int ok = 1;
                    for (int i = 0; i < C; ++i) ok &= (flags[sl * C + i] == 0);
                    a.syn_ok[fs(sl)] = uint8_t(ok);
                    a.iters[fs(sl)] = a.max_iter;
                }
            }
            cluster_sync_all();             // the byte arrays are reused by the next slot / frame
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
}

template <int WR, int H, int MAXT>
void *pick_x_c(int C) {
    switch (C) {
        case 2: return reinterpret_cast<void *>(&xband_kernel<WR, 3, H, 2, MAXT>);
        case 4: return reinterpret_cast<void *>(&xband_kernel<WR, 3, H, 4, MAXT>);
        case 8: return reinterpret_cast<void *>(&xband_kernel<WR, 3, H, 8, MAXT>);
        case 16: return reinterpret_cast<void *>(&xband_kernel<WR, 3, H, 16, MAXT>);
    }
    // latency views of frames that fit one SM: any C dividing the band rows
    // (C4: mb = 2700 = 2^2 3^3 5^2, C3: mb = 666 = 2 3^2 37), one row per thread
    if constexpr (H == 1) {
        switch (C) {
            case 3: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 3, MAXT>);
            case 5: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 5, MAXT>);
            case 6: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 6, MAXT>);
            case 9: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 9, MAXT>);
            case 10: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 10, MAXT>);
            case 12: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 12, MAXT>);
            case 15: return reinterpret_cast<void *>(&xband_kernel<WR, 3, 1, 15, MAXT>);
        }
    }
    return nullptr;
}

void *pick_xband_kernel(int wr, int wc, int H, int C, int threads) {
    if (wc != 3 || wr != 6) return nullptr;
    switch (H) {
        case 1: return threads <= 768 ? pick_x_c<6, 1, 768>(C) : pick_x_c<6, 1, 1024>(C);
        case 2: return threads <= 768 ? pick_x_c<6, 2, 768>(C) : pick_x_c<6, 2, 1024>(C);
        case 4: return pick_x_c<6, 4, 1024>(C);
    }
    return nullptr;
}

}  // namespace

bool xcluster_plan(const ldpc_code &c, int64_t frames, bool et, XClusterPlan &p) {
    if (et || !c.gallager || !c.regular_col || !c.dev.xcluster) return false;
    const int C = c.dev.xcluster;
    const int mbq = c.n / c.wr / C;
    const int H = c.dev.xrows;                    // as the bound tables were built
    p.threads = ((mbq + H - 1) / H + 31) / 32 * 32 + 32;     // compute warps + the producer warp
    // two frames in flight per cluster (xband2_kernel) when the view allows it
    // and the batch has at least two frames per co-resident cluster's worth
    // three frames in flight with the per-thread tables and band-0 E in TMEM
    // (xbandt_kernel): 6 regions + the hard-decision bytes in shared memory.
    // Opt-in (LDPC_XTMEM=1): measured 0.321 of the SFU model against 0.360 for
    // xband2_kernel
    if (c.dev.xslots == 2 && H == 1 && frames >= 3 && c.wr == 6 && c.wc == 3 && p.threads <= 768 && C == 16 &&
        !std::getenv("LDPC_XBAND_1SLOT") && std::getenv("LDPC_XTMEM") && std::atoi(std::getenv("LDPC_XTMEM")) == 1) {
        constexpr int NS = 3;
        const size_t nq = size_t(c.n / C);
        const size_t smem3 = 2 * NS * size_t(c.dev.xcap) * 4 + nq + 16 + 16 + size_t(NS) * 8 * (3 + size_t(c.wc - 1)) +
                             size_t(NS) * 4 * size_t(C);
        void *k3 = (c.n == 64800 && !std::getenv("LDPC_NO_NFIX"))
                       ? reinterpret_cast<void *>(&xbandt_kernel<6, 3, 16, 768, 64800, NS>)
                       : reinterpret_cast<void *>(&xbandt_kernel<6, 3, 16, 768, 0, NS>);
        if (smem3 + 1024 <= 227 * 1024 && ensure_smem_attribute(k3, smem3, true)) {
            int ncl = occupancy_clusters(k3, p.threads, smem3, C);
            if (ncl >= 1) {
                p.kernel = k3;
                p.cluster = C;
                p.smem = smem3;
                p.capacity = NS * int64_t(ncl);
                p.slots = NS;
                ncl = int(std::min<int64_t>(ncl, (frames + NS - 1) / NS));
                p.grid = ncl * C;
                p.ws_bytes = size_t(ncl) * NS * size_t(c.n) * 4;     // R' per (cluster, slot)
                return true;
            }
        }
    }
    if (c.dev.xslots == 2 && H == 1 && frames >= 2 && c.wr == 6 && c.wc == 3 && p.threads <= 768 &&
        !std::getenv("LDPC_XBAND_1SLOT")) {
        void *k2 = nullptr;
        if (C == 16) k2 = (c.n == 64800 && !std::getenv("LDPC_NO_NFIX"))
                              ? reinterpret_cast<void *>(&xband2_kernel<6, 3, 16, 768, 64800>)
                              : reinterpret_cast<void *>(&xband2_kernel<6, 3, 16, 768>);
        if (k2) {
            const size_t smem2 = xband2_smem_bytes(c.n, c.wc, c.wr, C, c.dev.xcap);
            if (ensure_smem_attribute(k2, smem2, C > 8)) {
                int ncl = occupancy_clusters(k2, p.threads, smem2, C);
                if (ncl >= 1) {
                    p.kernel = k2;
                    p.cluster = C;
                    p.smem = smem2;
                    p.capacity = 2 * int64_t(ncl);
                    p.slots = 2;
                    ncl = int(std::min<int64_t>(ncl, (frames + 1) / 2));
                    p.grid = ncl * C;
                    p.ws_bytes = 0;     // R' lives in TMEM
                    return true;
                }
            }
        }
    }
    void *k = nullptr;
    // compile-time n for C5 (n = 64800, C = 8, 736 threads)
    if (c.n == 64800 && c.wr == 6 && c.wc == 3 && C == 8 && H == 2 && p.threads <= 768 && !std::getenv("LDPC_NO_NFIX"))
        k = reinterpret_cast<void *>(&xband_kernel<6, 3, 2, 8, 768, 64800>);
    if (!k) k = pick_xband_kernel(c.wr, c.wc, H, C, p.threads);
    if (!k) return false;
    p.kernel = k;
    p.cluster = C;
    if ((p.threads - 32) * H < mbq || C * H > 32) return false;
    p.smem = xband_smem_bytes(c.n, c.wc, c.wr, C, c.dev.xcap, H);
    if (!ensure_smem_attribute(k, p.smem, C > 8)) return false;
    int nclusters = occupancy_clusters(k, p.threads, p.smem, C);
    if (nclusters < 1) return false;
    p.capacity = nclusters;
    nclusters = int(std::min<int64_t>(nclusters, std::max<int64_t>(frames, 1)));
    p.grid = nclusters * C;
    p.ws_bytes = 0;
    return true;
}

ldpc_status xcluster_launch(const ldpc_code &c, const XClusterPlan &p, const float *llr, int64_t frames,
                            const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                            void *ws, size_t ws_bytes, void *stream) {
    if (p.ws_bytes > 0 && (!ws || ws_bytes < p.ws_bytes)) return LDPC_ERR_ARG;
    XArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.adapt_votes = std::getenv("LDPC_XVOTE_ALWAYS") ? 0 : 1;
    a.rws = static_cast<float *>(ws);
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
