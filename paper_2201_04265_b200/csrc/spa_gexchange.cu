// spa_gexchange.cu -- Sum-Product decoding of frames too large for one SM
// (C5: n = 64800) by GROUPS of G CTAs that exchange message segments through
// L2-resident global staging buffers instead of cluster shared memory
// (variant 9).
//
// Same algorithm, ownership, tables, two frames in flight and arithmetic as
// xband2_kernel (spa_cluster.cu; Eqs. 4-8, flooding, Alg. 1
// P:351-369).  What changes is the transport:
//   * a 16-CTA cluster places only 7 per B200 (112 SMs; shared memory forces
//     one CTA per SM and clusters live inside a GPC), while groups need no
//     cluster: 9 groups of 16 CTAs use 144 SMs;
//   * a SENDER warp bulk-copies each finished segment from shared memory into
//     the destination's staging image (cp.async.bulk.global.shared::cta), waits
//     for its copies, and release-increments the destination's arrival counter;
//   * a RECEIVER warp acquire-polls its own counter until every segment of the
//     exchange has arrived and then bulk-loads the whole staging image into the
//     region (cp.async.bulk.shared::cluster.global, complete_tx on the region
//     barrier the compute warps wait on).
// Staging images are double-buffered by exchange parity.  Why no buffer is
// overwritten while still needed: a sender writes exchange p + 2 of (slot,
// direction) into the buffer of exchange p only after receiving data that its
// destination produced from exchange p + 1, which the destination computed
// after its receiver had loaded exchange p; a region is reloaded only after
// every sender of the new data consumed our previous data, which we signalled
// after our own outgoing copies from that region had completed (wait_group 0).
// The groups' CTAs must be co-resident: cooperative launch, one CTA per SM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {
using namespace band;

__device__ __forceinline__ uint32_t gx_saddr(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void gx_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void gx_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void gx_mbar_arm(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gx_mbar_wait(uint32_t bar, uint32_t parity) {
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
// shared -> global bulk copy (bulk-group completion), and its wait
__device__ __forceinline__ void gx_store(void *gdst, uint32_t ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void gx_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;" ::: "memory");
}
// global -> shared bulk copy completing on an mbarrier of this CTA
__device__ __forceinline__ void gx_load(uint32_t sdst, const void *gsrc, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
                 "l"(gsrc), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void gx_fence_proxy_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void gx_fence_proxy_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void gx_signal(unsigned *ctr) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}
__device__ __forceinline__ unsigned gx_poll(const unsigned *ctr) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    return v;
}

template <int D>
__device__ __forceinline__ void gx_ld_u32_row(const uint32_t *p, uint32_t (&o)[D]) {
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

struct GXArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    int32_t adapt_votes;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
    int32_t groups;
    unsigned *arrivals;      // [groups][2 slots][2 dirs][G] arrival counters (zeroed per launch)
    unsigned *gbar;          // [groups] group barrier counters (zeroed per launch)
    char *stage;             // [groups][2 slots][2 dirs][2 parities][G] staging images of cap_b bytes
    float *rws;              // [groups][2 slots][n] R' = clamp(R) log2(e)
    uint8_t *zbyte;          // [groups][2 parities][2 slots][n] final hard decisions
    int32_t *synd;           // [groups][2 parities][2 slots][G] per-CTA syndrome flags
};

__device__ __forceinline__ void gx_group_barrier(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (gx_poll(ctr) < target) {
        }
        __threadfence();
    }
    __syncthreads();
}

// Warps: TW / 32 compute warps, a sender warp, a receiver warp.
template <int WR, int WC, int G, int MAXT, int NFIX = 0>
__global__ void __launch_bounds__(MAXT, 1) gband2_kernel(const GXArgs a) {
    extern __shared__ __align__(128) char smem[];
    constexpr int NB = WC - 1, NC = NB;
    constexpr int DIR_L = 0, DIR_E = 1;
    const DeviceCode &code = a.code;
    const int n = NFIX ? NFIX : code.n, mb = NFIX ? NFIX / WR : code.mb, mbq = mb / G, nq = n / G;
    const int TW = NFIX ? xband_threads(NFIX / WR / G) : int(blockDim.x) - 64, tt = threadIdx.x, lane = tt & 31;
    const bool sender = tt >= TW && tt < TW + 32, receiver = tt >= TW + 32, compute = tt < TW;
    const uint32_t cap_b = uint32_t(code.xcap) * 4u;
    const int q = int(blockIdx.x) % G, grp = int(blockIdx.x) / G;
    char *varr[2] = {smem, smem + 2 * cap_b};
    char *rowr[2] = {smem + cap_b, smem + 3 * cap_b};
    uint32_t *vtab = reinterpret_cast<uint32_t *>(smem + 4 * cap_b);
    uint32_t *rtab = vtab + size_t(nq) * NB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + ((4 * cap_b + 8u * uint32_t(NB * nq) + 15u) & ~15u));
    constexpr int NBAR = 3 + NC;                 // per slot: var, row, vchunk, cchunk[NC]
    const uint32_t bar0 = gx_saddr(bars);
    auto vbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR); };
    auto rbar = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 1); };
    auto vchunk = [&](int sl) { return bar0 + 8u * uint32_t(sl * NBAR + 2); };
    auto cchunk = [&](int sl, int c) { return bar0 + 8u * uint32_t(sl * NBAR + 3 + c); };
    const int nkey = G * G * NC;
    const int32_t *varOff = code.xband_seg, *rowOff = code.xband_seg + nkey, *sbytes = code.xband_seg + 2 * nkey;
    auto key = [](int s, int d, int c) { return (s * G + d) * NC + c; };
    auto rslot = [&](int sl) { return a.rws + (size_t(grp) * 2 + size_t(sl)) * size_t(n); };
    auto arrivals = [&](int sl, int dir, int d) { return a.arrivals + ((size_t(grp) * 2 + sl) * 2 + dir) * G + d; };
    auto stage = [&](int sl, int dir, uint32_t par, int d) {
        return a.stage + ((((size_t(grp) * 2 + sl) * 2 + dir) * 2 + par) * G + d) * size_t(cap_b);
    };
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
    if (tt == 0) {
        for (int sl = 0; sl < 2; ++sl) {
            gx_mbar_init(vbar(sl), 1);
            gx_mbar_init(rbar(sl), 1);
            gx_mbar_init(vchunk(sl), uint32_t(TW / 32));
            for (int c = 0; c < NC; ++c) gx_mbar_init(cchunk(sl, c), uint32_t(TW / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto chunk_done = [&](uint32_t bar) {
        gx_fence_proxy_smem();
        __syncwarp();
        if (lane == 0) gx_mbar_arrive(bar);
    };
    // sender: exchange counters per slot (parity of the staging buffer)
    uint32_t nv[2] = {0, 0}, nc[2] = {0, 0};
    // receiver: exchanges received per slot and direction
    uint32_t rl[2] = {0, 0}, re[2] = {0, 0};
    // compute: region barrier phases
    uint32_t wl[2] = {0, 0}, we[2] = {0, 0};
    constexpr unsigned kSegsPerExchange = unsigned(G * NC);    // every sender signals every chunk
    // sender: V-phase chunk of slot sl -> L segments (q, d, c) into d's ROW image
    auto ship_l = [&](int sl) {
        gx_mbar_wait(vchunk(sl), nv[sl] & 1u);
        const uint32_t par = nv[sl] & 1u;
        const uint32_t vs = gx_saddr(varr[sl]);
        for (int i = lane; i < G * NC; i += 32) {
            const int d = i / NC, c = i - d * NC;
            const int k = key(q, d, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes) gx_store(stage(sl, DIR_L, par, d) + __ldg(rowOff + k), vs + uint32_t(__ldg(varOff + k)), nbytes);
        }
        gx_store_commit_wait();
        gx_fence_proxy_global();
        for (int i = lane; i < G * NC; i += 32) gx_signal(arrivals(sl, DIR_L, i / NC));
        ++nv[sl];
    };
    // sender: C-phase chunk c of slot sl -> E segments (s, q, c) into s's VAR image
    auto ship_e = [&](int sl, int c) {
        gx_mbar_wait(cchunk(sl, c), nc[sl] & 1u);
        const uint32_t par = nc[sl] & 1u;
        const uint32_t rs = gx_saddr(rowr[sl]);
        if (lane < G) {
            const int s = lane;
            const int k = key(s, q, c);
            const uint32_t nbytes = uint32_t(__ldg(sbytes + k));
            if (nbytes) gx_store(stage(sl, DIR_E, par, s) + __ldg(varOff + k), rs + uint32_t(__ldg(rowOff + k)), nbytes);
        }
        gx_store_commit_wait();
        gx_fence_proxy_global();
        if (lane < G) gx_signal(arrivals(sl, DIR_E, lane));
        if (c == NC - 1) ++nc[sl];
    };
    // receiver: wait for every segment of the next exchange, then load the image
    auto recv = [&](int sl, int dir) {
        uint32_t &cnt = dir == DIR_L ? rl[sl] : re[sl];
        if (lane == 0) {
            const unsigned target = kSegsPerExchange * (cnt + 1);
            const unsigned *ctr = arrivals(sl, dir, q);
            while (gx_poll(ctr) < target) {
            }
            gx_fence_proxy_global();
            const uint32_t bar = dir == DIR_L ? rbar(sl) : vbar(sl);
            gx_mbar_arm(bar, cap_b);
            gx_load(gx_saddr(dir == DIR_L ? rowr[sl] : varr[sl]), stage(sl, dir, cnt & 1u, q), cap_b, bar);
        }
        __syncwarp();
        ++cnt;
    };
    auto wait_row = [&](int sl) {
        gx_mbar_wait(rbar(sl), wl[sl] & 1u);
        ++wl[sl];
    };
    auto wait_var = [&](int sl) {
        gx_mbar_wait(vbar(sl), we[sl] & 1u);
        ++we[sl];
    };

    const int r = tt;
    const bool own = compute && r < mbq;
    const int64_t npairs = (a.frames + 1) / 2;
    unsigned nbar = 0;
    uint32_t fpar = 0;
    for (int64_t pi = grp; pi < npairs; pi += a.groups, fpar ^= 1u) {
        int64_t fs[2] = {2 * pi, 2 * pi + 1};
        const int ns = fs[1] < a.frames ? 2 : 1;
        float e0[2][WR];
        uint32_t synd[2] = {0, 0};
        bool vote_on[2] = {true, true}, hit[2] = {false, false};
        if (sender) {
            for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            for (int t = 1; t <= a.max_iter; ++t) {
                for (int sl = 0; sl < ns; ++sl)
#pragma unroll
                    for (int c = 0; c < NC; ++c) ship_e(sl, c);
                for (int sl = 0; sl < ns; ++sl) ship_l(sl);
            }
        } else if (receiver) {
            for (int t = 1; t <= a.max_iter; ++t) {
                for (int sl = 0; sl < ns; ++sl) recv(sl, DIR_L);
                for (int sl = 0; sl < ns; ++sl) recv(sl, DIR_E);
            }
            for (int sl = 0; sl < ns; ++sl) recv(sl, DIR_L);     // final L for the syndrome
        } else {
            // ---- V-phase 0 of both slots: L = R, E = 0; band-0 check of t = 1
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
                if (sl < ns) {
                    float lv[WR];
                    if (own) {
                        const int v0 = (q * mbq + r) * WR;
                        lds_row<WR>(reinterpret_cast<const char *>(a.llr + fs[sl] * int64_t(n)), uint32_t(v0) * 4u, lv);
#pragma unroll
                        for (int j = 0; j < WR; ++j) lv[j] = fminf(fmaxf(lv[j], -30.0f), 30.0f) * kL2E;
                        sts_row<WR>(reinterpret_cast<char *>(rslot(sl)), uint32_t(v0) * 4u, lv);
                        const uint32_t *vt = vtab + size_t(r) * WR * NB;
#pragma unroll
                        for (int j = 0; j < WR; ++j)
#pragma unroll
                            for (int b = 0; b < NB; ++b) *reinterpret_cast<float *>(varr[sl] + vt[j * NB + b]) = lv[j];
                    }
                    chunk_done(vchunk(sl));
                    if (own) check_row<WR, true>(lv, e0[sl]);
                }
            }
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
                                gx_ld_u32_row<WR>(rtab + (size_t(b) * mbq + r) * WR, s_);
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
                        if (own) lds_row<WR>(reinterpret_cast<const char *>(rslot(sl)), uint32_t((q * mbq + r) * WR) * 4u, lv);
                        wait_var(sl);
                        if (own) {
                            uint32_t s_[WR * NB];
                            gx_ld_u32_row<WR * NB>(vtab + size_t(r) * WR * NB, s_);
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
            // ---- a6/a8: L_v sits in the VAR slot of (v, band 1); hard decisions
            // of the CTA's variables to the group's staging bytes, posteriors out
            for (int sl = 0; sl < ns; ++sl) {
                uint8_t *zb = a.zbyte + ((size_t(grp) * 2 + fpar) * 2 + sl) * size_t(n) + size_t(q) * nq;
                float *dst = a.posterior ? a.posterior + fs[sl] * int64_t(n) + int64_t(q) * nq : nullptr;
                for (int i = tt; i < nq; i += TW) {
                    const float lv = *reinterpret_cast<const float *>(varr[sl] + vtab[size_t(i) * NB]);
                    zb[i] = lv >= 0.0f ? 1 : 0;
                    if (dst) dst[i] = lv * kLn2;
                }
            }
        }
        // per-CTA syndrome flags and hard decisions -> group barrier -> outputs
        int32_t *sf = a.synd + ((size_t(grp) * 2 + fpar) * 2) * G;
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
            const int any = __syncthreads_or(synd[sl] != 0);
            if (tt == 0) sf[sl * G + q] = any;
        }
        nbar += G;
        gx_group_barrier(a.gbar + grp, nbar);
        if (compute) {
            const int nw = code.nw;
            const int w_lo = (q * nq + 31) / 32;
            const int w_hi = (q == G - 1) ? nw : ((q + 1) * nq + 31) / 32;
            for (int sl = 0; sl < ns; ++sl) {
                const uint8_t *zb = a.zbyte + ((size_t(grp) * 2 + fpar) * 2 + sl) * size_t(n);
                uint32_t *bits = a.bits + fs[sl] * int64_t(nw);
                for (int base = w_lo * 32; base < w_hi * 32; base += TW) {
                    const int v = base + tt;
                    if (v >= w_hi * 32) break;
                    const bool z = v < n && zb[v] != 0;
                    const uint32_t word = __ballot_sync(0xffffffffu, z);
                    if (lane == 0) bits[v >> 5] = word;
                }
                if (q == 0 && tt == 0) {
                    int ok = 1;
                    for (int i = 0; i < G; ++i) ok &= (sf[sl * G + i] == 0);
                    a.syn_ok[fs[sl]] = uint8_t(ok);
                    a.iters[fs[sl]] = a.max_iter;
                }
            }
        }
    }
    // launched as the dependent of xband2_kernel (the tail on the SMs its
    // clusters leave idle): this grid completes only after that one has, so
    // whatever the stream runs next sees both grids' outputs (a no-op for a
    // plain launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace

bool gx_plan(const ldpc_code &c, int64_t frames, bool et, GXPlan &p, int max_groups_cap) {
    if (et || !c.gallager || !c.regular_col || !c.dev.xcluster || c.dev.xslots != 2 || c.wr != 6 || c.wc != 3)
        return false;
    constexpr int G = 16;
    if (c.dev.xcluster != G || c.dev.xrows != 1) return false;
    const int mbq = c.n / c.wr / G;
    const int tw = (mbq + 31) / 32 * 32;
    p.threads = tw + 64;
    if (p.threads > 768) return false;
    void *k = (c.n == 64800 && !std::getenv("LDPC_NO_NFIX")) ? reinterpret_cast<void *>(&gband2_kernel<6, 3, G, 768, 64800>)
                                                            : reinterpret_cast<void *>(&gband2_kernel<6, 3, G, 768>);
    p.smem = xband2_smem_bytes(c.n, c.wc, c.wr, G, c.dev.xcap);
    if (p.smem + 1024 > 227 * 1024) return false;
    if (!ensure_smem_attribute(k, p.smem)) return false;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, p.threads, p.smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return false;
    }
    const int sms = device_attribute(cudaDevAttrMultiProcessorCount);
    int max_groups = sms * per_sm / G;
    if (max_groups_cap > 0) max_groups = std::min(max_groups, max_groups_cap);
    if (max_groups < 1) return false;
    p.groups = int(std::min<int64_t>(max_groups, std::max<int64_t>(1, (frames + 1) / 2)));
    p.kernel = k;
    p.capacity = 2 * int64_t(max_groups);
    p.grid = p.groups * G;
    const size_t cap_b = size_t(c.dev.xcap) * 4;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    p.off_arrivals = 0;
    p.off_gbar = al(size_t(p.groups) * 2 * 2 * G * 4);
    p.zero_bytes = al(p.off_gbar + size_t(p.groups) * 4);
    p.off_stage = p.zero_bytes;
    p.off_rws = al(p.off_stage + size_t(p.groups) * 2 * 2 * 2 * G * cap_b);
    p.off_zbyte = al(p.off_rws + size_t(p.groups) * 2 * size_t(c.n) * 4);
    p.off_synd = al(p.off_zbyte + size_t(p.groups) * 2 * 2 * size_t(c.n));
    p.ws_bytes = al(p.off_synd + size_t(p.groups) * 2 * 2 * G * 4);
    return true;
}

ldpc_status gx_launch(const ldpc_code &c, const GXPlan &p, const float *llr, int64_t frames, const ldpc_decode_opts &o,
                      uint32_t *bits, uint8_t *syn, int32_t *iters, float *post, void *ws, size_t ws_bytes,
                      void *stream, bool dependent) {
    if (!ws || ws_bytes < p.ws_bytes) return LDPC_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char *w = static_cast<char *>(ws);
    if (!dependent && cudaMemsetAsync(w, 0, p.zero_bytes, s) != cudaSuccess) return LDPC_ERR_CUDA;
    GXArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.adapt_votes = std::getenv("LDPC_XVOTE_ALWAYS") ? 0 : 1;
    a.bits = bits;
    a.syn_ok = syn;
    a.iters = iters;
    a.posterior = post;
    a.groups = p.groups;
    a.arrivals = reinterpret_cast<unsigned *>(w + p.off_arrivals);
    a.gbar = reinterpret_cast<unsigned *>(w + p.off_gbar);
    a.stage = w + p.off_stage;
    a.rws = reinterpret_cast<float *>(w + p.off_rws);
    a.zbyte = reinterpret_cast<uint8_t *>(w + p.off_zbyte);
    a.synd = reinterpret_cast<int32_t *>(w + p.off_synd);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    if (dependent) {
        // starts once every CTA of the exchange-cluster grid before it is
        // resident (griddepcontrol.launch_dependents there), on the SMs those
        // clusters leave free; no cooperative attribute: the 16 CTAs of a group
        // are co-resident because the grid fits the idle SMs, and a CTA that
        // had to wait for the primary grid to drain only delays its group
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
    } else {
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    }
    cfg.gridDim = dim3(unsigned(p.grid));
    cfg.blockDim = dim3(unsigned(p.threads));
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {&a};
    const cudaError_t e = cudaLaunchKernelExC(&cfg, p.kernel, args);
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // namespace ldpc
