// band_kernel.cuh -- the Gallager band decoder kernel template (see the
// comment at the top of spa_band.cu), shared by spa_band.cu (generic
// instantiations, launch code) and spa_band_fixed.cu (instantiations with the
// code length compiled in).  Included inside an anonymous namespace by each
// translation unit.
#pragma once

#ifndef BAND_FUSE0
#define BAND_FUSE0 true
#endif
#ifndef BAND_ADAPT_VOTES
#define BAND_ADAPT_VOTES 1
#endif
#ifndef BAND_C1_INTERLEAVE
#define BAND_C1_INTERLEAVE 1
#endif
#ifndef BAND_TMEM_OFFSETS
#define BAND_TMEM_OFFSETS 1
#endif
#ifndef BAND_EDET
#define BAND_EDET 1
#endif

struct BandArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    int32_t early_term;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
    unsigned long long *frame_counter;   // zeroed before launch; null: frames grid-stride
    float *r_global;                     // R' per CTA slot when R does not fit in smem
    int32_t r_in_smem;
    int32_t row_stride;                  // S = ceil(mb / B0): thread t owns rows t, t+S, ...
                                         // (balanced: every active thread gets B0 band-0 rows)
    // GEN (fused simulate, N4): R drawn in the prologue from (seed, frame0 + f)
    // and the codeword, counters added in the epilogue
    uint64_t seed;
    int64_t frame0;
    double sigma;
    const uint32_t *cw;
    const uint32_t *info;
    unsigned long long *counters;        // int64[6], as ldpc_count_errors
};

__device__ __forceinline__ bool cta_sync_or(bool p) { return __syncthreads_or(p ? 1 : 0) != 0; }

// WR: row weight, WC: column weight (bands), B0: max band-0 rows per thread.
// wc > 3 (Table I codes, n = 1032) use small CTAs: the 256-thread bound leaves
// room for the wider per-row state.
// MODE 0: check-major E; 1: variable-major E (VM); 2: VM + 16-bit L offsets.
// NFIX: 0, or the code length compiled in (the DVB-S2 short frame n = 16200 of
// C4): sizes, region bases, band offsets and the row stride become immediates
// (fewer integer instructions per edge-update; same arithmetic, same results).
// GEN: fused simulate (ldpc_decode_simulate): the prologue draws R
// exactly as ldpc_channel does (channel_common.cuh) instead of loading it, and
// the epilogue accumulates the counters of ldpc_count_errors per CTA (flushed
// with six atomics when the CTA runs out of frames).
// RPRE: band-0 rows whose R is prefetched before the check->variable barrier
// (only when R lives in global memory).
// NOVOTE: psi regime votes off.  The votes pay only when many iterations run
// after a frame has converged; with few iterations (C1: 20, Table I: 10) they
// are overhead and their branches and warp syncs lengthen the dependency
// chain (measured: C1 +35%, Table I +6..20%).  Chosen at plan time.
// LPR: lanes per check row.  2 splits every row over a lane pair (each lane
// WR/2 elements, check_row_pair): twice the threads per frame and half the
// serial chain, for batches too small to fill the GPU one thread per row
// (C1, Table I at 1000 frames).  Without psi votes the results are bit for
// bit those of LPR = 1.  NFIX kernels only.
// Launch bounds: the lane-pair kernels (NFIX) declare their exact block size
// and BAND_LPR2_MINB blocks per SM (Table I wc = 9: 5 fit shared memory).
#ifndef BAND_LPR2_MINB
#define BAND_LPR2_MINB 5
#endif
#ifndef BAND_C3R34_MINB
#define BAND_C3R34_MINB 3      // C3 R3/4 (352 threads): 3 blocks per SM, 56 registers (2 blocks, 80 registers, no spill: 0.795 vs 0.805)
#endif
#ifndef BAND_T1R34_MINB
#define BAND_T1R34_MINB 8      // Table I R3/4 (96 threads): 80 registers, no spill
#endif
#ifndef BAND_C2B2_MINB
#define BAND_C2B2_MINB 12      // C2 with two rows per thread (96 threads): 12 blocks (56 registers; 14 fit shared memory but spill at 40)
#endif
#ifndef BAND_NFIX_MINB
#define BAND_NFIX_MINB 1
#endif
// blocks per SM the compile-time-n kernels ask the register allocator for
// (BAND_NFIX_MINB 0: 1) -- as many as shared memory allows, where the
// registers then still fit without heavy spills: C2 (n = 1008): 7 (40
// registers), C3 (n = 3996): 2 (wr 6, 40 registers) / 3 (wr 12, 56).
// Measured: C3-R1/2 77.6 -> 91.4% of the SFU roofline, C3-R3/4 66.9 ->
// 69.2%, C2 51.2 -> 52.0%; C2 at 10 blocks (32 registers) 47.6%.
constexpr int band_lb_minb(int wr, int nfix, int lpr, int wc = 0, int b0 = 1) {
    return lpr == 2 ? BAND_LPR2_MINB
         : !BAND_NFIX_MINB ? 1
         : nfix == 1008 ? (b0 == 2 ? BAND_C2B2_MINB : 7) : nfix == 3996 ? (wr == 12 ? BAND_C3R34_MINB : wr == 4 ? 3 : b0 == 2 ? 3 : 2)
         : (nfix == 1032 && wc == 3) ? BAND_T1R34_MINB : 1;
}
constexpr int band_lb_threads(int wr, int wc, int b0, int nfix, int lpr) {
    return (lpr == 2 || band_lb_minb(wr, nfix, lpr, wc, b0) > 1) ? ((nfix / wr + b0 - 1) / b0 + 31) / 32 * 32 * lpr
                                                          : (wc > 3 ? 256 : 1024);
}
// LPR0: lanes per band-0 row (default LPR).  C1 runs one lane per row of
// bands >= 1 (32 rows, all 32 lanes) and a lane pair per band-0 row (16 rows
// on 32 lanes instead of 16), halving the variable phase's chain.
template <int WR, int WC, int B0, bool ET, int MODE, int NFIX = 0, bool GEN = false, int RPRE = 0, bool NOVOTE = false,
          int LPR = 1, int LPR0 = LPR>
__global__ void __launch_bounds__(band_lb_threads(WR, WC, B0, NFIX, LPR), band_lb_minb(WR, NFIX, LPR, WC, B0))
    band_kernel(const BandArgs a) {
    // measured on B200: +1.1 points on C4 (MODE 2), +0.8..1.3 on wr = 12 codes,
    // -2..3 on check-major wr = 4 / 6 codes (C3 R1/4, R1/2)
    // C1I (C1: n = 96, band-0 rows on lane pairs, no votes, fixed
    // iterations): every lane has one band-0 half row and one row of bands
    // 1-2.  The check phase runs both updates in one block so their two
    // dependency chains interleave (a 1000-frame C1 batch is one latency-bound
    // wave); the band-0 check therefore leaves the variable phase (no FUSE0).
    constexpr bool C1I = BAND_C1_INTERLEAVE && NFIX == 96 && LPR == 1 && LPR0 == 2 && B0 == 1 && !ET && NOVOTE &&
                         MODE == 0 && !GEN;
    constexpr bool FUSE0 = BAND_FUSE0 && (MODE == 2 || WR >= 12 || NOVOTE) && !C1I;
    // Adaptive psi votes (one lane per row): a warp votes in iteration t only
    // if one of its votes hit in t - 1, or t = 1 mod 4.  Votes that keep
    // failing (rows straddling the regime split) cost ~5 instructions per
    // edge-update; the tiers are exact or within the psi error budget.
    // Measured against always-on votes: C4 0.941 -> 0.952, C3-R3/4 0.778 ->
    // 0.792; worse on C3-R1/4 (-3%) and C3-R1/2 (-8%), and with votes under
    // early termination C2 -3% (1.0 dB) and -7% (3.0 dB) -- so only C4 and
    // the wr = 12 codes use it, and early termination stays vote-free.
    constexpr bool ADAPT = BAND_ADAPT_VOTES && !NOVOTE && !ET && LPR == 1 && LPR0 == 1 && (NFIX == 16200 || WR >= 12);
    constexpr bool VM = MODE >= 1, L16 = MODE == 2;
    // EDET: early termination decided at the end of the variable phase
    // (BAND_EDET, measured: DESIGN.md "C2")
    constexpr bool EDET = ET && BAND_EDET;
    // CSYN: the check phase carries the syndrome of z^{t-1} and the stop test
    // (ET without EDET; with EDET that test could never fire: the variable
    // phase of t - 1 has already tested the same z)
    constexpr bool CSYN = ET && !EDET;
    static_assert(LPR == 1 || (LPR == 2 && NFIX && !GEN && RPRE == 0 && WR % 2 == 0), "lane pairs: NFIX kernels");
    constexpr int WH = WR / LPR;          // elements of a row per lane
    extern __shared__ __align__(16) char smem[];
    __shared__ long long s_frame;
    const DeviceCode &code = a.code;
    // rows per row-pass (the row stride, a multiple of 32) and threads
    // (= TFIX * LPR): lane pairs double the threads of the same row passes
    constexpr int TFIX = NFIX ? (((NFIX / WR + B0 - 1) / B0 + 31) / 32 * 32) : 0;
    constexpr bool RFIX_SMEM = NFIX && size_t(WC + 1) * NFIX * 4 + 1024 <= 227 * 1024;
    const int n = NFIX ? NFIX : code.n, mb = NFIX ? NFIX / WR : code.mb;
    const int T = NFIX ? TFIX * LPR : int(blockDim.x), tt = threadIdx.x, S = NFIX ? TFIX : a.row_stride;
    const int pr = tt / LPR, h = tt % LPR;   // row slot, half of the row
    const uint32_t hoff = uint32_t(h * WH);  // first element of this lane
    // band-0 rows: LPR0 lanes each, row stride S0
    constexpr int WH0 = WR / LPR0;
    static_assert(LPR0 == LPR || (LPR == 1 && LPR0 == 2 && NFIX && !GEN && RPRE == 0 && WR % 2 == 0 &&
                                  NFIX / WR <= TFIX * LPR / LPR0 * B0),
                  "band-0 lane pairs: NFIX kernels whose band-0 rows fit the halved stride");
    const int S0 = S * LPR / LPR0;
    const int pr0 = tt / LPR0, h0 = tt % LPR0;
    const uint32_t hoff0 = uint32_t(h0 * WH0);
    const bool r_in_smem = NFIX ? RFIX_SMEM : a.r_in_smem != 0;
    constexpr int NB = WC - 1;          // bands held in shared memory
    constexpr int B1 = NB * B0;         // max rows of bands >= 1 per thread
    const uint32_t lbase = uint32_t(NB) * uint32_t(n) * 4u;
    const uint32_t rbase = lbase + uint32_t(n) * 4u;
    float *Ls = reinterpret_cast<float *>(smem + lbase);
    float *Rs = r_in_smem ? reinterpret_cast<float *>(smem + rbase) : a.r_global + size_t(blockIdx.x) * n;
    const int32_t *lidx = code.band_lidx;
    const int32_t *vpos = code.band_vpos;

    // rows too wide to saturate: the clamp tier's constant magnitudes
    // (band_common.cuh clamp_row_mags), computed once per CTA by warp 0 and
    // ordered before use by the frame loop's first barrier
    constexpr bool CMT = has_clamp_tier<WR>() && !ET && !NOVOTE && LPR == 1;
    __shared__ float s_cm[CMT ? WR : 1];
    if constexpr (CMT) {
        if (tt < 32) {
            float m[WR];
            clamp_row_mags<WR>(m);
            if (tt == 0)
#pragma unroll
                for (int j = 0; j < WR; ++j) s_cm[j] = m[j];
        }
    }
    const float *cmp = CMT ? s_cm : nullptr;

    unsigned long long cnt[6] = {0, 0, 0, 0, 0, 0};       // GEN: this CTA's counters (thread 0)
    __shared__ int s_err[2];
    // TMIDX (compile-time n with 16-bit offsets and one lane per row: C4):
    // constant per-thread data lives in Tensor Memory (otherwise idle
    // here) instead of being re-read every iteration -- the packed L offsets
    // of the thread's B1 rows of bands >= 1 (from L1/L2; written once per
    // launch) and the R' of its B0 band-0 rows (from an L2 slot, C4, or
    // shared memory, C3; copied from L = R' at each frame's ingest).  Warp w
    // owns lanes 32 (w % 4) .. + 31 and PERW columns from PERW (w / 4): row
    // k's offsets at OFFW k, its R' at B1 OFFW + RW k (tcgen05.ld, 12-cycle
    // latency).  The CTA allocates TMCOLS (a power of two; C3 runs 2-3 CTAs
    // per SM, all fit the 512 columns).
    // (C3 at 2-3 CTAs per SM with R in shared memory measured much worse with
    // it: 1.20 -> 0.95, 1.13 -> 1.00, 0.79 -> 0.59 of the SFU model -- C4 only.)
    constexpr bool TMIDX = L16 && LPR == 1 && LPR0 == 1 && NFIX == 16200 && BAND_TMEM_OFFSETS;
    constexpr int OFFW = pow2_at_least(WR / 2), RW = pow2_at_least(WR);
    constexpr int PERW = B1 * OFFW + B0 * RW;
    constexpr int TMCOLS = TMIDX ? pow2_at_least(PERW * ((TFIX / 32 + 3) / 4) < 32 ? 32 : PERW * ((TFIX / 32 + 3) / 4)) : 32;
    static_assert(!TMIDX || TMCOLS <= 256 || NFIX == 16200, "TMEM columns of a multi-CTA kernel");
    __shared__ uint32_t s_tmem;
    uint32_t tm_row0 = 0, tm_r0 = 0;
    if constexpr (TMIDX) {
        const uint32_t warp = uint32_t(tt) >> 5;
        if (warp == 0) {
            const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem));
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "n"(TMCOLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        tm_row0 = s_tmem + ((32u * (warp & 3u)) << 16) + uint32_t(PERW) * (warp >> 2);
        tm_r0 = tm_row0 + uint32_t(B1 * OFFW);
#pragma unroll
        for (int k = 0; k < B1; ++k) {
            const int r = pr + k * S;
            uint32_t w[OFFW];
#pragma unroll
            for (int i = 0; i < OFFW; ++i) w[i] = 0u;
            if (pr < S && r < NB * mb) {
                const uint32_t *p16 = reinterpret_cast<const uint32_t *>(code.band_lidx16 + size_t(r) * WR);
#pragma unroll
                for (int i = 0; i < WR / 2; ++i) w[i] = __ldg(p16 + i);
            }
            tmem_st<OFFW>(tm_row0 + uint32_t(OFFW * k), w);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    // frames: claimed from the counter (dynamic, batches beyond one wave), or
    // grid-stride when the launch holds every frame at once (no counter, so
    // no memset node before a small batch's decode; the previous frame index
    // stays in s_frame, so no register is live across the loop)
    if (tt == 0) s_frame = (long long)blockIdx.x - (long long)gridDim.x;
    for (;;) {
        if (tt == 0)
            s_frame = a.frame_counter ? (long long)atomicAdd(a.frame_counter, 1ull) : s_frame + gridDim.x;
        if (GEN && tt < 2) s_err[tt] = 0;
        __syncthreads();
        const long long f = s_frame;
        if (f >= a.frames) break;

        // a1/a2: ingest R (clamped +-30, log2 units), L = R, E = 0
        if constexpr (GEN) {
            // R of frame frame0 + f as ldpc_channel draws it (Eq. 4)
            const uint32_t *c = a.cw + f * (long long)code.nw;
            const uint64_t fr = uint64_t(a.frame0 + f);
            for (int v4 = tt; v4 < (n >> 2); v4 += T) {
                double z[4];
                channel_normals(a.seed, fr, v4, z);
                const uint32_t word = __ldg(c + (v4 >> 3)) >> ((4 * v4) & 31);
                float4 r;
                r.x = fminf(fmaxf(channel_llr(word & 1u, a.sigma, z[0]), -30.0f), 30.0f) * kL2E;
                r.y = fminf(fmaxf(channel_llr(word & 2u, a.sigma, z[1]), -30.0f), 30.0f) * kL2E;
                r.z = fminf(fmaxf(channel_llr(word & 4u, a.sigma, z[2]), -30.0f), 30.0f) * kL2E;
                r.w = fminf(fmaxf(channel_llr(word & 8u, a.sigma, z[3]), -30.0f), 30.0f) * kL2E;
                reinterpret_cast<float4 *>(Rs)[v4] = r;
                reinterpret_cast<float4 *>(Ls)[v4] = r;
            }
        } else {
            const float *src = a.llr + f * (long long)n;
            for (int v4 = tt; v4 < (n >> 2); v4 += T) {
                float4 r = __ldg(reinterpret_cast<const float4 *>(src) + v4);
                r.x = fminf(fmaxf(r.x, -30.0f), 30.0f) * kL2E;
                r.y = fminf(fmaxf(r.y, -30.0f), 30.0f) * kL2E;
                r.z = fminf(fmaxf(r.z, -30.0f), 30.0f) * kL2E;
                r.w = fminf(fmaxf(r.w, -30.0f), 30.0f) * kL2E;
                if (!TMIDX) reinterpret_cast<float4 *>(Rs)[v4] = r;      // TMIDX: R' goes to TMEM from L
                reinterpret_cast<float4 *>(Ls)[v4] = r;
            }
        }
        for (int i = tt; i < (NB * n) >> 2; i += T)
            reinterpret_cast<float4 *>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        float e0[B0][WH0];
#pragma unroll
        for (int k = 0; k < B0; ++k)
#pragma unroll
            for (int j = 0; j < WH0; ++j) e0[k][j] = 0.0f;
        __syncthreads();
        if constexpr (TMIDX) {
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = pr0 + k * S0;
                float rv[WR];
                uint32_t u[RW];
#pragma unroll
                for (int j = 0; j < RW; ++j) u[j] = 0u;
                if (pr0 < S0 && r < mb) {
                    lds_row<WR>(smem, lbase + uint32_t(r) * WR * 4u, rv);    // L = R' right after the ingest
#pragma unroll
                    for (int j = 0; j < WR; ++j) u[j] = __float_as_uint(rv[j]);
                }
                tmem_st<RW>(tm_r0 + uint32_t(RW * k), u);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }

        int32_t iters = a.max_iter;
        bool stopped = false;
        // Band-0 checks read only their own row's L, which the same thread has
        // just produced in the variable phase: the band-0 check of iteration
        // t+1 runs at the end of variable phase t from registers (FUSE0), and
        // the one of t = 1 here, from L = R.  Same rows per warp, same inputs:
        // results identical to running them in the check phase.
        uint32_t synd0 = 0;            // ET: band-0 rows' syndrome bits of z^{t-1}
        bool vote_on = true, vhit = false;  // ADAPT: warp-uniform
        if constexpr (FUSE0) {
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = pr0 + k * S0;
                const bool act = pr0 < S0 && r < mb;
                const unsigned pm = LPR0 > 1 ? __ballot_sync(0xffffffffu, act) : 0u;
                if (act) {
                    float x[WH0];
                    lds_row<WH0>(smem, lbase + (uint32_t(r) * WR + hoff0) * 4u, x);
                    if constexpr (ADAPT) vhit |= check_row_gated<WR>(x, e0[k], vote_on, cmp);
                    else check_any<WR, !ET && !NOVOTE, LPR0>(x, e0[k], h0, pm, cmp);
                }
            }
        }
        for (int t = 1; t <= a.max_iter; ++t) {
            if constexpr (ADAPT) {
                if (t > 1) {
                    vote_on = vhit || (t & 3) == 1;
                    vhit = false;
                }
            }
            // ---- a3: check-node phase (and syndrome of z^{t-1} when ET)
            uint32_t synd = FUSE0 ? synd0 : 0u;
            if constexpr (C1I) {
                const int r0 = pr0, r = pr;          // every lane: r0 < mb, r < NB mb
                float lv0[WH0], x0[WH0], x[WR], e[WR];
                lds_row<WH0>(smem, lbase + (uint32_t(r0) * WR + hoff0) * 4u, lv0);
#pragma unroll
                for (int j = 0; j < WH0; ++j) x0[j] = lv0[j] - e0[0][j];
                int32_t li[WR];
                ldg_idx<WR>(lidx + size_t(r) * WR, li);
                lds_row<WR>(smem, uint32_t(r) * WR * 4u, e);
#pragma unroll
                for (int j = 0; j < WR; ++j) x[j] = *reinterpret_cast<const float *>(smem + li[j]) - e[j];
                check_row_pair<WR, false>(x0, e0[0], h0, 0xffffffffu);
                check_row<WR, false>(x, e);
                sts_row<WR>(smem, uint32_t(r) * WR * 4u, e);
            }
#pragma unroll
            for (int k = 0; k < (FUSE0 || C1I ? 0 : B0); ++k) {
                const int r = pr0 + k * S0;
                const bool act = pr0 < S0 && r < mb;
                const unsigned pm = LPR0 > 1 ? __ballot_sync(0xffffffffu, act) : 0u;
                if (act) {
                    float lv[WH0], x[WH0];
                    lds_row<WH0>(smem, lbase + (uint32_t(r) * WR + hoff0) * 4u, lv);
                    uint32_t rp = 0;      // this row's syndrome bit (Eq. 1)
#pragma unroll
                    for (int j = 0; j < WH0; ++j) {
                        x[j] = lv[j] - e0[k][j];
                        if (CSYN) rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
                    }
                    if (CSYN && LPR0 > 1) rp ^= __shfl_xor_sync(pm, rp, 1);
                    synd |= rp;
                    if constexpr (ADAPT) vhit |= check_row_gated<WR>(x, e0[k], vote_on, cmp);
                    else check_any<WR, !ET && !NOVOTE, LPR0>(x, e0[k], h0, pm, cmp);
                }
            }
#pragma unroll
            for (int k = 0; k < (C1I ? 0 : B1); ++k) {
                const int r = pr + k * S;
                const bool act = pr < S && r < NB * mb;
                const unsigned pm = LPR > 1 ? __ballot_sync(0xffffffffu, act) : 0u;
                uint32_t tmw[TMIDX ? OFFW : 1];
                if constexpr (TMIDX) tmem_ld<OFFW>(tm_row0 + uint32_t(OFFW * k), tmw);
                if (act) {
                    int32_t li[WH];
                    float e[WH], x[WH];
                    if constexpr (TMIDX) {
#pragma unroll
                        for (int w = 0; w < WR / 2; ++w) {
                            li[2 * w] = int32_t(lbase + (tmw[w] & 0xffffu));
                            li[2 * w + 1] = int32_t(lbase + (tmw[w] >> 16));
                        }
                    } else if (L16 && LPR > 1) {
#pragma unroll
                        for (int j = 0; j < WH; ++j)
                            li[j] = int32_t(lbase + __ldg(code.band_lidx16 + size_t(r) * WR + hoff + j));
                    } else if (L16) {
                        // 16-bit offsets relative to L: half the index bytes through L1/L2
                        const uint32_t *p16 = reinterpret_cast<const uint32_t *>(code.band_lidx16 + size_t(r) * WR);
#pragma unroll
                        for (int w = 0; w < WR / 2; ++w) {
                            const uint32_t x = __ldg(p16 + w);
                            li[2 * w] = int32_t(lbase + (x & 0xffffu));
                            li[2 * w + 1] = int32_t(lbase + (x >> 16));
                        }
                    } else {
                        ldg_idx<WH>(lidx + size_t(r) * WR + hoff, li);
                    }
                    // VM: E_b is variable-major, at the variable's L offset + delta_b
                    const int32_t delta = VM ? int32_t((r / mb) * n * 4) - int32_t(lbase) : 0;
                    if (VM) {
#pragma unroll
                        for (int j = 0; j < WH; ++j) e[j] = *reinterpret_cast<const float *>(smem + li[j] + delta);
                    } else {
                        lds_row<WH>(smem, (uint32_t(r) * WR + hoff) * 4u, e);
                    }
                    uint32_t rp = 0;
#pragma unroll
                    for (int j = 0; j < WH; ++j) {
                        const float lv = *reinterpret_cast<const float *>(smem + li[j]);
                        x[j] = lv - e[j];
                        if (CSYN) rp ^= (lv >= 0.0f) ? 1u : 0u;
                    }
                    if (CSYN && LPR > 1) rp ^= __shfl_xor_sync(pm, rp, 1);
                    synd |= rp;
                    if constexpr (ADAPT) vhit |= check_row_gated<WR>(x, e, vote_on, cmp);
                    else check_any<WR, !ET && !NOVOTE, LPR>(x, e, h, pm, cmp);
                    if (VM) {
#pragma unroll
                        for (int j = 0; j < WH; ++j) *reinterpret_cast<float *>(smem + li[j] + delta) = e[j];
                    } else {
                        sts_row<WH>(smem, (uint32_t(r) * WR + hoff) * 4u, e);
                    }
                }
            }
            // R of this thread's first band-0 rows, loaded before the barrier so its
            // latency (an L2-resident slot when R does not fit shared memory)
            // overlaps the barrier wait instead of opening the variable phase
            constexpr int RP = B0 < RPRE ? B0 : RPRE;
            float rpre[RP > 0 ? RP : 1][WR];
            if (RP > 0 && !r_in_smem) {
#pragma unroll
                for (int k = 0; k < RP; ++k) {
                    const int r = pr + k * S;
                    if (pr < S && r < mb) lds_row<WR>(reinterpret_cast<const char *>(Rs), uint32_t(r) * WR * 4u, rpre[k]);
                }
            }
            if (CSYN) {
                const bool any = cta_sync_or(synd != 0);
                if (t > 1 && !any) {      // z^{t-1} has zero syndrome: stop (reading c6)
                    iters = t - 1;
                    stopped = true;
                    break;
                }
            } else {
                __syncthreads();
            }
            // ---- a4/a5: variable-node phase, Eq. 7 (owners of band-0 rows)
            synd0 = 0;
            uint32_t sv0 = 0;           // EDET: band-0 rows' syndrome bits of z^t
#pragma unroll
            for (int k = 0; k < B0; ++k) {
                const int r = pr0 + k * S0;
                const bool act = pr0 < S0 && r < mb;
                const unsigned pm = LPR0 > 1 ? __ballot_sync(0xffffffffu, act) : 0u;
                uint32_t tr[TMIDX ? RW : 1];
                if constexpr (TMIDX) tmem_ld<RW>(tm_r0 + uint32_t(RW * k), tr);
                if (act) {
                    float rv[WH0], lv[WH0];
                    if constexpr (TMIDX) {
#pragma unroll
                        for (int j = 0; j < WH0; ++j) rv[j] = __uint_as_float(tr[j]);
                    } else if (k < RP && !r_in_smem) {
#pragma unroll
                        for (int j = 0; j < WH0; ++j) rv[j] = rpre[k < RP ? k : 0][j];
                    } else {
                        lds_row<WH0>(reinterpret_cast<const char *>(Rs), (uint32_t(r) * WR + hoff0) * 4u, rv);
                    }
                    if (VM) {
                        // this row's variables are contiguous in every band's E_b
#pragma unroll
                        for (int j = 0; j < WH0; ++j) lv[j] = rv[j] + e0[k][j];
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            float eb[WH0];
                            lds_row<WH0>(smem, uint32_t(b) * n * 4u + (uint32_t(r) * WR + hoff0) * 4u, eb);
#pragma unroll
                            for (int j = 0; j < WH0; ++j) lv[j] += eb[j];
                        }
                    } else {
                        int32_t vp[WH0 * NB];
                        ldg_idx<WH0 * NB>(vpos + (size_t(r) * WR + hoff0) * NB, vp);
#pragma unroll
                        for (int j = 0; j < WH0; ++j) {
                            float s = rv[j] + e0[k][j];
#pragma unroll
                            for (int b = 0; b < NB; ++b) s += *reinterpret_cast<const float *>(smem + vp[j * NB + b]);
                            lv[j] = s;
                        }
                    }
                    sts_row<WH0>(smem, lbase + (uint32_t(r) * WR + hoff0) * 4u, lv);
                    if constexpr (EDET) {
                        uint32_t rp = 0;
#pragma unroll
                        for (int j = 0; j < WH0; ++j) rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
                        if (LPR0 > 1) rp ^= __shfl_xor_sync(pm, rp, 1);
                        sv0 |= rp;
                    }
                    if constexpr (FUSE0) {
                        if (CSYN) {
                            uint32_t rp = 0;      // this band-0 row's syndrome bit of z^t (Eq. 1)
#pragma unroll
                            for (int j = 0; j < WH0; ++j) rp ^= (lv[j] >= 0.0f) ? 1u : 0u;
                            if (LPR0 > 1) rp ^= __shfl_xor_sync(pm, rp, 1);
                            synd0 |= rp;
                        }
                        if (t < a.max_iter) {
                            float x[WH0];
#pragma unroll
                            for (int j = 0; j < WH0; ++j) x[j] = lv[j] - e0[k][j];
                            if constexpr (ADAPT) vhit |= check_row_gated<WR>(x, e0[k], vote_on, cmp);
                    else check_any<WR, !ET && !NOVOTE, LPR0>(x, e0[k], h0, pm, cmp);
                        }
                    }
                }
            }
            if constexpr (EDET) {
                // early detection (reading c6 / Q11): when no band-0 row of
                // z^t is unsatisfied, test the other bands' rows at once (sign
                // gathers only) and stop here -- iters = t, the posteriors just
                // written -- instead of one check phase later, whose psi work
                // would be thrown away.  Same stopping iteration and outputs.
                if (t < a.max_iter && !cta_sync_or(sv0 != 0)) {
                    uint32_t s12 = 0;
                    for (int r = tt; r < NB * mb; r += T) {
                        uint32_t rp = 0;
#pragma unroll
                        for (int j = 0; j < WR; ++j)
                            rp ^= (*reinterpret_cast<const float *>(smem + __ldg(lidx + size_t(r) * WR + j)) >= 0.0f)
                                      ? 1u
                                      : 0u;
                        s12 |= rp;
                    }
                    if (!cta_sync_or(s12 != 0)) {
                        iters = t;
                        stopped = true;
                        break;
                    }
                }
            } else {
                __syncthreads();
            }
        }
        // ---- a7: final syndrome when the loop ran to max_iter
        bool ok = stopped;
        if (!stopped) {
            uint32_t synd = 0;
            for (int r = tt; r < mb; r += T) {
                uint32_t rp = 0;
                for (int j = 0; j < WR; ++j) rp ^= (Ls[r * WR + j] >= 0.0f) ? 1u : 0u;
                synd |= rp;
            }
            for (int r = tt; r < NB * mb; r += T) {
                uint32_t rp = 0;
                for (int j = 0; j < WR; ++j)
                    rp ^= (*reinterpret_cast<const float *>(smem + __ldg(lidx + size_t(r) * WR + j)) >= 0.0f) ? 1u : 0u;
                synd |= rp;
            }
            ok = !cta_sync_or(synd != 0);
        }
        // ---- a6/a8: hard decisions (Eq. 8) packed by ballot, flags, posteriors
        const int nw = code.nw;
        uint32_t *bits = a.bits + f * (long long)nw;
        for (int v = tt; v < nw * 32; v += T) {
            const bool z = (v < n) ? (Ls[v] >= 0.0f) : false;
            const uint32_t word = __ballot_sync(0xffffffffu, z);
            if ((tt & 31) == 0) bits[v >> 5] = word;
        }
        if (a.posterior) {
            float *dst = a.posterior + f * (long long)n;
            for (int v = tt; v < n; v += T) dst[v] = Ls[v] * kLn2;
        }
        if (tt == 0) {
            a.syn_ok[f] = ok ? 1 : 0;
            a.iters[f] = iters;
        }
        if constexpr (GEN) {
            // a9 counters of this frame (reading Q14): info-bit errors
            // at perm[0..k), codeword-bit errors, frame error, undetected error
            const uint32_t *c = a.cw + f * (long long)code.nw;
            const uint32_t *m = a.info + f * (long long)code.kw;
            int ie = 0, ce = 0;
            for (int t = tt; t < code.k; t += T) {
                const int v = __ldg(code.perm + t);
                ie += (Ls[v] >= 0.0f) != bool((__ldg(m + (t >> 5)) >> (t & 31)) & 1u);
            }
            for (int v = tt; v < n; v += T) ce += (Ls[v] >= 0.0f) != bool((__ldg(c + (v >> 5)) >> (v & 31)) & 1u);
            ie = __reduce_add_sync(0xffffffffu, ie);
            ce = __reduce_add_sync(0xffffffffu, ce);
            if ((tt & 31) == 0) {
                atomicAdd(&s_err[0], ie);
                atomicAdd(&s_err[1], ce);
            }
            __syncthreads();
            if (tt == 0) {
                cnt[0] += unsigned(s_err[0]);
                cnt[1] += unsigned(s_err[1]);
                cnt[2] += s_err[0] > 0;
                cnt[3] += (ok && s_err[1] > 0);
                cnt[4] += unsigned(iters);
                cnt[5] += 1;
            }
        }
        __syncthreads();
    }
    if (GEN && tt == 0)
        for (int i = 0; i < 6; ++i)
            if (cnt[i]) atomicAdd(a.counters + i, cnt[i]);
    if constexpr (TMIDX) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if ((tt >> 5) == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "n"(TMCOLS) : "memory");
    }
}

