// band_common.cuh -- device helpers shared by the Gallager band decoders
// (spa_band.cu: one SM per frame; spa_cluster.cu: one cluster per frame):
// the log2-domain phi (psi), the check-node row update (Eq. 5, P:128-132,
// readings Q2/Q3/Q7 of DESIGN.md) and vectorised row loads/stores.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#ifndef LDPC_SCALAR_PSI
#define LDPC_SCALAR_PSI 0      // 1: psi pairs evaluated with scalar fp32 ops (A/B builds; results identical)
#endif

namespace ldpc {
namespace band {

constexpr float kL2E = 1.44269504088896341f;
constexpr float kLn2 = 0.693147180559945309f;
constexpr float kClampB = 43.2808512f;    // 30 log2(e)            (reading Q7)
constexpr float kEMaxB = 40.86313714f;    // log2(2e12 - 1) = E_MAX log2(e)
// psi(y) = log2(e) phi(y ln2), y >= 0:
//   y <= 1.8033688: psi = C1 - lg2(y) + y^2 q(y^2)     (one lg2)
//   y >  1.8033688: psi = t h(t^2),  t = 2^-y          (one ex2)
constexpr float kSplitB = 1.8033688f;
constexpr float kUltraLargeB = 10.0f;           // psi(y) = h0 2^-y within 3.2e-7 relative
constexpr float kUltraSmallB = 0.0009765625f;   // psi(y) = C1 - lg2(y) within 5e-9 relative
constexpr float kC1 = 1.528766373f;
constexpr float kQ0 = 0.0577617388f, kQ1 = -0.00161740689f, kQ2 = 5.33304814e-05f, kQ3 = -1.50169545e-06f;
constexpr float kH0 = 2.88539008f, kH1 = 0.961820197f, kH2 = 0.574983425f, kH3 = 0.461572595f;

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2a(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float psi(float y) {
    const float s = y * y;
    const float q = fmaf(fmaf(fmaf(kQ3, s, kQ2), s, kQ1), s, kQ0);
    const float small = fmaf(s, q, kC1) - lg2a(y);
    const float t = ex2a(-y);
    const float u = t * t;
    const float h = fmaf(fmaf(fmaf(kH3, u, kH2), u, kH1), u, kH0);
    const float large = t * h;
    return y > kSplitB ? large : small;
}
__device__ __forceinline__ float psi_small(float y) {
    const float s = y * y;
    const float q = fmaf(fmaf(fmaf(kQ3, s, kQ2), s, kQ1), s, kQ0);
    return fmaf(s, q, kC1) - lg2a(y);
}
__device__ __forceinline__ float psi_large(float y) {
    const float t = ex2a(-y);
    const float u = t * t;
    return t * fmaf(fmaf(fmaf(kH3, u, kH2), u, kH1), u, kH0);
}
// Deep-converged tiers (psi_row's votes take them only when the whole warp's
// inputs lie in their domain): y >= kUltraLargeB -> h0 2^-y (dropped terms
// <= 3.2e-7 relative); y <= kUltraSmallB -> C1 - lg2 y (dropped term
// <= 5.5e-8 against psi >= 11.5).  One SFU op and one FMA-pipe op each.
__device__ __forceinline__ float psi_deep_large(float y) { return kH0 * ex2a(-y); }
__device__ __forceinline__ float psi_deep_small(float y) { return kC1 - lg2a(y); }

// ---------------------------------------------------------------------------
// Packed evaluation (sm_100a FFMA2 / FMUL2 / FADD2: two fp32 lanes per
// instruction).  The decoders are issue-bound (profiles/issue.json), and psi's
// polynomial arithmetic is most of a non-converged row's instructions; a row's
// elements are evaluated in pairs with the .f32x2 forms of exactly the scalar
// operations above (same operands, same order, .rn each), so every element's
// result is bit-identical to psi / psi_small / psi_large / psi_deep_* -- only
// the issue count halves.  The MUFU ops and the regime select stay scalar.
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_splat(float c) { return f2_pack(c, c); }
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
    f2_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

enum PsiTier { kPsiFull = 0, kPsiSmall, kPsiLarge, kPsiDeepLarge, kPsiDeepSmall };

// small regime of a pair: fmaf(s, q(s), C1) - lg2(y), s = y^2
__device__ __forceinline__ f2_t psi2_small(f2_t y, float y0, float y1) {
    const f2_t s = f2_mul(y, y);
    const f2_t q = f2_fma(f2_fma(f2_fma(f2_splat(kQ3), s, f2_splat(kQ2)), s, f2_splat(kQ1)), s, f2_splat(kQ0));
    return f2_sub(f2_fma(s, q, f2_splat(kC1)), f2_pack(lg2a(y0), lg2a(y1)));
}
// large regime of a pair: t h(t^2), t = 2^-y
__device__ __forceinline__ f2_t psi2_large(float y0, float y1) {
    const f2_t t = f2_pack(ex2a(-y0), ex2a(-y1));
    const f2_t u = f2_mul(t, t);
    return f2_mul(t, f2_fma(f2_fma(f2_fma(f2_splat(kH3), u, f2_splat(kH2)), u, f2_splat(kH1)), u, f2_splat(kH0)));
}
template <int TIER>
__device__ __forceinline__ float psi1(float y) {
    if constexpr (TIER == kPsiFull) return psi(y);
    else if constexpr (TIER == kPsiSmall) return psi_small(y);
    else if constexpr (TIER == kPsiLarge) return psi_large(y);
    else if constexpr (TIER == kPsiDeepLarge) return psi_deep_large(y);
    else return psi_deep_small(y);
}
template <int TIER>
__device__ __forceinline__ void psi2(float y0, float y1, float &o0, float &o1) {
    const f2_t y = f2_pack(y0, y1);
    if constexpr (TIER == kPsiFull) {
        float s0, s1, l0, l1;
        f2_unpack(psi2_small(y, y0, y1), s0, s1);
        f2_unpack(psi2_large(y0, y1), l0, l1);
        o0 = y0 > kSplitB ? l0 : s0;
        o1 = y1 > kSplitB ? l1 : s1;
    } else if constexpr (TIER == kPsiSmall) {
        f2_unpack(psi2_small(y, y0, y1), o0, o1);
    } else if constexpr (TIER == kPsiLarge) {
        f2_unpack(psi2_large(y0, y1), o0, o1);
    } else if constexpr (TIER == kPsiDeepLarge) {
        f2_unpack(f2_mul(f2_splat(kH0), f2_pack(ex2a(-y0), ex2a(-y1))), o0, o1);
    } else {
        f2_unpack(f2_sub(f2_splat(kC1), f2_pack(lg2a(y0), lg2a(y1))), o0, o1);
    }
}
// one tier over a row: pairs packed, an odd last element scalar
template <int D, int TIER>
__device__ __forceinline__ void psi_eval(const float (&in)[D], float (&out)[D]) {
#if LDPC_SCALAR_PSI
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = psi1<TIER>(in[j]);
#else
#pragma unroll
    for (int j = 0; j + 1 < D; j += 2) psi2<TIER>(in[j], in[j + 1], out[j], out[j + 1]);
    if constexpr (D & 1) out[D - 1] = psi1<TIER>(in[D - 1]);
#endif
}

// psi over a row.  When every input of every active lane of the warp falls in
// one regime -- the common case once a frame has converged: |L_vc| large
// (first psi), exclusive sums tiny (second psi) -- only that regime is
// evaluated (one SFU op and 5 FMA-pipe ops instead of two and 11).
// LARGE_FIRST orders the two warp votes by the expected regime.  VOTE is off
// under early termination: a frame stops as soon as it converges, so the
// uniform regime never lasts and the votes would be pure overhead.
template <int D, bool LARGE_FIRST, bool VOTE>
__device__ __forceinline__ bool psi_row(const float (&in)[D], float (&out)[D]) {
    if (!VOTE) {
        psi_eval<D, kPsiFull>(in, out);
        return false;
    }
    const unsigned act = __activemask();
    float lo = in[0], hi = in[0];
#pragma unroll
    for (int j = 1; j < D; ++j) {
        if (LARGE_FIRST) lo = fminf(lo, in[j]);
        else hi = fmaxf(hi, in[j]);
    }
    // deep-converged tiers (psi_deep_large / psi_deep_small)
    if (LARGE_FIRST ? __all_sync(act, lo >= kUltraLargeB) : __all_sync(act, hi <= kUltraSmallB)) {
        psi_eval<D, LARGE_FIRST ? kPsiDeepLarge : kPsiDeepSmall>(in, out);
        return true;
    }
    if (LARGE_FIRST ? __all_sync(act, lo > kSplitB) : __all_sync(act, hi <= kSplitB)) {
        psi_eval<D, LARGE_FIRST ? kPsiLarge : kPsiSmall>(in, out);
        return true;
    }
#pragma unroll
    for (int j = 1; j < D; ++j) {
        if (LARGE_FIRST) hi = fmaxf(hi, in[j]);
        else lo = fminf(lo, in[j]);
    }
    if (LARGE_FIRST ? __all_sync(act, hi <= kSplitB) : __all_sync(act, lo > kSplitB)) {
        psi_eval<D, LARGE_FIRST ? kPsiSmall : kPsiLarge>(in, out);
        return true;
    }
    psi_eval<D, kPsiFull>(in, out);
    return false;
}

// Exclusive sums Phi_j = sum_{k != j} f_k of positive terms: never
// total-minus-self (inf - inf, cancellation); a pairwise tree for D = 4, 6
// (fewer adds, shorter chains; measured +1-2 points on C3/C4), prefix +
// suffix otherwise (a tree for D = 12 measured -0.6 on C3-R3/4).
template <int D>
__device__ __forceinline__ void exclusive_sums(const float (&f)[D], float (&ex)[D]) {
#if !LDPC_SCALAR_PSI
    // the same sums, pairs of outputs on the packed pipe (each element's
    // operands and order unchanged: bit-identical)
    if constexpr (D == 6) {
        const float a01 = f[0] + f[1], a23 = f[2] + f[3], a45 = f[4] + f[5];
        float o01, o23;
        f2_unpack(f2_add(f2_pack(a23, a01), f2_splat(a45)), o01, o23);
        const float o45 = a01 + a23;
        f2_unpack(f2_add(f2_pack(f[1], f[0]), f2_splat(o01)), ex[0], ex[1]);
        f2_unpack(f2_add(f2_pack(f[3], f[2]), f2_splat(o23)), ex[2], ex[3]);
        f2_unpack(f2_add(f2_pack(f[5], f[4]), f2_splat(o45)), ex[4], ex[5]);
        return;
    } else if constexpr (D == 4) {
        const float a01 = f[0] + f[1], a23 = f[2] + f[3];
        f2_unpack(f2_add(f2_pack(f[1], f[0]), f2_splat(a23)), ex[0], ex[1]);
        f2_unpack(f2_add(f2_pack(f[3], f[2]), f2_splat(a01)), ex[2], ex[3]);
        return;
    }
#endif
    if constexpr (D == 6) {
        const float a01 = f[0] + f[1], a23 = f[2] + f[3], a45 = f[4] + f[5];
        const float o01 = a23 + a45, o23 = a01 + a45, o45 = a01 + a23;
        ex[0] = f[1] + o01; ex[1] = f[0] + o01;
        ex[2] = f[3] + o23; ex[3] = f[2] + o23;
        ex[4] = f[5] + o45; ex[5] = f[4] + o45;
    } else if constexpr (D == 4) {
        const float a01 = f[0] + f[1], a23 = f[2] + f[3];
        ex[0] = f[1] + a23; ex[1] = f[0] + a23;
        ex[2] = f[3] + a01; ex[3] = f[2] + a01;
    } else {
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            ex[j] = acc;
            acc += f[j];
        }
        acc = 0.0f;
#pragma unroll
        for (int j = D - 1; j >= 0; --j) {
            ex[j] += acc;
            acc += f[j];
        }
    }
}

// Saturation bound of a degree-D row: when every |L'_vc| of the row is >= it,
// E'_cv = +-E_MAX for every edge, whichever psi tier would evaluate it: each
// term is psi(y) = h0 2^-y (1 + O(2^-2y)) in every tier (relative excess
// < 1e-25 at y >= 42), so every exclusive sum is <= (D-1) h0 2^-y_sat, and
// its psi, >= C1 - lg2(sum) in every tier, is >= E_MAX + 0.02 -- a margin far
// above the approx instructions' ~1e-6 error, so the clamp min(psi, E_MAX)
// returns E_MAX bit for bit.  Reachable only below the input clamp: D <= 6
// (y_sat = 43.205 for D = 6, 42.468 for D = 4; the clamp is 43.281).
template <int D>
__host__ __device__ constexpr float sat_bound() {
    // log2((D-1) h0) for D = 2..7 (h0 = 2.88539008 = 2 log2 e)
    return D == 2 ? 40.863137f - 1.528766f + 1.528766f + 0.02f
         : D == 3 ? 40.863137f - 1.528766f + 2.528766f + 0.02f
         : D == 4 ? 40.863137f - 1.528766f + 3.113729f + 0.02f
         : D == 5 ? 40.863137f - 1.528766f + 3.528766f + 0.02f
         : D == 6 ? 40.863137f - 1.528766f + 3.850694f + 0.02f
                  : 1e30f;
}

// Check-node update of one row (Eq. 5, readings Q2/Q3/Q7) in log2 units.
// x[j] = L'_v - E'_cv (not yet clamped); e[j] <- new E'_cv.
// Rows too wide to saturate (sat_bound > clamp, D >= 7) still reach a fixed
// output once every input sits at the clamp: with the whole warp there, the
// votes take the deep tiers, and E_j = +-M_j with M_j a constant of the
// kernel -- clamp_row_mags computes it once per CTA through the very same
// code (psi_row deep tiers, exclusive_sums), so the shortcut is bit-exact.
template <int D>
__device__ __forceinline__ void clamp_row_mags(float (&m)[D]) {
    float ax[D], f[D], ex[D], g[D];
#pragma unroll
    for (int j = 0; j < D; ++j) ax[j] = kClampB;
    psi_row<D, true, true>(ax, f);
    exclusive_sums<D>(f, ex);
    psi_row<D, false, true>(ex, g);
#pragma unroll
    for (int j = 0; j < D; ++j) m[j] = fminf(g[j], kEMaxB);
}
template <int D>
__host__ __device__ constexpr bool has_clamp_tier() { return sat_bound<D>() > kClampB; }

// cm: the row's clamp magnitudes (clamp_row_mags, shared memory; used when
// has_clamp_tier<D>() and VOTE; may be null otherwise).
template <int D, bool VOTE>
__device__ __forceinline__ bool check_row(const float (&x)[D], float (&e)[D], const float *cm = nullptr) {
    float f[D];
    uint32_t sx = (D & 1) ? 0x80000000u : 0u;     // (-1)^{d_c}
#pragma unroll
    for (int j = 0; j < D; ++j) sx ^= __float_as_uint(x[j]);
    // min_j |x_j| decides both shortcut tiers before the clamped inputs are
    // formed (both bounds are <= the clamp, so min |x| >= b <=> min
    // min(|x|, clamp) >= b: the same decisions)
    float lo_abs = fabsf(x[0]);
    if constexpr (VOTE && (sat_bound<D>() <= kClampB || has_clamp_tier<D>())) {
#pragma unroll
        for (int j = 1; j < D; ++j) lo_abs = fminf(lo_abs, fabsf(x[j]));
    }
    if constexpr (VOTE && sat_bound<D>() <= kClampB) {
        // saturated rows (every input at the clamp: a converged frame under
        // fixed iterations): E = +-E_MAX exactly as the full update gives it
        if (__all_sync(__activemask(), lo_abs >= sat_bound<D>())) {
            // sign(e_j) = sign(sx) ^ sign(x_j), magnitude E_MAX: with t =
            // sign(sx) | E_MAX once per row, one 3-input LOP3 per element
            const uint32_t tsat = (sx & 0x80000000u) | __float_as_uint(kEMaxB);
#pragma unroll
            for (int j = 0; j < D; ++j) e[j] = __uint_as_float((__float_as_uint(x[j]) & 0x80000000u) ^ tsat);
            return true;
        }
    }
    if constexpr (VOTE && has_clamp_tier<D>()) {
        if (cm && __all_sync(__activemask(), lo_abs >= kClampB)) {
            const uint32_t sxm = sx & 0x80000000u;
#pragma unroll
            for (int j = 0; j < D; ++j)
                e[j] = __uint_as_float(__float_as_uint(cm[j]) | ((__float_as_uint(x[j]) & 0x80000000u) ^ sxm));
            return true;
        }
    }
    float ax[D];
#pragma unroll
    for (int j = 0; j < D; ++j) ax[j] = fminf(fabsf(x[j]), kClampB);
    bool hit = psi_row<D, true, VOTE>(ax, f);
    float ex[D];
    exclusive_sums<D>(f, ex);
    float g[D];
    hit |= psi_row<D, false, VOTE>(ex, g);
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const float mag = fminf(g[j], kEMaxB);
        const uint32_t sgn = (sx ^ __float_as_uint(x[j])) & 0x80000000u;
        e[j] = __uint_as_float(__float_as_uint(mag) | sgn);
    }
    return hit;
}

// Adaptive votes (kernels whose frames stay unconverged for long stretches,
// e.g. C5 at 1.2 dB): vote_now (warp-uniform) selects the voted update
// (tiers; returns whether one was taken) or the plain two-regime one, whose
// vote instructions would be pure overhead on rows that straddle regimes.
// Both are Eq. 5 within the psi error budget (tests/test_gpu_psi.py).
template <int D>
__device__ __forceinline__ bool check_row_gated(const float (&x)[D], float (&e)[D], bool vote_now,
                                                const float *cm = nullptr) {
    if (vote_now) return check_row<D, true>(x, e, cm);
    check_row<D, false>(x, e);
    return false;
}

// check_row split over a lane pair (band_kernel LPR = 2): lane h = lane & 1
// holds elements [h D/2, (h+1) D/2) of the row (x, e of D/2 entries); its
// partner is lane ^ 1 of the same warp.  The exclusive sums reproduce
// check_row's association exactly (pairwise tree for D = 4, 6; prefix and
// suffix otherwise, each half continuing the other's running sum), so
// without psi votes a row decodes bit for bit as in check_row.
// pm: the warp's lanes running this call (both lanes of every pair).
template <int D, bool VOTE>
__device__ __forceinline__ void check_row_pair(const float (&x)[D / 2], float (&e)[D / 2], int h, unsigned pm) {
    constexpr int W = D / 2;
    static_assert(D % 2 == 0, "lane pairs split even degrees");
    float f[W], ax[W];
    uint32_t sl = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) {
        sl ^= __float_as_uint(x[j]);
        ax[j] = fminf(fabsf(x[j]), kClampB);
    }
    const uint32_t sx = sl ^ __shfl_xor_sync(pm, sl, 1) ^ ((D & 1) ? 0x80000000u : 0u);
    if constexpr (VOTE && sat_bound<D>() <= kClampB) {
        float lo = ax[0];
#pragma unroll
        for (int j = 1; j < W; ++j) lo = fminf(lo, ax[j]);
        if (__all_sync(__activemask(), lo >= sat_bound<D>())) {
            const uint32_t tsat = (sx & 0x80000000u) | __float_as_uint(kEMaxB);
#pragma unroll
            for (int j = 0; j < W; ++j) e[j] = __uint_as_float((__float_as_uint(x[j]) & 0x80000000u) ^ tsat);
            return;
        }
    }
    psi_row<W, true, VOTE>(ax, f);
    float ex[W];
    if constexpr (D == 6) {
        // half 0: f0 f1 f2, half 1: f3 f4 f5; a01 + a45 etc. as check_row<6>
        const float mine = h ? f[0] : f[2];                        // f3 / f2
        const float other = __shfl_xor_sync(pm, mine, 1);  // f2 / f3
        const float pr = h ? f[1] + f[2] : f[0] + f[1];             // a45 / a01
        const float opr = __shfl_xor_sync(pm, pr, 1);      // a01 / a45
        const float a23 = h ? other + f[0] : f[2] + other;          // f2 + f3
        if (h == 0) {
            const float o01 = a23 + opr;      // a23 + a45
            const float o23 = pr + opr;       // a01 + a45
            ex[0] = f[1] + o01;
            ex[1] = f[0] + o01;
            ex[2] = other + o23;              // f3 + o23
        } else {
            const float o23 = opr + pr;       // a01 + a45
            const float o45 = opr + a23;      // a01 + a23
            ex[0] = other + o23;              // f2 + o23
            ex[1] = f[2] + o45;               // f5 + o45
            ex[2] = f[1] + o45;               // f4 + o45
        }
    } else if constexpr (D == 4) {
        const float pr = f[0] + f[1];
        const float opr = __shfl_xor_sync(pm, pr, 1);
        ex[0] = f[1] + opr;
        ex[1] = f[0] + opr;
    } else {
        // forward sum of half 0 and backward sum of half 1, exchanged
        float fw = 0.0f, bw = 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) fw += f[j];
#pragma unroll
        for (int j = W - 1; j >= 0; --j) bw += f[j];
        const float got = __shfl_xor_sync(pm, h ? bw : fw, 1);
        float acc = h ? got : 0.0f;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            ex[j] = acc;
            acc += f[j];
        }
        acc = h ? 0.0f : got;
#pragma unroll
        for (int j = W - 1; j >= 0; --j) {
            ex[j] += acc;
            acc += f[j];
        }
    }
    float g[W];
    psi_row<W, false, VOTE>(ex, g);
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const float mag = fminf(g[j], kEMaxB);
        const uint32_t sgn = (sx ^ __float_as_uint(x[j])) & 0x80000000u;
        e[j] = __uint_as_float(__float_as_uint(mag) | sgn);
    }
}

// One row's update by one lane (LPR = 1) or a lane pair (LPR = 2).
template <int D, bool VOTE, int LPR>
__device__ __forceinline__ void check_any(const float (&x)[D / LPR], float (&e)[D / LPR], int h, unsigned pm,
                                          const float *cm = nullptr) {
    if constexpr (LPR == 1) {
        check_row<D, VOTE>(x, e, cm);
    } else {
        check_row_pair<D, VOTE>(x, e, h, pm);
    }
}

// Tensor Memory as per-thread storage (32x32b shapes: lane i of the warp
// reads / writes TMEM lane (lane base + i); N consecutive columns).
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t a, const uint32_t (&v)[N]) {
    static_assert(N == 2 || N == 4 || N == 8 || N == 16, "tcgen05.st shapes used here");
    if constexpr (N == 2) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(v[0]), "r"(v[1]) : "memory");
    } else if constexpr (N == 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v[0]), "r"(v[1]),
                     "r"(v[2]), "r"(v[3])
                     : "memory");
    } else if constexpr (N == 8) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(a), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16};" ::"r"(a),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
            "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
    }
}
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t a, uint32_t (&v)[N]) {
    static_assert(N == 2 || N == 4 || N == 8 || N == 16, "tcgen05.ld shapes used here");
    if constexpr (N == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(a) : "memory");
    } else if constexpr (N == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(a)
                     : "memory");
    } else if constexpr (N == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(a)
                     : "memory");
    } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(a)
            : "memory");
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
constexpr int pow2_at_least(int x) { return x <= 2 ? 2 : x <= 4 ? 4 : x <= 8 ? 8 : x <= 16 ? 16 : x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : x <= 256 ? 256 : 512; }

template <int D>
__device__ __forceinline__ void lds_row(const char *smem, uint32_t byte_off, float (&o)[D]) {
    const float *p = reinterpret_cast<const float *>(smem + byte_off);
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4) {
            float4 t = *reinterpret_cast<const float4 *>(p + j);
            o[j] = t.x; o[j + 1] = t.y; o[j + 2] = t.z; o[j + 3] = t.w;
        }
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2) {
            float2 t = *reinterpret_cast<const float2 *>(p + j);
            o[j] = t.x; o[j + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) o[j] = p[j];
    }
}
template <int D>
__device__ __forceinline__ void sts_row(char *smem, uint32_t byte_off, const float (&o)[D]) {
    float *p = reinterpret_cast<float *>(smem + byte_off);
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4) *reinterpret_cast<float4 *>(p + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2) *reinterpret_cast<float2 *>(p + j) = make_float2(o[j], o[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = o[j];
    }
}
template <int D>
__device__ __forceinline__ void ldg_idx(const int32_t *p, int32_t (&o)[D]) {
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4) {
            int4 t = __ldg(reinterpret_cast<const int4 *>(p + j));
            o[j] = t.x; o[j + 1] = t.y; o[j + 2] = t.z; o[j + 3] = t.w;
        }
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2) {
            int2 t = __ldg(reinterpret_cast<const int2 *>(p + j));
            o[j] = t.x; o[j + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) o[j] = __ldg(p + j);
    }
}

}  // namespace band
}  // namespace ldpc
