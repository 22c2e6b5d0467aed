// spa_decode.cu -- batched Sum-Product (belief propagation) decoding on
// sm_100a.  Paper: Eqs. 4-8, flooding schedule of Alg. 1
// (P:351-369), batch processing.  DESIGN.md §"Kernels" explains
// the mapping; the host entry points are at the bottom (ldpc_decode,
// ldpc_decode_workspace_bytes).
//
// Check-node update in the log domain (Eq. 5 with readings Q2/Q3):
//   x_e  = clamp(L_v - E_cv, +-30)                 (L_vc of Eq. 6, formed lazily)
//   E_cv = (-1)^{d_c} * prod_{e' != e} sgn(x_e') * min(phi(sum_{e' != e} phi(|x_e'|)), E_MAX)
//   phi(x) = -ln tanh(x/2) = ln((1 + e^-x) / (1 - e^-x))   (self-inverse on (0, inf))
// The exclusive sums are prefix + suffix sums (never total-minus-self, which
// loses the small terms next to a large one in fp32).
// Variable-node update (Eq. 7): L_v = R_v + sum_c E_cv; z_v = [L_v >= 0] (Eq. 8).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "ldpc_internal.h"

namespace ldpc {
namespace {

// ---------------------------------------------------------------------------
// phi(x) for x >= 0 in two regimes:
//   x <= 1.25: phi = ln(2/x) + s q(s),  s = x^2      (lg2 on the SFU + 3 FMA)
//   x >  1.25: phi = t h(t^2),          t = e^-x     (ex2 on the SFU + 3 FMA)
// q, h: least-squares fits of (phi - ln(2/x))/x^2 on (0, 1.25] and phi/t on
// [1.25, 30]; max relative error of the formula 1.6e-7, of the fp32
// evaluation <= 1.8e-6 (rounding of x*log2(e) at x -> 30).  Both branches are
// evaluated (2 MUFU per phi, the price the roofline charges) and selected.
constexpr float kPhiSplit = 1.25f;
constexpr float kLn2 = 0.693147180559945309f;
constexpr float kNegLog2e = -1.44269504088896341f;
constexpr float kQ0 = 0.0833325741f, kQ1 = -0.00485671821f, kQ2 = 0.000333309889f, kQ3 = -1.95345602e-05f;
constexpr float kH0 = 2.0f, kH1 = 0.666682958f, kH2 = 0.39854814f, kH3 = 0.319937743f;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float phi(float x) {
    const float s = x * x;
    float q = fmaf(fmaf(fmaf(kQ3, s, kQ2), s, kQ1), s, kQ0);
    const float small = fmaf(s, q, fmaf(lg2_approx(x), -kLn2, kLn2));
    const float t = ex2_approx(x * kNegLog2e);
    const float u = t * t;
    const float h = fmaf(fmaf(fmaf(kH3, u, kH2), u, kH1), u, kH0);
    const float large = t * h;
    return x > kPhiSplit ? large : small;
}

// ---------------------------------------------------------------------------
// Team synchronisation: a team of T threads (T a multiple of 32) decodes one
// frame; several teams share a CTA and sync on named barriers 1..15.
__device__ __forceinline__ void team_sync(int bar_id, int nthreads) {
    if (nthreads == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(nthreads) : "memory");
    }
}
__device__ __forceinline__ bool team_sync_or(int bar_id, int nthreads, bool pred) {
    if (nthreads == 32) return __any_sync(0xffffffffu, pred);
    int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.s32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\t"
        "selp.s32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(int(pred)), "r"(bar_id), "r"(nthreads)
        : "memory");
    return r != 0;
}

// Per-frame decoder state: E[nnz] (padded to 4), L[n], R[n] (padded to 4).
__host__ __device__ __forceinline__ int64_t state_floats(int64_t nnz, int64_t n) {
    return ((nnz + 3) & ~int64_t(3)) + ((2 * n + 3) & ~int64_t(3));
}

struct DecodeArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    int32_t early_term;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
    float *ws;            // global-state variant: per-team E, L, R
    int32_t team_threads;
    int32_t teams_per_cta;
    int64_t ws_stride;    // floats per team in ws
};

// Vector load/store of D consecutive floats / ints starting at a multiple of D.
template <int D>
__device__ __forceinline__ void load_row(const float *p, float (&o)[D]) {
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
__device__ __forceinline__ void store_row(float *p, const float (&o)[D]) {
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4)
            *reinterpret_cast<float4 *>(p + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2) *reinterpret_cast<float2 *>(p + j) = make_float2(o[j], o[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) p[j] = o[j];
    }
}
template <int D>
__device__ __forceinline__ void load_idx(const int32_t *p, int32_t (&o)[D]) {
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

// Check-node phase for one check (Eq. 5).  REG: every check has degree D
// (edge ids c*D .. c*D+D, vectorised); otherwise degree d <= D, edges from
// row_ptr, padded with phi = 0 (exact under + ).  Returns the parity of the
// hard decisions [L_v >= 0] on the check (the syndrome bit of z, Eq. 1).
template <int D, bool REG>
__device__ __forceinline__ uint32_t check_update(const DeviceCode &code, int c, float *E, const float *L) {
    int base, d;
    if constexpr (REG) {
        base = c * D;
        d = D;
    } else {
        base = __ldg(code.row_ptr + c);
        d = __ldg(code.row_ptr + c + 1) - base;
    }
    float e[D];
    int32_t vi[D];
    if constexpr (REG) {
        load_row<D>(E + base, e);
        load_idx<D>(code.col_idx + base, vi);
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            e[j] = (j < d) ? E[base + j] : 0.0f;
            vi[j] = (j < d) ? __ldg(code.col_idx + base + j) : 0;
        }
    }
    float f[D];
    uint32_t sbits = 0, synd = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        if (REG || j < d) {
            const float lv = L[vi[j]];
            const float x = lv - e[j];
            synd ^= (lv >= 0.0f) ? 1u : 0u;
            sbits |= (__float_as_uint(x) >> 31) << j;
            f[j] = phi(fminf(fabsf(x), kLlrClamp));
        } else {
            f[j] = 0.0f;
        }
    }
    // exclusive sums: prefix then suffix (never total - self)
    float ex[D];
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
    const uint32_t par = (__popc(sbits) ^ uint32_t(d)) & 1u;   // (-1)^d * prod of all signs
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const float mag = fminf(phi(ex[j]), kEMax);
        const uint32_t s = ((sbits >> j) ^ par) & 1u;
        e[j] = __uint_as_float(__float_as_uint(mag) | (s << 31));
    }
    if constexpr (REG) {
        store_row<D>(E + base, e);
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (j < d) E[base + j] = e[j];
    }
    return synd;
}

// Syndrome bit of z = [L >= 0] on check c (Eq. 1), no message update.
template <int D, bool REG>
__device__ __forceinline__ uint32_t check_syndrome(const DeviceCode &code, int c, const float *L) {
    int base, d;
    if constexpr (REG) {
        base = c * D;
        d = D;
    } else {
        base = __ldg(code.row_ptr + c);
        d = __ldg(code.row_ptr + c + 1) - base;
    }
    uint32_t s = 0;
    for (int j = 0; j < d; ++j) s ^= (L[__ldg(code.col_idx + base + j)] >= 0.0f) ? 1u : 0u;
    return s;
}

// One team decodes one frame at a time; STATE_SMEM: E, L, R live in shared
// memory (n small enough), else in the global workspace slice of the team.
template <int D, bool REG, bool STATE_SMEM>
__global__ void __launch_bounds__(1024) spa_decode_kernel(const DecodeArgs a) {
    extern __shared__ __align__(16) float smem[];
    const DeviceCode &code = a.code;
    const int T = a.team_threads;
    const int team = threadIdx.x / T;
    const int tt = threadIdx.x - team * T;
    const int bar = team + 1;
    const int n = code.n, m = code.m, nnz = code.nnz;
    const int64_t team_global = int64_t(blockIdx.x) * a.teams_per_cta + team;
    const int64_t nteams = int64_t(gridDim.x) * a.teams_per_cta;
    const int64_t per_team = state_floats(nnz, n);
    float *E, *L, *R;
    if constexpr (STATE_SMEM) {
        E = smem + per_team * team;
    } else {
        E = a.ws + a.ws_stride * team_global;
    }
    L = E + ((nnz + 3) & ~3);
    R = L + n;

    for (int64_t f = team_global; f < a.frames; f += nteams) {
        // a1: LLR ingest (clamped, reading Q7); a2: E = 0, L = R
        const float *src = a.llr + f * int64_t(n);
        if ((n & 3) == 0) {
            for (int v4 = tt; v4 < (n >> 2); v4 += T) {
                float4 r = __ldg(reinterpret_cast<const float4 *>(src) + v4);
                r.x = fminf(fmaxf(r.x, -kLlrClamp), kLlrClamp);
                r.y = fminf(fmaxf(r.y, -kLlrClamp), kLlrClamp);
                r.z = fminf(fmaxf(r.z, -kLlrClamp), kLlrClamp);
                r.w = fminf(fmaxf(r.w, -kLlrClamp), kLlrClamp);
                reinterpret_cast<float4 *>(R)[v4] = r;
                reinterpret_cast<float4 *>(L)[v4] = r;
            }
        } else {
            for (int v = tt; v < n; v += T) {
                float r = fminf(fmaxf(__ldg(src + v), -kLlrClamp), kLlrClamp);
                R[v] = r;
                L[v] = r;
            }
        }
        for (int e = tt; e < nnz; e += T) E[e] = 0.0f;
        team_sync(bar, T);

        int32_t iters = a.max_iter;
        bool stopped = false;
        for (int t = 1; t <= a.max_iter; ++t) {
            // a3: check-node phase (also yields the syndrome of z^{t-1})
            uint32_t synd = 0;
            for (int c = tt; c < m; c += T) synd |= check_update<D, REG>(code, c, E, L);
            if (a.early_term) {
                const bool any = team_sync_or(bar, T, synd != 0);
                if (t > 1 && !any) {        // z^{t-1} is a codeword: stop (reading c6)
                    iters = t - 1;
                    stopped = true;
                    break;
                }
            } else {
                team_sync(bar, T);
            }
            // a4/a5: variable-node phase, total LLR (Eq. 7)
            for (int v = tt; v < n; v += T) {
                float s = R[v];
                int p0, p1;
                if (code.regular_col) {
                    p0 = v * code.max_col_deg;
                    p1 = p0 + code.max_col_deg;
                } else {
                    p0 = __ldg(code.var_ptr + v);
                    p1 = __ldg(code.var_ptr + v + 1);
                }
                for (int q = p0; q < p1; ++q) s += E[__ldg(code.var_edges + q)];
                L[v] = s;
            }
            team_sync(bar, T);
        }
        // a7: final syndrome when the loop ran to max_iter
        bool ok;
        if (stopped) {
            ok = true;
        } else {
            uint32_t synd = 0;
            for (int c = tt; c < m; c += T) synd |= check_syndrome<D, REG>(code, c, L);
            ok = !team_sync_or(bar, T, synd != 0);
        }
        // a6/a8: hard decisions (Eq. 8) packed by warp ballot, flags, posteriors
        const int nw = code.nw;
        uint32_t *bits = a.bits + f * int64_t(nw);
        for (int v = tt; v < nw * 32; v += T) {
            const bool z = (v < n) ? (L[v] >= 0.0f) : false;
            const uint32_t word = __ballot_sync(0xffffffffu, z);
            if ((threadIdx.x & 31) == 0) bits[v >> 5] = word;
        }
        if (a.posterior) {
            float *dst = a.posterior + f * int64_t(n);
            for (int v = tt; v < n; v += T) dst[v] = L[v];
        }
        if (tt == 0) {
            a.syn_ok[f] = ok ? 1 : 0;
            a.iters[f] = iters;
        }
        team_sync(bar, T);   // L/E/R are reused by the next frame
    }
}

__global__ void phi_probe_kernel(const float *x, float *y, int64_t count) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        y[i] = phi(x[i]);
}

// ---------------------------------------------------------------------------
struct Plan {
    int variant;        // 1 = smem team, 2 = global-state CTA
    int D;
    bool reg;
    int team_threads;
    int teams_per_cta;
    size_t smem_bytes;
    int grid;
    size_t ws_bytes;
    int64_t ws_stride;
};

template <int D, bool REG, bool SM>
void *kernel_ptr() {
    return reinterpret_cast<void *>(&spa_decode_kernel<D, REG, SM>);
}

void *select_kernel(int D, bool reg, bool smem) {
#define LDPC_K(DD)                                                                   \
    case DD:                                                                         \
        return reg ? (smem ? kernel_ptr<DD, true, true>() : kernel_ptr<DD, true, false>()) \
                   : (smem ? kernel_ptr<DD, false, true>() : kernel_ptr<DD, false, false>());
    switch (D) {
        LDPC_K(2)
        LDPC_K(3)
        LDPC_K(4)
        LDPC_K(6)
        LDPC_K(8)
        LDPC_K(12)
        LDPC_K(16)
        LDPC_K(32)
    }
#undef LDPC_K
    return nullptr;
}

int degree_bucket(int d, bool reg) {
    if (reg && (d == 2 || d == 3 || d == 4 || d == 6 || d == 8 || d == 12 || d == 16 || d == 32)) return d;
    const int b[] = {2, 4, 6, 8, 12, 16, 32};
    for (int x : b)
        if (d <= x) return x;
    return -1;
}

struct DeviceProps {
    int sms = 0;
    size_t smem_optin = 0;
};
DeviceProps device_props() {
    DeviceProps p;
    p.sms = device_attribute(cudaDevAttrMultiProcessorCount);
    p.smem_optin = size_t(std::max(device_attribute(cudaDevAttrMaxSharedMemoryPerBlockOptin), 0));
    return p;
}

ldpc_status make_plan(const ldpc_code &c, int64_t frames, const ldpc_decode_opts &o, Plan &p) {
    const int dmax = std::max(c.max_row_deg, 1);
    const bool reg = c.regular_row && c.m > 0;
    p.D = degree_bucket(dmax, reg);
    if (p.D < 0) return LDPC_ERR_UNSUPPORTED;
    p.reg = reg && p.D == dmax;
    const DeviceProps dp = device_props();
    if (dp.sms <= 0) return LDPC_ERR_CUDA;
    const int64_t per_team_floats = state_floats(c.nnz, c.n);
    const size_t per_team_bytes = size_t(per_team_floats) * sizeof(float);
    const int work = std::max(c.n, c.m);
    int T = ((work / 4 + 31) / 32) * 32;
    T = std::min(std::max(T, 32), 1024);
    const bool fits = per_team_bytes <= dp.smem_optin;
    int variant = o.variant;
    if (variant == 0) variant = fits ? 1 : 2;
    if (variant == 1 && !fits) return LDPC_ERR_UNSUPPORTED;
    if (variant != 1 && variant != 2) return LDPC_ERR_ARG;
    p.variant = variant;
    void *k = select_kernel(p.D, p.reg, variant == 1);
    if (!k) return LDPC_ERR_UNSUPPORTED;
    if (variant == 1) {
        // teams per CTA: limited by smem, 1024 threads and 15 named barriers
        int teams = int(std::min<size_t>(dp.smem_optin / per_team_bytes, size_t(1024 / T)));
        teams = std::max(1, std::min(teams, 15));
        if (T == 32) teams = std::min(teams, 1024 / 32);
        p.team_threads = T;
        p.teams_per_cta = teams;
        p.smem_bytes = per_team_bytes * size_t(teams);
        if (!ensure_smem_attribute(k, p.smem_bytes)) return LDPC_ERR_CUDA;
        int blocks_per_sm = occupancy_blocks(k, T * teams, p.smem_bytes);
        if (blocks_per_sm < 0) return LDPC_ERR_CUDA;
        blocks_per_sm = std::max(blocks_per_sm, 1);
        const int64_t want = (frames + teams - 1) / teams;
        p.grid = int(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(dp.sms) * blocks_per_sm)));
        p.ws_bytes = 0;
        p.ws_stride = 0;
    } else {
        p.team_threads = 1024;
        p.teams_per_cta = 1;
        p.smem_bytes = 0;
        int blocks_per_sm = occupancy_blocks(k, 1024, 0);
        if (blocks_per_sm < 0) return LDPC_ERR_CUDA;
        blocks_per_sm = std::max(blocks_per_sm, 1);
        p.grid = int(std::max<int64_t>(1, std::min<int64_t>(frames, int64_t(dp.sms) * blocks_per_sm)));
        p.ws_stride = per_team_floats;
        p.ws_bytes = size_t(p.grid) * per_team_bytes;
    }
    return LDPC_OK;
}

}  // namespace
}  // namespace ldpc

namespace ldpc {
namespace {
// The decoder ldpc_decode runs (opts->variant 0 resolved) and its plan.
// Auto order: the Gallager band kernel when a frame fits one SM -- unless the
// batch is too small to fill the GPU one frame per SM and the code has an
// exchange (cluster) view, which then decodes each frame on C SMs for lower
// latency; the exchange cluster kernel for frames larger than one SM (else
// the L2-gather cluster kernel); the generic CSR kernels otherwise.
struct Resolved {
    int variant = 0;
    EdgePlan edge;
    BandPlan band;
    XClusterPlan x;
    GXPlan gx;
    ClusterPlan cl;
    Plan gen;
    // variant 7 with two-frame 16-CTA clusters: the last tail_frames frames run
    // on the global-exchange kernel over the SMs those clusters leave idle,
    // launched as their programmatic dependent (tail_plan)
    GXPlan tail;
    int64_t tail_frames = 0;
};

// Frames for the global-exchange tail next to xband2_kernel's clusters: 16-CTA
// clusters place 7 per B200 (112 SMs), so 36 SMs hold two more 16-CTA groups.
// The split balances the two kernels' rounds of frame pairs: a group decodes a
// pair at `rate` x a cluster's speed (LDPC_XTAIL_RATE; measured on C5 beside
// the clusters: 0.326 ms per cluster round, 0.59 ms per group round, i.e.
// 0.55).  The default sits a little below the balance point: a tail
// that finishes early idles 32 SMs briefly, one that finishes late holds up
// the whole batch.  LDPC_XTAIL=0 turns the tail off.  Only for batches of many
// rounds, where the split's rounding is small.
void tail_plan(const ldpc_code &c, int64_t frames, const ldpc_decode_opts &o, Resolved &r) {
    r.tail_frames = 0;
    const char *env = std::getenv("LDPC_XTAIL");
    if (env && std::atoi(env) == 0) return;
    if (r.x.cluster != 16 || r.x.pairs_capacity() < 1) return;
    const int64_t sms = device_attribute(cudaDevAttrMultiProcessorCount);
    const int idle = int(sms - r.x.pairs_capacity() * r.x.cluster);
    const int groups = idle / 16;
    if (groups < 1) return;
    const double rate = std::getenv("LDPC_XTAIL_RATE") ? std::atof(std::getenv("LDPC_XTAIL_RATE")) : 0.53;
    const int64_t pairs = (frames + 1) / 2;
    const double share = groups * rate / (groups * rate + double(r.x.pairs_capacity()));
    const int64_t min_rounds = 8;
    if (pairs < min_rounds * (r.x.pairs_capacity() + groups)) return;
    int64_t tail_pairs = int64_t(double(pairs) * share / groups + 0.5) * groups;
    if (tail_pairs < groups) return;
    if (!gx_plan(c, 2 * tail_pairs, o.early_term != 0, r.tail, groups)) return;
    r.tail_frames = std::min<int64_t>(2 * tail_pairs, frames - 2);
}

ldpc_status resolve(const ldpc_code &c, int64_t frames, const ldpc_decode_opts &o, Resolved &r) {
    const int v = o.variant;
    const bool et = o.early_term != 0;
    frames = std::max<int64_t>(frames, 1);
    const bool want_band = v == 0 || v == 3 || v == 4 || v == 6;
    const bool band_ok = want_band && band_plan(c, frames, et, v, r.band, o.max_iter);
    if (want_band && v != 0) {
        if (!band_ok) return LDPC_ERR_UNSUPPORTED;
        r.variant = r.band.mode == 2 ? 6 : (r.band.vm ? 4 : 3);
        return LDPC_OK;
    }
    if (v == 8) {
        if (!edge_plan(c, frames, et, o.max_iter, r.edge)) return LDPC_ERR_UNSUPPORTED;
        r.variant = 8;
        return LDPC_OK;
    }
    // No more frames than SMs (stream mode): every frame has an SM to itself
    // under either kernel, and the lane-per-edge kernel (a frame over G x more
    // lanes) finishes it sooner where the band kernel leaves the SM's four
    // schedulers idle (<= 2 warps per frame) or runs long serial chains (>= 64
    // edges per thread and iteration); elsewhere, and with more frames per SM,
    // its extra instructions per edge (padding lanes, shuffles, ballots) cost
    // more than they save (measured).
    const int64_t sms = device_attribute(cudaDevAttrMultiProcessorCount);
    auto edge_small = [&](int64_t band_threads) {
        if (v != 0 || std::getenv("LDPC_NO_EDGE") || frames > sms) return false;
        if (band_threads > 0) {
            const int64_t b0 = (c.dev.mb + band_threads - 1) / band_threads;
            const int64_t chain = int64_t(c.dev.wc) * b0 * c.dev.wr;
            if (band_threads > 64 && chain < 64) return false;
        }
        return edge_plan(c, frames, et, o.max_iter, r.edge);
    };
    const bool x_ok = (v == 0 || v == 7) && xcluster_plan(c, frames, et, r.x);
    if (v == 7) {
        if (!x_ok) return LDPC_ERR_UNSUPPORTED;
        r.variant = 7;
        tail_plan(c, frames, o, r);
        return LDPC_OK;
    }
    if (v == 9) {
        if (!gx_plan(c, frames, et, r.gx)) return LDPC_ERR_UNSUPPORTED;
        r.variant = 9;
        return LDPC_OK;
    }
    if (band_ok) {
        // rounds of the one-SM-per-frame kernel vs rounds of C-SM clusters, a
        // cluster round costing ~2/C of a band round (measured per-SM rate of
        // the exchange kernel is about half the band kernel's)
        // (only while the band kernel leaves SMs idle, frames <= SMs: small
        // latency-view CTAs co-reside many per SM, which this cost model
        // does not price)
        if (x_ok && frames <= sms) {
            const int64_t rb = (frames + r.band.capacity - 1) / r.band.capacity;
            const int64_t rx = (frames + r.x.capacity - 1) / r.x.capacity;
            if (rx * 2 < rb * r.x.cluster) {
                r.variant = 7;
                return LDPC_OK;
            }
        }
        if (edge_small(r.band.threads)) {
            r.variant = 8;
            return LDPC_OK;
        }
        r.variant = r.band.mode == 2 ? 6 : (r.band.vm ? 4 : 3);
        return LDPC_OK;
    }
    if (x_ok) {
        // frames larger than one SM: the global-exchange kernel places 144
        // CTAs where 16-CTA clusters place 112 (LDPC_GX=0/1 overrides)
        const char *gxe = std::getenv("LDPC_GX");
        if (v == 0 && gxe && std::atoi(gxe) == 1 && r.x.capacity >= 2 && gx_plan(c, frames, et, r.gx)) {
            r.variant = 9;
            return LDPC_OK;
        }
        r.variant = 7;
        tail_plan(c, frames, o, r);
        return LDPC_OK;
    }
    if (v == 0 || v == 5) {
        if (cluster_plan(c, frames, et, r.cl)) {
            r.variant = 5;
            return LDPC_OK;
        }
        if (v == 5) return LDPC_ERR_UNSUPPORTED;
    }
    if (edge_small(0)) {
        r.variant = 8;
        return LDPC_OK;
    }
    const ldpc_status s = make_plan(c, frames, o, r.gen);
    if (s != LDPC_OK) return s;
    r.variant = r.gen.variant;
    return LDPC_OK;
}
}  // namespace
}  // namespace ldpc

extern "C" {

ldpc_status ldpc_decode_variant(const ldpc_code *code, int64_t frames, const ldpc_decode_opts *opts,
                                int32_t *variant) {
    if (!code || !opts || !variant || frames < 0) return LDPC_ERR_ARG;
    *variant = 0;
    ldpc::Resolved r;
    const ldpc_status s = ldpc::resolve(*code, frames, *opts, r);
    if (s == LDPC_OK) *variant = r.variant;
    return s;
}

ldpc_status ldpc_decode_workspace_bytes(const ldpc_code *code, int64_t frames, const ldpc_decode_opts *opts,
                                        size_t *bytes) {
    if (!code || !opts || !bytes || frames < 0) return LDPC_ERR_ARG;
    ldpc::Resolved r;
    const ldpc_status s = ldpc::resolve(*code, frames, *opts, r);
    if (s != LDPC_OK) return s;
    switch (r.variant) {
        case 3: case 4: case 6: *bytes = r.band.ws_bytes; break;
        case 7: *bytes = r.tail_frames ? std::max(r.x.ws_bytes, r.tail.ws_bytes) : r.x.ws_bytes; break;
        case 9: *bytes = r.gx.ws_bytes; break;
        case 5: *bytes = r.cl.ws_bytes; break;
        // variant 8 needs none; where the band kernel could decode the code, its
        // workspace is reported so one buffer also serves ldpc_decode_simulate
        case 8: *bytes = r.band.kernel ? r.band.ws_bytes : 0; break;
        default: *bytes = r.gen.ws_bytes; break;
    }
    return LDPC_OK;
}

ldpc_status ldpc_decode(const ldpc_code *code, const float *d_llr, int64_t frames, const ldpc_decode_opts *opts,
                        uint32_t *d_bits, uint8_t *d_syndrome_ok, int32_t *d_iters, float *d_posterior,
                        void *d_ws, size_t ws_bytes, void *stream) {
    if (!code || !opts || frames < 0) return LDPC_ERR_ARG;
    if (!code->d_buf) return LDPC_ERR_STATE;
    if (opts->max_iter < 1) return LDPC_ERR_ARG;
    if (frames == 0) return LDPC_OK;
    if (!d_llr || !d_bits || !d_syndrome_ok || !d_iters) return LDPC_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(d_llr) & 15u) return LDPC_ERR_ARG;
    ldpc::Resolved r;
    const ldpc_status rs = ldpc::resolve(*code, frames, *opts, r);
    if (rs != LDPC_OK) return rs;
    switch (r.variant) {
        case 3: case 4: case 6:
            return ldpc::band_launch(*code, r.band, d_llr, frames, *opts, d_bits, d_syndrome_ok, d_iters, d_posterior,
                                     d_ws, ws_bytes, stream);
        case 7: {
            if (!r.tail_frames)
                return ldpc::xcluster_launch(*code, r.x, d_llr, frames, *opts, d_bits, d_syndrome_ok, d_iters,
                                             d_posterior, d_ws, ws_bytes, stream);
            // frames [0, f1) on the exchange clusters, [f1, frames) on the
            // global-exchange groups beside them (tail_plan); the tail's
            // counters are zeroed first so nothing separates the two launches
            if (r.x.ws_bytes || !d_ws || ws_bytes < r.tail.ws_bytes) return LDPC_ERR_ARG;
            const int64_t f1 = frames - r.tail_frames;
            if (cudaMemsetAsync(d_ws, 0, r.tail.zero_bytes, static_cast<cudaStream_t>(stream)) != cudaSuccess)
                return LDPC_ERR_CUDA;
            const ldpc_status s1 = ldpc::xcluster_launch(*code, r.x, d_llr, f1, *opts, d_bits, d_syndrome_ok, d_iters,
                                                         d_posterior, nullptr, 0, stream);
            if (s1 != LDPC_OK) return s1;
            const int64_t nw = code->dev.nw, n = code->dev.n;
            return ldpc::gx_launch(*code, r.tail, d_llr + f1 * n, r.tail_frames, *opts, d_bits + f1 * nw,
                                   d_syndrome_ok + f1, d_iters + f1, d_posterior ? d_posterior + f1 * n : nullptr,
                                   d_ws, ws_bytes, stream, true);
        }
        case 9:
            return ldpc::gx_launch(*code, r.gx, d_llr, frames, *opts, d_bits, d_syndrome_ok, d_iters, d_posterior,
                                   d_ws, ws_bytes, stream);
        case 8:
            return ldpc::edge_launch(*code, r.edge, d_llr, frames, *opts, d_bits, d_syndrome_ok, d_iters, d_posterior,
                                     stream);
        case 5:
            return ldpc::cluster_launch(*code, r.cl, d_llr, frames, *opts, d_bits, d_syndrome_ok, d_iters,
                                        d_posterior, d_ws, ws_bytes, stream);
        default: break;
    }
    const ldpc::Plan &p = r.gen;
    if (p.ws_bytes > 0 && (!d_ws || ws_bytes < p.ws_bytes)) return LDPC_ERR_ARG;
    ldpc::DecodeArgs a;
    a.code = code->dev;
    a.llr = d_llr;
    a.frames = frames;
    a.max_iter = opts->max_iter;
    a.early_term = opts->early_term ? 1 : 0;
    a.bits = d_bits;
    a.syn_ok = d_syndrome_ok;
    a.iters = d_iters;
    a.posterior = d_posterior;
    a.ws = static_cast<float *>(d_ws);
    a.team_threads = p.team_threads;
    a.teams_per_cta = p.teams_per_cta;
    a.ws_stride = p.ws_stride;
    void *k = ldpc::select_kernel(p.D, p.reg, p.variant == 1);
    void *args[] = {&a};
    cudaError_t e = cudaLaunchKernel(k, dim3(unsigned(p.grid)), dim3(unsigned(p.team_threads * p.teams_per_cta)),
                                     args, p.smem_bytes, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

ldpc_status ldpc_debug_phi(const float *d_x, float *d_y, int64_t count, void *stream) {
    if (count < 0 || (count > 0 && (!d_x || !d_y))) return LDPC_ERR_ARG;
    if (count == 0) return LDPC_OK;
    const int grid = int(std::min<int64_t>((count + 255) / 256, 148 * 32));
    ldpc::phi_probe_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_x, d_y, count);
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // extern "C"
