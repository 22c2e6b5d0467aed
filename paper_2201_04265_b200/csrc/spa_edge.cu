// spa_edge.cu -- lane-per-edge Sum-Product decoder for small batches
// (ldpc_decode variant 8).
//
// Same algorithm, same arithmetic (log2-domain psi, clamps, sign rule) as the
// band decoder (band_kernel.cuh; paper P:120-150 Eqs. 5-7, readings Q2/Q3/Q7
// of DESIGN.md), laid out for the latency-bound regime: a batch too small to
// fill the GPU with one thread per check row (C1, Table I at 1000 frames, one
// frame at a time).  There a frame's time is the length of one warp's
// instruction stream, so the frame is spread thinner:
//   * every check row owns a group of G lanes (G = the power of two >= its
//     degree), one lane per edge; the exclusive sums Sum_{k != j} f_k are a
//     butterfly over the group (sibling, other pair, other quad, ...: log2 G
//     shuffles, never total-minus-self) and the sign product is one ballot;
//   * a thread keeps its KC edge slots (rows g, g + G', ... of its group) --
//     the L offset and the message E_cv -- in registers across iterations;
//     E also goes to shared memory at its CSR edge id for the variable phase;
//   * the variable phase (Eq. 7) is one thread per variable.
// Any code with row degree <= 32 (ldpc_make_H or an external H); one CTA per
// frame, frames strided over the grid.  Shared memory per CTA: E[nnz], L[n],
// R[n] (fp32).
#include "band_common.cuh"
#include "ldpc_internal.h"

#include <algorithm>
#include <cstdlib>

namespace ldpc {
namespace {

using namespace band;

struct EdgeArgs {
    DeviceCode code;
    const float *llr;
    int64_t frames;
    int32_t max_iter;
    uint32_t *bits;
    uint8_t *syn_ok;
    int32_t *iters;
    float *posterior;
};

// Sum of f over the other lanes of this lane's G-lane group (butterfly tree;
// both lanes of a pair form the same sums: + is commutative).
template <int G>
__device__ __forceinline__ float group_exclusive_sum(float f) {
    float ex = __shfl_xor_sync(0xffffffffu, f, 1);
    float acc = f + ex;
#pragma unroll
    for (int s = 2; s < G; s <<= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, acc, s);
        ex += o;
        acc += o;
    }
    return ex;
}

// The band kernel's pairwise tree for rows of degree 6 (band_common.cuh
// check_row<6>: ex_j = f_sibling + (a_lo + a_hi), the two other pairs' sums in
// index order), so that both kernels round alike; padding lanes 6, 7 get an
// unused value.  (For degree 4 the butterfly above is that tree already.)
__device__ __forceinline__ float group_exclusive_sum_tree6(float f, int lane) {
    const float sib = __shfl_xor_sync(0xffffffffu, f, 1);
    const float p = f + sib;
    const int base = lane & ~7, P = (lane & 7) >> 1;
    const int lo = P == 0 ? 1 : 0, hi = P == 2 ? 1 : 2;
    const float qlo = __shfl_sync(0xffffffffu, p, base + 2 * lo);
    const float qhi = __shfl_sync(0xffffffffu, p, base + 2 * hi);
    return sib + (qlo + qhi);
}

// Parity of the ballot bits of this lane's G-lane group.
template <int G>
__device__ __forceinline__ uint32_t group_parity(unsigned ballot, int lane) {
    constexpr unsigned kMask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
    return uint32_t(__popc((ballot >> (lane & ~(G - 1))) & kMask)) & 1u;
}

// TREE6: every row has degree 6 (G = 8) and the sums follow the band tree.
template <int G, int KC, bool VOTE, bool ET, bool TREE6 = false>
__global__ void __launch_bounds__(1024) edge_kernel(const EdgeArgs a) {
    extern __shared__ __align__(16) float smem[];
    const DeviceCode &code = a.code;
    const int n = code.n, m = code.m;
    const int T = int(blockDim.x), tt = int(threadIdx.x), lane = tt & 31;
    const int j = tt & (G - 1), ngroups = T / G, g = tt / G;
    float *E = smem;                                   // [nnz] at CSR edge ids
    float *L = smem + ((code.nnz + 3) & ~3);           // [n]
    float *R = L + ((n + 3) & ~3);                     // [n]

    // this thread's edge slots: row g + k ngroups, element j (frame-independent)
    int32_t eid[KC], vof[KC];
    uint32_t odd = 0;                                  // bit k: row degree odd ((-1)^{d_c})
#pragma unroll
    for (int k = 0; k < KC; ++k) {
        const int r = g + k * ngroups;
        eid[k] = -1;
        vof[k] = 0;
        if (r < m) {
            const int b = __ldg(code.row_ptr + r), d = __ldg(code.row_ptr + r + 1) - b;
            odd |= uint32_t(d & 1) << k;
            if (j < d) {
                eid[k] = b + j;
                vof[k] = __ldg(code.col_idx + b + j);
            }
        }
    }

    for (int64_t f = blockIdx.x; f < a.frames; f += gridDim.x) {
        // a1/a2: R (clamped +-30, log2 units), L = R, E = 0
        const float *src = a.llr + f * (int64_t)n;
        for (int v = tt; v < n; v += T) {
            const float r = fminf(fmaxf(__ldg(src + v), -30.0f), 30.0f) * kL2E;
            R[v] = r;
            L[v] = r;
        }
        float e[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) e[k] = 0.0f;
        __syncthreads();

        int32_t iters = a.max_iter;
        bool stopped = false;
        for (int t = 1; t <= a.max_iter; ++t) {
            // ---- a3: check-node phase, Eq. 5 (and the syndrome of z^{t-1} when ET)
            uint32_t synd = 0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const bool act = eid[k] >= 0;
                const float lv = act ? L[vof[k]] : 0.0f;
                const float x = lv - e[k];
                if (ET) synd |= group_parity<G>(__ballot_sync(0xffffffffu, act && lv >= 0.0f), lane);
                // padding lanes: psi input in the deep-large tier (keeps the
                // warp votes uniform), contribution 0 (exact under +)
                const float ax[1] = {act ? fminf(fabsf(x), kClampB) : kClampB};
                float fo[1];
                psi_row<1, true, VOTE>(ax, fo);
                const float fa = act ? fo[0] : 0.0f;
                const float ex[1] = {TREE6 ? group_exclusive_sum_tree6(fa, lane) : group_exclusive_sum<G>(fa)};
                float go[1];
                psi_row<1, false, VOTE>(ex, go);
                const uint32_t sx = __float_as_uint(x) >> 31;
                const uint32_t par = group_parity<G>(__ballot_sync(0xffffffffu, act && sx), lane) ^ ((odd >> k) & 1u);
                const float mag = fminf(go[0], kEMaxB);
                e[k] = __uint_as_float(__float_as_uint(mag) | ((par ^ sx) << 31));
                if (act) E[eid[k]] = e[k];
            }
            if (ET) {
                const bool any = __syncthreads_or(synd != 0) != 0;
                if (t > 1 && !any) {      // z^{t-1} has zero syndrome: stop (reading c6)
                    iters = t - 1;
                    stopped = true;
                    break;
                }
            } else {
                __syncthreads();
            }
            // ---- a4/a5: variable-node phase, Eq. 7
            for (int v = tt; v < n; v += T) {
                float s = R[v];
                const int b = __ldg(code.var_ptr + v), d = __ldg(code.var_ptr + v + 1) - b;
                for (int i = 0; i < d; ++i) s += E[__ldg(code.var_edges + b + i)];
                L[v] = s;
            }
            __syncthreads();
        }
        // ---- a7: final syndrome when the loop ran to max_iter
        bool ok = stopped;
        if (!stopped) {
            uint32_t synd = 0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const bool act = eid[k] >= 0;
                synd |= group_parity<G>(__ballot_sync(0xffffffffu, act && L[vof[k]] >= 0.0f), lane);
            }
            ok = __syncthreads_or(synd != 0) == 0;
        }
        // ---- a6/a8: hard decisions (Eq. 8) packed by ballot, flags, posteriors
        const int nw = code.nw;
        uint32_t *bits = a.bits + f * (int64_t)nw;
        for (int v = tt; v < nw * 32; v += T) {
            const bool z = (v < n) ? (L[v] >= 0.0f) : false;
            const uint32_t word = __ballot_sync(0xffffffffu, z);
            if (lane == 0) bits[v >> 5] = word;
        }
        if (a.posterior) {
            float *dst = a.posterior + f * (int64_t)n;
            for (int v = tt; v < n; v += T) dst[v] = L[v] * kLn2;
        }
        if (tt == 0) {
            a.syn_ok[f] = ok ? 1 : 0;
            a.iters[f] = iters;
        }
        __syncthreads();
    }
}

template <int G, int KC, bool TREE6>
void *pick_vote(bool vote, bool et) {
    if (et) return reinterpret_cast<void *>(&edge_kernel<G, KC, false, true, TREE6>);
    return vote ? reinterpret_cast<void *>(&edge_kernel<G, KC, true, false, TREE6>)
                : reinterpret_cast<void *>(&edge_kernel<G, KC, false, false, TREE6>);
}
template <int G, bool TREE6 = false>
void *pick_kc(int kc, bool vote, bool et) {
    switch (kc) {
        case 1: return pick_vote<G, 1, TREE6>(vote, et);
        case 2: return pick_vote<G, 2, TREE6>(vote, et);
        case 4: return pick_vote<G, 4, TREE6>(vote, et);
        case 8: return pick_vote<G, 8, TREE6>(vote, et);
        case 16: return pick_vote<G, 16, TREE6>(vote, et);
        default: return nullptr;
    }
}
void *pick_edge_kernel(int G, int kc, bool vote, bool et, bool tree6) {
    switch (G) {
        case 4: return pick_kc<4>(kc, vote, et);
        case 8: return tree6 ? pick_kc<8, true>(kc, vote, et) : pick_kc<8>(kc, vote, et);
        case 16: return pick_kc<16>(kc, vote, et);
        case 32: return pick_kc<32>(kc, vote, et);
        default: return nullptr;
    }
}

}  // namespace

// Plan: G from the largest row degree; threads per frame T = the groups
// needed for KC rows per group, KC the smallest of {1, 2, 4, 8, 16} whose T
// keeps frames x T within the GPU's resident threads (more rows per group
// only lengthen a frame when every frame is resident anyway).  Votes: as the
// band decoder (off under early termination and for <= 20 iterations).
bool edge_plan(const ldpc_code &c, int64_t frames, bool et, int max_iter, EdgePlan &p) {
    const DeviceCode &d = c.dev;
    if (d.m < 1 || d.n < 1 || d.max_row_deg < 1 || d.max_row_deg > 32) return false;
    const int G = d.max_row_deg <= 4 ? 4 : d.max_row_deg <= 8 ? 8 : d.max_row_deg <= 16 ? 16 : 32;
    const size_t smem = 4 * (size_t((d.nnz + 3) & ~3) + 2 * size_t((d.n + 3) & ~3));
    if (smem > 227 * 1024) return false;
    const int sms = device_attribute(cudaDevAttrMultiProcessorCount);
    const int64_t resident = int64_t(std::max(sms, 1)) * 2048;
    const int64_t target = std::max<int64_t>(32, resident / std::max<int64_t>(frames, 1));
    int kc = 0, T = 0;
    for (int k : {1, 2, 4, 8, 16}) {
        const int groups = (d.m + k - 1) / k;
        const int64_t t = (int64_t(groups) * G + 31) / 32 * 32;
        if (t > 1024) continue;
        kc = k;
        T = int(t);
        if (t <= target) break;
    }
    if (!kc) return false;
    const bool vote = !et && max_iter > 20 && !std::getenv("LDPC_EDGE_NOVOTE");
    // rows of degree 6 use the band kernel's sum tree: without votes (ET, or
    // <= 20 iterations) a frame then decodes bit for bit as in the band
    // kernel, whichever of the two a batch size selects
    const bool tree6 = d.regular_row && d.max_row_deg == 6;
    p.kernel = pick_edge_kernel(G, kc, vote, et, tree6);
    if (!p.kernel) return false;
    p.G = G;
    p.kc = kc;
    p.threads = T;
    p.smem = smem;
    if (!ensure_smem_attribute(p.kernel, smem)) return false;
    const int per_sm = occupancy_blocks(p.kernel, T, smem);
    if (per_sm < 1) return false;
    p.capacity = int64_t(per_sm) * sms;
    p.grid = int(std::min<int64_t>(frames, p.capacity));
    return true;
}

ldpc_status edge_launch(const ldpc_code &c, const EdgePlan &p, const float *llr, int64_t frames,
                        const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                        void *stream) {
    EdgeArgs a;
    a.code = c.dev;
    a.llr = llr;
    a.frames = frames;
    a.max_iter = o.max_iter;
    a.bits = bits;
    a.syn_ok = syn;
    a.iters = iters;
    a.posterior = post;
    void *args[] = {&a};
    const cudaError_t e = cudaLaunchKernel(p.kernel, dim3(unsigned(std::max(p.grid, 1))), dim3(unsigned(p.threads)),
                                           args, p.smem, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // namespace ldpc
