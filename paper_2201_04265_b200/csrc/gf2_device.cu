// gf2_device.cu -- the standard-form generator on the GPU:
// the same Gauss-Jordan elimination as ldpc_make_G (Eq. 2-3; P:329;
// reading Q13: columns scanned right to left, pivot = the lowest row at or
// below the current rank with the column's bit set, eliminated from every
// other row).  The reduced row echelon form is unique, so a correct
// elimination reproduces the host's rank, perm and P bit for bit.
//
// H is bit-packed row-major in the caller's workspace (m rows x W = ceil(n/64)
// uint64 words; C5: 262 MB).  One persistent cooperative kernel walks the n
// columns:
//   * pivot search: every thread scans logical positions >= rank and
//     atomicMin's (position << 32 | physical row) into a slot (two slots
//     alternate so no extra barrier resets them); grid sync;
//   * row swaps are logical: thread 0 swaps two entries of `order`;
//   * elimination: one warp per physical row; a row with the column's bit set
//     XORs the pivot row in with coalesced 8-byte accesses; grid sync.
// A second kernel extracts P (one warp per parity column, ballot-packed along
// the info positions).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "ldpc_internal.h"

namespace cg = cooperative_groups;

namespace ldpc {
namespace {

struct GjArgs {
    uint64_t *M;                    // m x W
    int32_t m, n, W;
    int32_t *order;                 // logical position -> physical row
    int32_t *pivot_row;             // [n]: physical row of column j's pivot, -1 for a free column
    unsigned long long *slot;       // [2] pivot-search slots
    int32_t *rank_out;
};

__global__ void __launch_bounds__(512) gj_kernel(const GjArgs a) {
    cg::grid_group g = cg::this_grid();
    const int64_t gtid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t gthreads = int64_t(gridDim.x) * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = gtid >> 5, gwarps = gthreads >> 5;
    const int W = a.W, m = a.m;
    int rank = 0;
    int parity = 0;
    for (int j = a.n - 1; j >= 0; --j) {
        if (rank >= m) {
            if (gtid == 0) a.pivot_row[j] = -1;
            continue;
        }
        const int w = j >> 6;
        const uint64_t bit = uint64_t(1) << (j & 63);
        unsigned long long *slot = a.slot + parity;
        // pivot search over logical positions [rank, m)
        for (int64_t pos = rank + gtid; pos < m; pos += gthreads) {
            const int r = __ldcg(a.order + pos);
            if (__ldcg(a.M + int64_t(r) * W + w) & bit)
                atomicMin(slot, (static_cast<unsigned long long>(pos) << 32) | unsigned(r));
        }
        __threadfence();
        g.sync();
        const unsigned long long best = __ldcg(slot);
        // the other slot is free again: reset it for the next column
        if (gtid == 0) __stcg(a.slot + (parity ^ 1), ~0ull);
        parity ^= 1;
        if (best == ~0ull) {
            if (gtid == 0) a.pivot_row[j] = -1;
            __threadfence();
            g.sync();               // the reset above must land before the next search
            continue;
        }
        const int p = int(best >> 32), prow = int(best & 0xffffffffu);
        if (gtid == 0) {
            const int rrow = __ldcg(a.order + rank);
            __stcg(a.order + rank, prow);
            __stcg(a.order + p, rrow);
            a.pivot_row[j] = prow;
        }
        // eliminate column j from every other row
        const uint64_t *src = a.M + int64_t(prow) * W;
        for (int64_t r = gwarp; r < m; r += gwarps) {
            if (r == prow) continue;
            uint64_t *dst = a.M + r * W;
            if (!(__ldcg(dst + w) & bit)) continue;          // warp-uniform
            for (int q = lane; q < W; q += 32) __stcg(dst + q, __ldcg(dst + q) ^ __ldcg(src + q));
        }
        ++rank;
        __threadfence();            // every thread's row updates reach L2 before the barrier
        g.sync();
    }
    if (gtid == 0) *a.rank_out = rank;
}

// H (CSR) -> bit-packed rows
__global__ void pack_rows_kernel(const int32_t *row_ptr, const int32_t *col_idx, int m, int W, uint64_t *M) {
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x)
        for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            const int v = col_idx[e];
            M[r * W + (v >> 6)] ^= uint64_t(1) << (v & 63);
        }
}

// P[a][b] = RREF[pivot_row(perm[k+b])][perm[a]], packed as pcols[b][a/32]
__global__ void extract_p_kernel(const uint64_t *M, int W, const int32_t *perm, const int32_t *pivot_row, int k,
                                 int npar, uint32_t *pcols) {
    const int lane = threadIdx.x & 31;
    const int kw = (k + 31) / 32;
    for (int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; b < npar;
         b += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t *row = M + int64_t(pivot_row[perm[k + b]]) * W;
        for (int a0 = 0; a0 < kw * 32; a0 += 32) {
            const int a = a0 + lane;
            bool one = false;
            if (a < k) {
                const int fa = perm[a];
                one = (__ldg(row + (fa >> 6)) >> (fa & 63)) & 1u;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, one);
            if (lane == 0) pcols[b * kw + (a0 >> 5)] = word;
        }
    }
}

size_t align256z(size_t x) { return (x + 255) & ~size_t(255); }

struct GjLayout {
    size_t M, order, pivot, slot, rank, rowp, coli, perm, pcols, total;
};
GjLayout gj_layout(const ldpc_code &c) {
    GjLayout L{};
    const size_t W = (size_t(c.n) + 63) / 64;
    size_t off = 0;
    L.M = off;     off = align256z(off + size_t(c.m) * W * 8);
    L.order = off; off = align256z(off + size_t(std::max(c.m, 1)) * 4);
    L.pivot = off; off = align256z(off + size_t(c.n) * 4);
    L.slot = off;  off = align256z(off + 16);
    L.rank = off;  off = align256z(off + 4);
    L.rowp = off;  off = align256z(off + (size_t(c.m) + 1) * 4);
    L.coli = off;  off = align256z(off + size_t(std::max(c.nnz, 1)) * 4);
    L.perm = off;  off = align256z(off + size_t(c.n) * 4);
    // P: at most (n - 1) parity columns x ceil(n/32) words
    L.pcols = off; off = align256z(off + size_t(c.n) * ((size_t(c.n) + 31) / 32) * 4);
    L.total = off;
    return L;
}

}  // namespace
}  // namespace ldpc

extern "C" {

ldpc_status ldpc_make_G_device_workspace_bytes(const ldpc_code *code, size_t *bytes) {
    if (!code || !bytes) return LDPC_ERR_ARG;
    *bytes = ldpc::gj_layout(*code).total;
    return LDPC_OK;
}

ldpc_status ldpc_make_G_device(ldpc_code *code, void *d_ws, size_t ws_bytes, void *stream) {
    if (!code || !d_ws) return LDPC_ERR_ARG;
    ldpc_code &c = *code;
    const ldpc::GjLayout L = ldpc::gj_layout(c);
    if (ws_bytes < L.total || (reinterpret_cast<uintptr_t>(d_ws) & 255u)) return LDPC_ERR_ARG;
    if (c.m == 0) return ldpc_make_G(code);       // no checks: nothing to eliminate
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char *base = static_cast<char *>(d_ws);
    const int W = (c.n + 63) / 64;
    ldpc::GjArgs a{};
    a.M = reinterpret_cast<uint64_t *>(base + L.M);
    a.m = c.m;
    a.n = c.n;
    a.W = W;
    a.order = reinterpret_cast<int32_t *>(base + L.order);
    a.pivot_row = reinterpret_cast<int32_t *>(base + L.pivot);
    a.slot = reinterpret_cast<unsigned long long *>(base + L.slot);
    a.rank_out = reinterpret_cast<int32_t *>(base + L.rank);
    int32_t *d_rowp = reinterpret_cast<int32_t *>(base + L.rowp);
    int32_t *d_coli = reinterpret_cast<int32_t *>(base + L.coli);
    std::vector<int32_t> order(size_t(c.m));
    for (int32_t i = 0; i < c.m; ++i) order[size_t(i)] = i;
    const unsigned long long init_slot[2] = {~0ull, ~0ull};
    bool ok = cudaMemsetAsync(a.M, 0, size_t(c.m) * size_t(W) * 8, s) == cudaSuccess &&
              cudaMemcpyAsync(a.order, order.data(), order.size() * 4, cudaMemcpyHostToDevice, s) == cudaSuccess &&
              cudaMemcpyAsync(a.slot, init_slot, 16, cudaMemcpyHostToDevice, s) == cudaSuccess &&
              cudaMemcpyAsync(d_rowp, c.row_ptr.data(), c.row_ptr.size() * 4, cudaMemcpyHostToDevice, s) == cudaSuccess &&
              (c.nnz == 0 ||
               cudaMemcpyAsync(d_coli, c.col_idx.data(), c.col_idx.size() * 4, cudaMemcpyHostToDevice, s) == cudaSuccess);
    if (!ok) return LDPC_ERR_CUDA;
    const int sms = ldpc::device_attribute(cudaDevAttrMultiProcessorCount);
    ldpc::pack_rows_kernel<<<std::max(1, std::min(sms * 8, (c.m + 255) / 256)), 256, 0, s>>>(d_rowp, d_coli, c.m, W,
                                                                                             a.M);
    // cooperative launch: every CTA co-resident
    int per_sm = ldpc::occupancy_blocks(reinterpret_cast<const void *>(&ldpc::gj_kernel), 512, 0);
    if (per_sm < 1 || sms < 1) return LDPC_ERR_CUDA;
    int grid = sms * std::min(per_sm, 2);
    if (const char *e = std::getenv("LDPC_GJ_GRID")) grid = std::max(1, std::min(grid, std::atoi(e)));   // debug
    void *args[] = {&a};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(&ldpc::gj_kernel), dim3(unsigned(grid)), dim3(512),
                                    args, 0, s) != cudaSuccess)
        return LDPC_ERR_CUDA;
    std::vector<int32_t> pivot_row(size_t(c.n));
    int32_t rank = 0;
    if (cudaMemcpyAsync(pivot_row.data(), a.pivot_row, size_t(c.n) * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&rank, a.rank_out, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return LDPC_ERR_CUDA;
    if (std::getenv("LDPC_GJ_VERIFY")) {
        // debug: every pivot column must be set in its pivot row only
        std::vector<uint64_t> Mh(size_t(c.m) * size_t(W));
        cudaMemcpy(Mh.data(), a.M, Mh.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int32_t j = c.n - 1; j >= 0 && bad < 5; --j) {
            if (pivot_row[size_t(j)] < 0) continue;
            int cnt = 0;
            for (int32_t r = 0; r < c.m; ++r) cnt += (Mh[size_t(r) * W + size_t(j >> 6)] >> (j & 63)) & 1u;
            if (cnt != 1 || !((Mh[size_t(pivot_row[size_t(j)]) * W + size_t(j >> 6)] >> (j & 63)) & 1u)) {
                std::fprintf(stderr, "gj verify: column %d pivot row %d has %d rows set\n", j, pivot_row[size_t(j)], cnt);
                ++bad;
            }
        }
        std::fprintf(stderr, "gj verify: rank %d, %d bad columns shown\n", rank, bad);
    }
    const int32_t k = c.n - rank;
    if (k == 0) return LDPC_ERR_NO_INFO_BITS;
    // perm = [free columns ascending, pivot columns ascending] (reading Q13)
    std::vector<int32_t> perm(size_t(c.n)), pinv(size_t(c.n));
    {
        int32_t nf = 0, np = 0;
        for (int32_t j = 0; j < c.n; ++j)
            if (pivot_row[size_t(j)] < 0) perm[size_t(nf++)] = j;
        for (int32_t j = 0; j < c.n; ++j)
            if (pivot_row[size_t(j)] >= 0) perm[size_t(k + np++)] = j;
        for (int32_t t = 0; t < c.n; ++t) pinv[size_t(perm[size_t(t)])] = t;
    }
    const int npar = c.n - k, kw = (k + 31) / 32;
    int32_t *d_perm = reinterpret_cast<int32_t *>(base + L.perm);
    uint32_t *d_pcols = reinterpret_cast<uint32_t *>(base + L.pcols);
    std::vector<uint32_t> pcols(size_t(npar) * size_t(kw));
    if (cudaMemcpyAsync(d_perm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, s) != cudaSuccess) return LDPC_ERR_CUDA;
    ldpc::extract_p_kernel<<<std::max(1, std::min(sms * 16, (npar + 7) / 8)), 256, 0, s>>>(a.M, W, d_perm, a.pivot_row,
                                                                                          k, npar, d_pcols);
    if (cudaMemcpyAsync(pcols.data(), d_pcols, pcols.size() * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return LDPC_ERR_CUDA;
    c.perm.swap(perm);
    c.pinv.swap(pinv);
    c.pcols.swap(pcols);
    c.rank = rank;
    c.k = k;
    c.has_G = true;
    c.bound_G = false;
    return LDPC_OK;
}

}  // extern "C"
