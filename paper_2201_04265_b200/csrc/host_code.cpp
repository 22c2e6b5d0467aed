// host_code.cpp -- host side of the C ABI: code construction (Gallager H,
// external CSR), standard-form generator (GF(2) Gauss-Jordan), queries, the
// device image, and the frame partition.  Independent of oracle/ (shares no
// code with it); bit-exactness with it is asserted by tests/test_host_vs_oracle.py.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <thread>
#include <string>
#include <vector>

#include "ldpc_internal.h"

namespace {

// ---------------------------------------------------------------------------
// SplitMix64 (Steele/Lea/Flood 2014) and an unbiased bounded draw by
// rejection: r is rejected when r >= 2^64 - (2^64 mod s) (reading Q12).
struct SplitMix64 {
    uint64_t s;
    explicit SplitMix64(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t bound) {
        const uint64_t rem = (~bound + 1) % bound;          // 2^64 mod bound
        const uint64_t limit = ~rem + 1;                     // 2^64 - rem (0 when rem == 0)
        for (;;) {
            uint64_t r = next();
            if (rem == 0 || r < limit) return r % bound;
        }
    }
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

void build_csc(ldpc_code &c) {
    c.var_ptr.assign(size_t(c.n) + 1, 0);
    for (int32_t e = 0; e < c.nnz; ++e) c.var_ptr[size_t(c.col_idx[e]) + 1]++;
    for (int32_t v = 0; v < c.n; ++v) c.var_ptr[size_t(v) + 1] += c.var_ptr[v];
    c.var_edges.assign(size_t(c.nnz), 0);
    std::vector<int32_t> cursor(c.var_ptr.begin(), c.var_ptr.end() - 1);
    for (int32_t chk = 0; chk < c.m; ++chk)            // ascending check order per variable
        for (int32_t e = c.row_ptr[chk]; e < c.row_ptr[chk + 1]; ++e)
            c.var_edges[size_t(cursor[c.col_idx[e]]++)] = e;
    c.max_row_deg = 0;
    int32_t min_row = c.m ? INT32_MAX : 0;
    for (int32_t chk = 0; chk < c.m; ++chk) {
        int32_t d = c.row_ptr[chk + 1] - c.row_ptr[chk];
        c.max_row_deg = std::max(c.max_row_deg, d);
        min_row = std::min(min_row, d);
    }
    c.max_col_deg = 0;
    int32_t min_col = c.n ? INT32_MAX : 0;
    for (int32_t v = 0; v < c.n; ++v) {
        int32_t d = c.var_ptr[v + 1] - c.var_ptr[v];
        c.max_col_deg = std::max(c.max_col_deg, d);
        min_col = std::min(min_col, d);
    }
    c.regular_row = (min_row == c.max_row_deg);
    c.regular_col = (min_col == c.max_col_deg);
}

unsigned worker_count() {
    unsigned h = std::thread::hardware_concurrency();
    return std::max(1u, std::min(h ? h : 1u, 64u));
}

}  // namespace

namespace ldpc {
namespace {
std::mutex g_launch_mu;
std::map<std::pair<int, int>, int> g_dev_attr;                                   // (device, attr)
std::map<std::pair<int, const void *>, size_t> g_smem_attr;                       // (device, kernel)
std::map<std::tuple<int, const void *, int, size_t, int>, int> g_occupancy;      // (device, kernel, T, smem, C)
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
}  // namespace

int device_attribute(int attr) {
    const int d = current_device();
    std::lock_guard<std::mutex> lk(g_launch_mu);
    auto it = g_dev_attr.find({d, attr});
    if (it != g_dev_attr.end()) return it->second;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, static_cast<cudaDeviceAttr>(attr), d) != cudaSuccess) return -1;
    g_dev_attr[{d, attr}] = v;
    return v;
}

bool ensure_smem_attribute(const void *kernel, size_t smem, bool nonportable_cluster) {
    const int d = current_device();
    std::lock_guard<std::mutex> lk(g_launch_mu);
    size_t &have = g_smem_attr[{d, kernel}];
    if (have >= smem && have > 0) return true;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(std::max(smem, have))) !=
        cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (nonportable_cluster && cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                                   cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    have = std::max(smem, std::max<size_t>(have, 1));
    return true;
}

int occupancy_blocks(const void *kernel, int threads, size_t smem) {
    const int d = current_device();
    {
        std::lock_guard<std::mutex> lk(g_launch_mu);
        auto it = g_occupancy.find({d, kernel, threads, smem, 0});
        if (it != g_occupancy.end()) return it->second;
    }
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::lock_guard<std::mutex> lk(g_launch_mu);
    g_occupancy[{d, kernel, threads, smem, 0}] = v;
    return v;
}

int occupancy_clusters(const void *kernel, int threads, size_t smem, int cluster) {
    const int d = current_device();
    {
        std::lock_guard<std::mutex> lk(g_launch_mu);
        auto it = g_occupancy.find({d, kernel, threads, smem, cluster});
        if (it != g_occupancy.end()) return it->second;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(cluster));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int v = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&v, kernel, &cfg);
    if (e != cudaSuccess) {
        if (std::getenv("LDPC_DEBUG"))
            std::fprintf(stderr, "ldpc occupancy_clusters: %s (C=%d, threads %d, smem %zu)\n", cudaGetErrorString(e),
                         cluster, threads, smem);
        cudaGetLastError();
        return -1;
    }
    std::lock_guard<std::mutex> lk(g_launch_mu);
    g_occupancy[{d, kernel, threads, smem, cluster}] = v;
    return v;
}

DeviceLayout compute_layout(const ldpc_code &c, bool with_G) {
    DeviceLayout L;
    size_t off = 0;
    L.row_ptr = off;   off = align256(off + sizeof(int32_t) * (size_t(c.m) + 1));
    L.col_idx = off;   off = align256(off + sizeof(int32_t) * size_t(std::max(c.nnz, 1)));
    L.var_ptr = off;   off = align256(off + sizeof(int32_t) * (size_t(c.n) + 1));
    L.var_edges = off; off = align256(off + sizeof(int32_t) * size_t(std::max(c.nnz, 1)));
    if (c.gallager && c.wc >= 2) {
        const size_t nb = size_t(c.wc - 1) * size_t(c.n);
        L.band_lidx = off; off = align256(off + sizeof(int32_t) * nb);
        L.band_vpos = off; off = align256(off + sizeof(int32_t) * nb);
        if (c.n <= 16383) {
            L.band_lidx16 = off; off = align256(off + sizeof(uint16_t) * nb);
        }
        if (band_cluster_size(c.n, c.wc, c.wr) > 0) {
            L.cband_lidx = off; off = align256(off + sizeof(int32_t) * nb);
            L.cband_vpos = off; off = align256(off + sizeof(int32_t) * nb);
        }
        if (const int C = xband_cluster_size(c.n, c.wc, c.wr)) {
            L.xband_ridx = off; off = align256(off + sizeof(uint16_t) * nb);
            L.xband_sidx = off; off = align256(off + sizeof(uint16_t) * nb);
            const size_t H = size_t(xband_rows_host(c.n / c.wr / C));
            L.xband_seg = off;  off = align256(off + sizeof(int32_t) * 3 * size_t(C) * size_t(C) * H * H * size_t(c.wc - 1));
        }
    }
    if (with_G) {
        size_t kw = (size_t(c.k) + 31) / 32;
        L.perm = off;  off = align256(off + sizeof(int32_t) * size_t(c.n));
        L.pinv = off;  off = align256(off + sizeof(int32_t) * size_t(c.n));
        const size_t npp = (size_t(c.n - c.k) + kEncColTile - 1) / kEncColTile * kEncColTile;
        L.pt = off;    off = align256(off + sizeof(uint32_t) * std::max<size_t>(kw * npp, 1));
        L.asmtab = off; off = align256(off + sizeof(uint32_t) * 16 * ((size_t(c.n) + 31) / 32));
    }
    L.total = off;
    return L;
}

// Shared-memory bank balancing of the 16-bit band view (MODE 2 band kernel).
// In the check phase a warp processes 32 consecutive band-b rows (positions
// 32u .. 32u+31 of the concatenated band index, u any) and, for element j,
// gathers L (and E, at a band-constant offset) of the rows' j-th variables:
// one shared-memory instruction whose cost is the largest number of the 32
// addresses in one bank (random Tanner-graph rows: 3.5 wavefronts on
// average).  Neither the order of a band's rows nor the order of a row's wr
// variables matters to the algorithm (E is stored at variable positions and a
// check node is symmetric), so both are chosen here: rows are moved between a
// band's 32-row windows to flatten each window's histogram of variable banks
// (swap local search on sum (count - wr)^2), then each row's variables are
// assigned to elements so that every element column of the window hits
// distinct banks where possible (greedy + pairwise repair).  rel holds 4 v per
// (band, position, element) (the byte offset of L_v relative to L; a
// band-constant shift does not change conflicts); only its order changes.
// Deterministic.
// Proper edge colouring of a bipartite multigraph with K colours (Koenig:
// possible when every node has degree <= K).  Edges e = (eu[e], ev[e]) are
// coloured one by one; when no colour is free at both ends, the path from
// the v end alternating colours a (free at u) and b (free at v) is flipped --
// it cannot reach u (bipartite) -- which frees a at v.  ecol[e] in [0, K).
static void koenig_colour(const std::vector<int32_t> &eu, const std::vector<int32_t> &ev, int32_t nu, int32_t nv,
                          int32_t K, std::vector<int32_t> &ecol) {
    const size_t ne = eu.size();
    ecol.assign(ne, -1);
    std::vector<int32_t> at_u(size_t(nu) * K, -1), at_v(size_t(nv) * K, -1), path;
    for (size_t e = 0; e < ne; ++e) {
        const int32_t u = eu[e], v = ev[e];
        int32_t a = -1, b = -1, c = -1;
        for (int32_t k = 0; k < K; ++k) {
            const bool fu = at_u[size_t(u) * K + k] < 0, fv = at_v[size_t(v) * K + k] < 0;
            if (fu && fv) { c = k; break; }
            if (fu && a < 0) a = k;
            if (fv && b < 0) b = k;
        }
        if (c < 0) {
            path.clear();
            int32_t node = v, cc = a;
            bool at_v_side = true;
            for (;;) {
                const int32_t ed = at_v_side ? at_v[size_t(node) * K + cc] : at_u[size_t(node) * K + cc];
                if (ed < 0) break;
                path.push_back(ed);
                node = at_v_side ? eu[size_t(ed)] : ev[size_t(ed)];
                at_v_side = !at_v_side;
                cc = cc == a ? b : a;
            }
            for (int32_t ed : path) {
                at_u[size_t(eu[size_t(ed)]) * K + ecol[size_t(ed)]] = -1;
                at_v[size_t(ev[size_t(ed)]) * K + ecol[size_t(ed)]] = -1;
            }
            for (int32_t ed : path) {
                ecol[size_t(ed)] = ecol[size_t(ed)] == a ? b : a;
                at_u[size_t(eu[size_t(ed)]) * K + ecol[size_t(ed)]] = ed;
                at_v[size_t(ev[size_t(ed)]) * K + ecol[size_t(ed)]] = ed;
            }
            c = a;
        }
        ecol[e] = c;
        at_u[size_t(u) * K + c] = int32_t(e);
        at_v[size_t(v) * K + c] = int32_t(e);
    }
}

// Element columns of one window: wb[i*wr + j] = bank of row i's j-th element
// (nr rows); col[i*wr + j] = the column it is stored in.  A column's cost is
// its largest bank multiplicity.  With c_q the window's count of bank q and
// g = max(0, max_q c_q - wr): g "double" columns take each bank at most
// twice, the other wr - g at most once, so the window costs wr + g
// wavefronts over its wr gathers (the least a histogram with a bank seen
// wr + g times allows when every bank fits in two double columns).  Which of
// a row's elements go to the double columns is a bipartite flow: row i sends
// exactly g, bank q receives between c_q - (wr - g) and 2g; then the single
// part (degrees <= wr - g) and the double part (banks split in two nodes of
// degree <= g) are each Koenig-coloured.  If that flow does not exist, g is
// raised; past wr, every bank is split in nodes of <= wr edges and coloured
// with wr colours (a bank seen c times lands <= ceil(c / wr) times a column).
static void color_window_elements(const std::vector<int32_t> &wb, int32_t nr, int32_t wr, std::vector<int32_t> &col) {
    col.assign(size_t(nr) * wr, 0);
    int32_t cnt[32] = {0};
    for (int32_t i = 0; i < nr * wr; ++i) cnt[wb[size_t(i)]]++;
    const int32_t cmax = *std::max_element(cnt, cnt + 32);
    std::vector<int32_t> eu, ev, ecol, mult(size_t(nr) * 32), flow(size_t(nr) * 32), prev(nr + 32 + 2);
    bool done = false;
    for (int32_t g = std::max(0, cmax - wr); g < wr && !done; ++g) {
        bool ok = true;
        std::vector<uint8_t> dbl(size_t(nr) * wr, 0);
        if (g > 0) {
            std::fill(mult.begin(), mult.end(), 0);
            std::fill(flow.begin(), flow.end(), 0);
            for (int32_t i = 0; i < nr; ++i)
                for (int32_t j = 0; j < wr; ++j) mult[size_t(i) * 32 + wb[size_t(i) * wr + j]]++;
            std::vector<int32_t> rowf(nr, 0), bankf(32, 0), lo(32), hi(32);
            for (int q = 0; q < 32; ++q) lo[q] = std::max(0, cnt[q] - (wr - g));
            // BFS augmenting paths s -> row -> bank (forward if flow < mult,
            // backward if flow > 0) -> t; bound[] caps bank -> t
            auto augment = [&](const std::vector<int32_t> &bound) {
                for (;;) {
                    // nodes: rows 0..nr-1, banks nr..nr+31
                    std::fill(prev.begin(), prev.end(), -2);
                    std::vector<int32_t> qu;
                    for (int32_t i = 0; i < nr; ++i)
                        if (rowf[size_t(i)] < g) { prev[size_t(i)] = -1; qu.push_back(i); }
                    int32_t hit = -1;
                    for (size_t h = 0; h < qu.size() && hit < 0; ++h) {
                        const int32_t x = qu[h];
                        if (x < nr) {
                            for (int q = 0; q < 32; ++q)
                                if (prev[size_t(nr + q)] == -2 && flow[size_t(x) * 32 + q] < mult[size_t(x) * 32 + q]) {
                                    prev[size_t(nr + q)] = x;
                                    if (bankf[q] < bound[q]) { hit = nr + q; break; }
                                    qu.push_back(nr + q);
                                }
                        } else {
                            const int q = x - nr;
                            for (int32_t i = 0; i < nr; ++i)
                                if (prev[size_t(i)] == -2 && flow[size_t(i) * 32 + q] > 0) {
                                    prev[size_t(i)] = x;
                                    qu.push_back(i);
                                }
                        }
                    }
                    if (hit < 0) return;
                    bankf[hit - nr]++;
                    int32_t x = hit;
                    while (prev[size_t(x)] != -1) {
                        const int32_t y = prev[size_t(x)];
                        if (x >= nr) flow[size_t(y) * 32 + (x - nr)]++;      // row y -> bank x
                        else flow[size_t(x) * 32 + (y - nr)]--;              // bank y -> row x (undo)
                        x = y;
                    }
                    rowf[size_t(x)]++;
                }
            };
            augment(lo);
            for (int q = 0; q < 32; ++q) ok = ok && bankf[q] >= lo[q];
            if (ok) {
                for (int q = 0; q < 32; ++q) hi[q] = 2 * g;
                augment(hi);
                for (int32_t i = 0; i < nr; ++i) ok = ok && rowf[size_t(i)] == g;
            }
            if (!ok) continue;
            for (int32_t i = 0; i < nr; ++i) {
                int32_t take[32];
                for (int q = 0; q < 32; ++q) take[q] = flow[size_t(i) * 32 + q];
                for (int32_t j = 0; j < wr; ++j)
                    if (take[wb[size_t(i) * wr + j]] > 0) { take[wb[size_t(i) * wr + j]]--; dbl[size_t(i) * wr + j] = 1; }
            }
        }
        // single part: colours [0, wr - g)
        eu.clear(); ev.clear();
        std::vector<size_t> idx;
        for (int32_t i = 0; i < nr * wr; ++i)
            if (!dbl[size_t(i)]) { eu.push_back(i / wr); ev.push_back(wb[size_t(i)]); idx.push_back(size_t(i)); }
        koenig_colour(eu, ev, nr, 32, wr - g, ecol);
        for (size_t e = 0; e < idx.size(); ++e) col[idx[e]] = ecol[e];
        if (g > 0) {
            eu.clear(); ev.clear(); idx.clear();
            int32_t seen[32] = {0};
            for (int32_t i = 0; i < nr * wr; ++i)
                if (dbl[size_t(i)]) {
                    const int32_t q = wb[size_t(i)];
                    eu.push_back(i / wr);
                    ev.push_back(q * 2 + seen[q]++ / g);
                    idx.push_back(size_t(i));
                }
            koenig_colour(eu, ev, nr, 64, g, ecol);
            for (size_t e = 0; e < idx.size(); ++e) col[idx[e]] = wr - g + ecol[e];
        }
        done = true;
    }
    if (!done) {
        // fallback: banks split in nodes of <= wr edges, wr colours
        int32_t seen[32] = {0};
        const int32_t maxk = (cmax + wr - 1) / wr;
        eu.clear(); ev.clear();
        for (int32_t i = 0; i < nr * wr; ++i) {
            const int32_t q = wb[size_t(i)];
            eu.push_back(i / wr);
            ev.push_back(q * maxk + seen[q]++ / wr);
        }
        koenig_colour(eu, ev, nr, 32 * maxk, wr, ecol);
        for (int32_t i = 0; i < nr * wr; ++i) col[size_t(i)] = ecol[size_t(i)];
    }
    // every row's columns must be a permutation of 0..wr-1 (they are by
    // construction; a row that is not keeps its order)
    for (int32_t i = 0; i < nr; ++i) {
        uint64_t m = 0;
        for (int32_t j = 0; j < wr; ++j) m |= uint64_t(1) << col[size_t(i) * wr + j];
        if (m != (wr == 64 ? ~uint64_t(0) : (uint64_t(1) << wr) - 1))
            for (int32_t j = 0; j < wr; ++j) col[size_t(i) * wr + j] = j;
    }
}

// Core of the balancing: rows[0 .. nrows*wr) (byte offsets; bank = offset/4
// mod 32) are partitioned into the given windows (start, len) of consecutive
// row positions.  Rows are moved between windows to flatten each window's
// bank histogram, then each row's elements are ordered so that every element
// column of a window hits distinct banks where possible.
void balance_windows(int32_t *rowsv, int32_t nrows, int32_t wr, const std::vector<int32_t> &wstart,
                     const std::vector<int32_t> &wlen, SplitMix64 &rng) {
    auto bank = [](int32_t off) { return int((off >> 2) & 31); };
    const int32_t nw = int32_t(wstart.size());
    if (nw < 1 || nrows < 1) return;
    std::vector<int32_t> row_win(static_cast<size_t>(nrows));
    for (int32_t w = 0; w < nw; ++w)
        for (int32_t i = 0; i < wlen[size_t(w)]; ++i) row_win[size_t(wstart[size_t(w)] + i)] = w;
    std::vector<int32_t> H(size_t(nw) * 32, 0);
    for (int32_t r = 0; r < nrows; ++r)
        for (int32_t j = 0; j < wr; ++j) H[size_t(row_win[size_t(r)]) * 32 + bank(rowsv[size_t(r) * wr + j])]++;
    // cost: squared deviation from the flat histogram plus a heavy penalty on
    // counts above the element count wr (ceil of the flat count for a short
    // window): a bank seen at most wr times in a window can be spread over the
    // wr element columns without a conflict (below), one seen more cannot
    std::vector<int32_t> capw(static_cast<size_t>(nw));
    for (int32_t w = 0; w < nw; ++w) capw[size_t(w)] = (wlen[size_t(w)] * wr + 31) / 32;
    auto cost_of = [&](int32_t w, const int32_t *h) {
        int64_t s = 0;
        const int32_t cap = capw[size_t(w)];
        for (int q = 0; q < 32; ++q) {
            const int64_t d = int64_t(h[q]) * 32 - int64_t(wlen[size_t(w)]) * wr;
            const int64_t o = std::max<int64_t>(0, h[q] - cap);
            s += d * d + o * o * 65536;
        }
        return s;
    };
    auto try_swap = [&](int32_t r, int32_t s, int32_t *ha, int32_t *hb, int64_t &delta) {
        const int32_t wa = row_win[size_t(r)], wb = row_win[size_t(s)];
        std::copy(&H[size_t(wa) * 32], &H[size_t(wa) * 32] + 32, ha);
        std::copy(&H[size_t(wb) * 32], &H[size_t(wb) * 32] + 32, hb);
        const int64_t c0 = cost_of(wa, ha) + cost_of(wb, hb);
        for (int32_t j = 0; j < wr; ++j) {
            const int br = bank(rowsv[size_t(r) * wr + j]), bs = bank(rowsv[size_t(s) * wr + j]);
            ha[br]--; ha[bs]++; hb[bs]--; hb[br]++;
        }
        delta = cost_of(wa, ha) + cost_of(wb, hb) - c0;
    };
    auto commit_swap = [&](int32_t r, int32_t s, const int32_t *ha, const int32_t *hb) {
        const int32_t wa = row_win[size_t(r)], wb = row_win[size_t(s)];
        std::copy(ha, ha + 32, &H[size_t(wa) * 32]);
        std::copy(hb, hb + 32, &H[size_t(wb) * 32]);
        row_win[size_t(r)] = wb;
        row_win[size_t(s)] = wa;
    };
    if (nw > 1) {
        const int64_t attempts = int64_t(nrows) * 200;
        int32_t ha[32], hb[32];
        for (int64_t t = 0; t < attempts; ++t) {
            const int32_t r = int32_t(rng.next() % uint64_t(nrows)), s = int32_t(rng.next() % uint64_t(nrows));
            if (row_win[size_t(r)] == row_win[size_t(s)]) continue;
            int64_t d;
            try_swap(r, s, ha, hb, d);
            if (d < 0) commit_swap(r, s, ha, hb);
        }
        // targeted passes: for every over-full (window, bank), move one of the
        // window's rows holding that bank out, to the best of a few random
        // partners
        int32_t bha[32], bhb[32];
        std::vector<std::vector<int32_t>> mem(static_cast<size_t>(nw));
        for (int pass = 0; pass < 60; ++pass) {
            for (auto &m : mem) m.clear();
            for (int32_t r = 0; r < nrows; ++r) mem[size_t(row_win[size_t(r)])].push_back(r);
            int64_t moved = 0;
            for (int32_t w = 0; w < nw; ++w)
                for (int q = 0; q < 32; ++q) {
                    if (H[size_t(w) * 32 + q] <= capw[size_t(w)]) continue;
                    int32_t cand[64], nc = 0;
                    for (int32_t r : mem[size_t(w)]) {
                        if (row_win[size_t(r)] != w) continue;
                        for (int32_t j = 0; j < wr; ++j)
                            if (bank(rowsv[size_t(r) * wr + j]) == q) { if (nc < 64) cand[nc++] = r; break; }
                    }
                    if (!nc) continue;
                    const int32_t r = cand[rng.next() % uint64_t(nc)];
                    int64_t best = 0;
                    int32_t bs = -1;
                    for (int k = 0; k < 48; ++k) {
                        const int32_t s = int32_t(rng.next() % uint64_t(nrows));
                        if (row_win[size_t(s)] == w) continue;
                        int64_t d;
                        try_swap(r, s, ha, hb, d);
                        if (d < best) { best = d; bs = s; std::copy(ha, ha + 32, bha); std::copy(hb, hb + 32, bhb); }
                    }
                    if (bs >= 0) { commit_swap(r, bs, bha, bhb); ++moved; }
                }
            if (!moved) break;
        }
    }
    std::vector<std::vector<int32_t>> members(static_cast<size_t>(nw));
    for (int32_t r = 0; r < nrows; ++r) members[size_t(row_win[size_t(r)])].push_back(r);
    std::vector<int32_t> out(static_cast<size_t>(nrows) * wr);
    // Element order of a window (color_window_elements): every element column
    // of the window hits distinct banks where the window's histogram allows.
    std::vector<int32_t> wb, col;
    for (int32_t w = 0; w < nw; ++w) {
        const auto &mem = members[size_t(w)];
        const int32_t nr = int32_t(mem.size());
        wb.resize(size_t(nr) * wr);
        for (int32_t i = 0; i < nr; ++i)
            for (int32_t j = 0; j < wr; ++j) wb[size_t(i) * wr + j] = bank(rowsv[size_t(mem[size_t(i)]) * wr + j]);
        color_window_elements(wb, nr, wr, col);
        int32_t *dst = out.data() + size_t(wstart[size_t(w)]) * wr;
        for (int32_t i = 0; i < nr; ++i)
            for (int32_t j = 0; j < wr; ++j)
                dst[size_t(i) * wr + col[size_t(i) * wr + j]] = rowsv[size_t(mem[size_t(i)]) * wr + j];
    }
    std::copy(out.begin(), out.end(), rowsv);
}

// Mean wavefronts per gather of a balanced (or not) row array (debug).
double window_wavefronts(const int32_t *rowsv, int32_t wr, const std::vector<int32_t> &wstart,
                         const std::vector<int32_t> &wlen) {
    double tot = 0;
    int nins = 0;
    for (size_t w = 0; w < wstart.size(); ++w)
        for (int32_t j = 0; j < wr; ++j) {
            int h[32] = {0}, mx = 0;
            for (int32_t i = 0; i < wlen[w]; ++i) mx = std::max(mx, ++h[(rowsv[size_t(wstart[w] + i) * wr + j] >> 2) & 31]);
            tot += mx;
            ++nins;
        }
    return nins ? tot / nins : 0.0;
}

void bank_balance_rows(int32_t n, int32_t wc, int32_t wr, std::vector<int32_t> &rel) {
    const int32_t mb = n / wr, NB = wc - 1;
    // only the band kernels (a frame in one SM's shared memory) gather through this view
    if (wr > 32 || mb < 64 || !band_frame_fits_sm(n, wc)) return;
    SplitMix64 rng(0x9e3779b97f4a7c15ull ^ uint64_t(n));
    for (int32_t b = 0; b < NB; ++b) {
        int32_t *band = rel.data() + size_t(b) * size_t(n);
        // windows: 32-aligned blocks of the concatenated row index, clipped to this band
        const int32_t base = b * mb;
        std::vector<int32_t> wstart, wlen;
        for (int32_t r = base; r < base + mb;) {
            const int32_t end = std::min(base + mb, (r / 32 + 1) * 32);
            wstart.push_back(r - base);
            wlen.push_back(end - r);
            r = end;
        }
        balance_windows(band, mb, wr, wstart, wlen, rng);
        if (std::getenv("LDPC_DEBUG"))
            std::fprintf(stderr, "ldpc bank_balance: band %d: %.3f wavefronts per gather\n", b + 1,
                         window_wavefronts(band, wr, wstart, wlen));
    }
}

// Message-segment tables of the exchange cluster kernel (spa_cluster.cu).
// CTA q owns band rows [q mbq, (q+1) mbq) of every band and the variables
// [q nq, (q+1) nq) of its band-0 rows.  With T = xband_threads(mbq) compute
// threads and H = xband_rows_per_thread(mbq), local band-0 row rl is
// processed in V-phase chunk h = rl / T, and local row lr of band b >= 1 in
// C-phase chunk c = (b-1) H + lr / T.  Every band-b >= 1 edge (b, p) joins
// variable owner s = pi_b[p] / nq and row owner d = (p / wr) / mbq.  The edge
// has ONE slot in s's VAR region (E_cv arrives there, L_vc is written over
// it) and ONE in d's ROW region (L_vc arrives there, E_cv is written over it).
// Edges sharing (s, d, h, c) form a segment, contiguous and in ascending p in
// both regions:
//   var region of s: segments ordered by (h, d, c) -- V chunk h ships its
//                                                    C NC segments (NC = (wc-1) H)
//   row region of d: segments ordered by (c, s, h) -- C chunk c ships its C H
// Segments are padded to 16 bytes (bulk-copy granularity).  Outputs:
//   ridx[(b-1) n + p]    = byte slot of edge (b, p) in d's row region
//   sidx[v (wc-1) + b-1] = byte slot of edge (b, pi_b^-1(v)) in s's var region
//   seg = { varOff, rowOff, bytes }, three int32 arrays indexed by
//         key(s, d, h, c) = ((s C + d) H + h) NC + c.
// Returns the exact region capacity in floats (the largest region).
int32_t xband_tables(const ldpc_code &c, int C, std::vector<uint16_t> &ridx, std::vector<uint16_t> &sidx,
                     std::vector<int32_t> &seg) {
    const int32_t n = c.n, wc = c.wc, wr = c.wr, NB = wc - 1, mbq = n / wr / C, nq = mbq * wr;
    const int32_t T = xband_threads_host(mbq), H = xband_rows_host(mbq), NC = NB * H;
    const size_t nb = size_t(NB) * size_t(n), nkey = size_t(C) * C * H * NC;
    auto key = [&](int32_t s, int32_t d, int32_t h, int32_t ch) { return ((size_t(s) * C + d) * H + h) * NC + ch; };
    std::vector<int32_t> cnt(nkey, 0), rank(nb), kof(nb);
    for (int32_t b = 0; b < NB; ++b)
        for (int32_t p = 0; p < n; ++p) {
            const int32_t v = c.col_idx[size_t(b + 1) * n + p];
            const int32_t s = v / nq, d = (p / wr) / mbq, h = ((v - s * nq) / wr) / T;
            const int32_t ch = b * H + ((p / wr) - d * mbq) / T;
            const size_t k = key(s, d, h, ch);
            kof[size_t(b) * n + p] = int32_t(k);
            rank[size_t(b) * n + p] = cnt[k]++;
        }
    auto pad = [](int32_t x) { return (x + 3) & ~3; };
    seg.assign(3 * nkey, 0);
    int32_t *varOff = seg.data(), *rowOff = seg.data() + nkey, *bytes = seg.data() + 2 * nkey;
    int32_t cap = 0;
    for (int32_t s = 0; s < C; ++s) {
        int32_t o = 0;
        for (int32_t h = 0; h < H; ++h)
            for (int32_t d = 0; d < C; ++d)
                for (int32_t ch = 0; ch < NC; ++ch) { varOff[key(s, d, h, ch)] = 4 * o; o += pad(cnt[key(s, d, h, ch)]); }
        cap = std::max(cap, o);
    }
    for (int32_t d = 0; d < C; ++d) {
        int32_t o = 0;
        for (int32_t ch = 0; ch < NC; ++ch)
            for (int32_t s = 0; s < C; ++s)
                for (int32_t h = 0; h < H; ++h) { rowOff[key(s, d, h, ch)] = 4 * o; o += pad(cnt[key(s, d, h, ch)]); }
        cap = std::max(cap, o);
    }
    for (size_t i = 0; i < nkey; ++i) bytes[i] = 4 * pad(cnt[i]);
    if (cap > kXbandMaxCapacity) return cap;     // 16-bit byte slots overflow: the caller drops the view
    // V-phase bank balancing through the ranks: an edge's rank inside its
    // segment fixes its VAR-region bank ((varOff + r) mod 32) and its ROW
    // slot.  A V-phase warp instruction gathers (variable j, band b) of the 32
    // band-0 rows of one warp window, so ranks are dealt greedily to give each
    // such instruction distinct banks (the C-phase is balanced afterwards by
    // reordering rows and elements, which keeps the ranks).
    if (!std::getenv("LDPC_NO_BANKOPT")) {
        std::vector<std::vector<int32_t>> avail(nkey * 32);
        for (size_t k = 0; k < nkey; ++k)
            for (int32_t r = cnt[k] - 1; r >= 0; --r) avail[k * 32 + size_t((varOff[k] / 4 + r) & 31)].push_back(r);
        const int32_t nwin = (T + 31) / 32;
        const size_t ninstr = size_t(C) * H * nwin * wr * NB;
        std::vector<std::vector<int32_t>> instr(ninstr);
        for (int32_t b = 0; b < NB; ++b)
            for (int32_t p = 0; p < n; ++p) {
                const int32_t v = c.col_idx[size_t(b + 1) * n + p];
                const int32_t s = v / nq, vl = v - s * nq, rl = vl / wr, j = vl - rl * wr;
                const int32_t h = rl / T, w = (rl % T) / 32;
                instr[((size_t(s) * H + h) * nwin + w) * size_t(wr * NB) + size_t(j * NB + b)].push_back(b * n + p);
            }
        double before = 0, after = 0;
        int ninst = 0;
        for (auto &ins : instr) {
            if (ins.empty()) continue;
            if (std::getenv("LDPC_DEBUG")) {
                int hcount[32] = {0}, mx = 0;
                for (int32_t e : ins) mx = std::max(mx, ++hcount[(varOff[size_t(kof[size_t(e)])] / 4 + rank[size_t(e)]) & 31]);
                before += mx;
            }
            // edges with the fewest usable banks first
            std::vector<std::pair<int, int32_t>> order;
            for (int32_t e : ins) {
                const size_t k = size_t(kof[size_t(e)]);
                int opts = 0;
                for (int m = 0; m < 32; ++m) opts += !avail[k * 32 + size_t(m)].empty();
                order.push_back({opts, e});
            }
            std::sort(order.begin(), order.end());
            uint32_t used = 0;
            int hcount[32] = {0};
            for (const auto &oe : order) {
                const int32_t e = oe.second;
                const size_t k = size_t(kof[size_t(e)]);
                int best = -1;
                size_t bs = 0;
                for (int m = 0; m < 32; ++m) {
                    const size_t sz = avail[k * 32 + size_t(m)].size();
                    if (sz && !(used >> m & 1u) && sz > bs) { bs = sz; best = m; }
                }
                if (best < 0)
                    for (int m = 0; m < 32; ++m) {
                        const size_t sz = avail[k * 32 + size_t(m)].size();
                        if (sz > bs) { bs = sz; best = m; }
                    }
                rank[size_t(e)] = avail[k * 32 + size_t(best)].back();
                avail[k * 32 + size_t(best)].pop_back();
                used |= 1u << best;
                hcount[best]++;
            }
            if (std::getenv("LDPC_DEBUG")) {
                int mx = 0;
                for (int m = 0; m < 32; ++m) mx = std::max(mx, hcount[m]);
                after += mx;
                ++ninst;
            }
        }
        if (std::getenv("LDPC_DEBUG") && ninst)
            std::fprintf(stderr, "ldpc xband bank_balance: V-phase %.3f -> %.3f wavefronts per gather\n", before / ninst,
                         after / ninst);
    }
    ridx.assign(nb, 0);
    sidx.assign(nb, 0);
    for (int32_t b = 0; b < NB; ++b)
        for (int32_t p = 0; p < n; ++p) {
            const int32_t v = c.col_idx[size_t(b + 1) * n + p];
            const size_t k = size_t(kof[size_t(b) * n + p]);
            const int32_t r = rank[size_t(b) * n + p];
            ridx[size_t(b) * n + p] = uint16_t(rowOff[k] + 4 * r);
            sidx[size_t(v) * NB + b] = uint16_t(varOff[k] + 4 * r);
        }
    // Bank balancing of the C-phase gathers (see balance_windows): a CTA's
    // band-b rows of one row step (one C chunk: their segments are fixed) may
    // be processed in any order and a row's slots listed in any order, so both
    // are chosen to spread each warp's 32 row-region addresses over the banks.
    if (!std::getenv("LDPC_NO_BANKOPT")) {
        SplitMix64 rng(0x7f4a7c159e3779b9ull ^ uint64_t(n) ^ (uint64_t(C) << 32));
        std::vector<int32_t> rows;
        double before = 0, after = 0;
        int nchunks = 0;
        for (int32_t d = 0; d < C; ++d)
            for (int32_t b = 0; b < NB; ++b)
                for (int32_t k0 = 0; k0 < mbq; k0 += T) {
                    const int32_t nr = std::min(T, mbq - k0);
                    uint16_t *base = ridx.data() + size_t(b) * n + size_t(d * mbq + k0) * wr;
                    rows.assign(base, base + size_t(nr) * wr);
                    std::vector<int32_t> wstart, wlen;
                    for (int32_t r = 0; r < nr; r += 32) {
                        wstart.push_back(r);
                        wlen.push_back(std::min(32, nr - r));
                    }
                    if (std::getenv("LDPC_DEBUG")) before += window_wavefronts(rows.data(), wr, wstart, wlen);
                    balance_windows(rows.data(), nr, wr, wstart, wlen, rng);
                    if (std::getenv("LDPC_DEBUG")) after += window_wavefronts(rows.data(), wr, wstart, wlen);
                    ++nchunks;
                    for (size_t i = 0; i < rows.size(); ++i) base[i] = uint16_t(rows[i]);
                }
        if (std::getenv("LDPC_DEBUG"))
            std::fprintf(stderr, "ldpc xband bank_balance: C-phase %.3f -> %.3f wavefronts per gather\n",
                         before / std::max(nchunks, 1), after / std::max(nchunks, 1));
    }
    return cap;
}
// Encoder assemble table (codec_kernels.cu encode_assemble_dep_kernel).  The
// codeword in H order interleaves the message bits (positions perm[0..k)) and
// the parity bits (perm[k..n)); both halves of perm ascend (reading Q13:
// [free ascending, pivots ascending]), so codeword word j takes the next
// popc(info mask) message bits starting at message bit a_j and the next
// parity bits starting at 32 j - a_j, each deposited into its mask's
// positions.  The deposit is Hacker's Delight's expand (7-5) with the five
// move masks of each mask precomputed here.  Per word, 16 uint32: info mask,
// parity mask, a_j, 0, move masks of the info mask [5], of the parity mask
// [5], 0 x 3.  False (no table) if a half of perm does not ascend.
static void expand_moves(uint32_t m, uint32_t mv_out[5]) {
    uint32_t mk = ~m << 1;
    for (int i = 0; i < 5; ++i) {
        uint32_t mp = mk ^ (mk << 1);
        mp ^= mp << 2;
        mp ^= mp << 4;
        mp ^= mp << 8;
        mp ^= mp << 16;
        const uint32_t mv = mp & m;
        mv_out[i] = mv;
        m = (m ^ mv) | (mv >> (1 << i));
        mk &= ~mp;
    }
}
bool assemble_table(const ldpc_code &c, std::vector<uint32_t> &tab) {
    const int32_t n = c.n, k = c.k;
    for (int32_t t = 1; t < n; ++t)
        if (t != k && c.perm[size_t(t)] <= c.perm[size_t(t - 1)]) return false;
    const int32_t nw = (n + 31) / 32;
    tab.assign(size_t(nw) * 16, 0u);
    int32_t a = 0;          // message bits before word j
    for (int32_t j = 0; j < nw; ++j) {
        uint32_t mi = 0, mp = 0;
        for (int32_t b = 0; b < 32; ++b) {
            const int32_t v = 32 * j + b;
            if (v >= n) break;
            if (c.pinv[size_t(v)] < k) mi |= 1u << b;
            else mp |= 1u << b;
        }
        uint32_t *e = &tab[size_t(j) * 16];
        e[0] = mi;
        e[1] = mp;
        e[2] = uint32_t(a);
        expand_moves(mi, e + 4);
        expand_moves(mp, e + 9);
        a += __builtin_popcount(mi);
    }
    return a == k;
}

}  // namespace ldpc

extern "C" {

const char *ldpc_status_str(ldpc_status s) {
    switch (s) {
        case LDPC_OK: return "ok";
        case LDPC_ERR_ARG: return "invalid argument";
        case LDPC_ERR_NOT_DIVISIBLE: return "wr does not divide n";
        case LDPC_ERR_NO_INFO_BITS: return "code has no information bits (k == 0)";
        case LDPC_ERR_DIM: return "dimension mismatch";
        case LDPC_ERR_STATE: return "call out of order (make_G / bind_device missing)";
        case LDPC_ERR_UNSUPPORTED: return "unsupported code or decoder variant for this code";
        case LDPC_ERR_CUDA: return "CUDA runtime error";
        case LDPC_ERR_NOMEM: return "out of host memory";
    }
    return "unknown status";
}

// Gallager band construction, P:37 / P:598.
ldpc_status ldpc_make_H(int32_t n, int32_t wc, int32_t wr, uint64_t seed, ldpc_code **out) {
    if (!out) return LDPC_ERR_ARG;
    *out = nullptr;
    if (n <= 0 || wc < 1 || wr < 2 || wc >= wr || wr > ldpc::kMaxCheckDegree) return LDPC_ERR_ARG;
    if (n % wr) return LDPC_ERR_NOT_DIVISIBLE;
    ldpc_code *c = new (std::nothrow) ldpc_code;
    if (!c) return LDPC_ERR_NOMEM;
    try {
        const int32_t mb = n / wr;
        c->n = n; c->m = mb * wc; c->nnz = c->m * wr;
        c->wc = wc; c->wr = wr; c->gallager = 1;
        c->design_rate = 1.0 - double(wc) / double(wr);
        c->row_ptr.resize(size_t(c->m) + 1);
        for (int32_t r = 0; r <= c->m; ++r) c->row_ptr[r] = r * wr;
        c->col_idx.resize(size_t(c->nnz));
        std::vector<int32_t> pi(static_cast<size_t>(n));
        SplitMix64 rng(seed);
        for (int32_t band = 0; band < wc; ++band) {
            for (int32_t i = 0; i < n; ++i) pi[i] = i;
            if (band > 0)
                for (int32_t i = n - 1; i > 0; --i) {
                    int32_t j = int32_t(rng.below(uint64_t(i) + 1));
                    std::swap(pi[i], pi[j]);
                }
            // row band*mb + r holds pi[r*wr .. r*wr+wr): edge ids are band*n + position
            std::copy(pi.begin(), pi.end(), c->col_idx.begin() + size_t(band) * n);
        }
        build_csc(*c);
    } catch (...) {
        delete c;
        return LDPC_ERR_NOMEM;
    }
    *out = c;
    return LDPC_OK;
}

ldpc_status ldpc_code_from_csr(int32_t m, int32_t n, const int32_t *row_ptr, const int32_t *col_idx,
                               ldpc_code **out) {
    if (!out) return LDPC_ERR_ARG;
    *out = nullptr;
    if (m < 0 || n <= 0 || !row_ptr || (row_ptr[m] > 0 && !col_idx) || row_ptr[0] != 0)
        return LDPC_ERR_ARG;
    for (int32_t r = 0; r < m; ++r) {
        int32_t d = row_ptr[r + 1] - row_ptr[r];
        if (d < 0) return LDPC_ERR_ARG;
        if (d > ldpc::kMaxCheckDegree) return LDPC_ERR_UNSUPPORTED;
    }
    std::vector<uint8_t> seen(static_cast<size_t>(n), 0);
    for (int32_t r = 0; r < m; ++r) {
        for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            int32_t v = col_idx[e];
            if (v < 0 || v >= n || seen[v]) {
                for (int32_t q = row_ptr[r]; q < e; ++q) seen[col_idx[q]] = 0;
                return LDPC_ERR_ARG;
            }
            seen[v] = 1;
        }
        for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) seen[col_idx[e]] = 0;
    }
    ldpc_code *c = new (std::nothrow) ldpc_code;
    if (!c) return LDPC_ERR_NOMEM;
    try {
        c->n = n; c->m = m; c->nnz = row_ptr[m];
        c->row_ptr.assign(row_ptr, row_ptr + m + 1);
        c->col_idx.assign(col_idx, col_idx + c->nnz);
        c->design_rate = 1.0 - double(m) / double(n);
        build_csc(*c);
    } catch (...) {
        delete c;
        return LDPC_ERR_NOMEM;
    }
    *out = c;
    return LDPC_OK;
}

// MacKay alist (P:4 "Any Binary Parity Check matrix ... can be
// used"): "n m", "max_col_weight max_row_weight", the n column weights, the m
// row weights, n lines of 1-based row indices per column, m lines of 1-based
// column indices per row, each line zero-padded to the maximum weight.  Index
// lists are written in ascending order.
ldpc_status ldpc_code_write_alist(const ldpc_code *code, char *buf, size_t cap, size_t *len) {
    if (!code || !len) return LDPC_ERR_ARG;
    const int32_t n = code->n, m = code->m;
    std::vector<int32_t> edge_row(size_t(std::max(code->nnz, 1)));
    for (int32_t r = 0; r < m; ++r)
        for (int32_t e = code->row_ptr[r]; e < code->row_ptr[r + 1]; ++e) edge_row[e] = r;
    std::string s;
    s.reserve(size_t(code->nnz) * 14 + size_t(n + m) * 4 + 64);
    auto line = [&](const std::vector<int32_t> &v, int32_t pad_to) {
        for (size_t i = 0; i < v.size(); ++i) {
            if (i) s += ' ';
            s += std::to_string(v[i]);
        }
        for (int32_t i = int32_t(v.size()); i < pad_to; ++i) {
            if (i) s += ' ';
            s += '0';
        }
        s += '\n';
    };
    line({n, m}, 0);
    line({code->max_col_deg, code->max_row_deg}, 0);
    std::vector<int32_t> v;
    v.clear();
    for (int32_t j = 0; j < n; ++j) v.push_back(code->var_ptr[j + 1] - code->var_ptr[j]);
    line(v, 0);
    v.clear();
    for (int32_t r = 0; r < m; ++r) v.push_back(code->row_ptr[r + 1] - code->row_ptr[r]);
    line(v, 0);
    for (int32_t j = 0; j < n; ++j) {
        v.clear();
        for (int32_t t = code->var_ptr[j]; t < code->var_ptr[j + 1]; ++t) v.push_back(edge_row[code->var_edges[t]] + 1);
        std::sort(v.begin(), v.end());
        line(v, code->max_col_deg);
    }
    for (int32_t r = 0; r < m; ++r) {
        v.assign(code->col_idx.begin() + code->row_ptr[r], code->col_idx.begin() + code->row_ptr[r + 1]);
        for (auto &x : v) x += 1;
        std::sort(v.begin(), v.end());
        line(v, code->max_row_deg);
    }
    *len = s.size();
    if (!buf) return LDPC_OK;
    if (cap < s.size() + 1) return LDPC_ERR_DIM;
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
    return LDPC_OK;
}

ldpc_status ldpc_code_from_alist(const char *text, size_t len, ldpc_code **out) {
    if (!out) return LDPC_ERR_ARG;
    *out = nullptr;
    if (!text) return LDPC_ERR_ARG;
    // split into lines of non-negative integers (blank lines skipped)
    std::vector<std::vector<int64_t>> lines;
    std::vector<int64_t> cur;
    int64_t val = 0;
    bool in_num = false;
    for (size_t i = 0; i <= len; ++i) {
        const char ch = i < len ? text[i] : '\n';
        if (ch >= '0' && ch <= '9') {
            val = val * 10 + (ch - '0');
            if (val > (int64_t(1) << 31)) return LDPC_ERR_ARG;
            in_num = true;
            continue;
        }
        if (in_num) {
            cur.push_back(val);
            val = 0;
            in_num = false;
        }
        if (ch == '\n') {
            if (!cur.empty()) lines.push_back(cur);
            cur.clear();
        } else if (ch != ' ' && ch != '\t' && ch != '\r' && ch != '\0') {
            return LDPC_ERR_ARG;
        }
    }
    if (lines.size() < 4 || lines[0].size() != 2 || lines[1].size() != 2) return LDPC_ERR_ARG;
    const int64_t n = lines[0][0], m = lines[0][1];
    if (n <= 0 || m < 0 || n > (int64_t(1) << 28) || m > (int64_t(1) << 28)) return LDPC_ERR_ARG;
    if (lines[2].size() != size_t(n) || lines[3].size() != size_t(m)) return LDPC_ERR_DIM;
    if (lines.size() != size_t(4 + n + m)) return LDPC_ERR_DIM;
    const int64_t maxc = lines[1][0], maxr = lines[1][1];
    // rows -> CSR (1-based column indices, zeros are padding)
    std::vector<int32_t> row_ptr(size_t(m) + 1, 0), col_idx;
    for (int64_t r = 0; r < m; ++r) {
        const auto &L = lines[size_t(4 + n + r)];
        int64_t w = 0;
        bool padding = false;
        for (int64_t x : L) {
            if (x == 0) { padding = true; continue; }
            if (padding || x > n) return LDPC_ERR_DIM;          // index after padding, or out of range
            col_idx.push_back(int32_t(x - 1));
            ++w;
        }
        if (w != lines[3][size_t(r)] || w > maxr || int64_t(L.size()) > std::max<int64_t>(maxr, w)) return LDPC_ERR_DIM;
        row_ptr[size_t(r) + 1] = int32_t(col_idx.size());
    }
    // columns must describe the same matrix
    std::vector<std::vector<int32_t>> col_rows(static_cast<size_t>(n));
    for (int64_t r = 0; r < m; ++r)
        for (int32_t e = row_ptr[size_t(r)]; e < row_ptr[size_t(r) + 1]; ++e) col_rows[size_t(col_idx[e])].push_back(int32_t(r));
    for (int64_t j = 0; j < n; ++j) {
        const auto &L = lines[size_t(4 + j)];
        std::vector<int32_t> rows;
        bool padding = false;
        for (int64_t x : L) {
            if (x == 0) { padding = true; continue; }
            if (padding || x > m) return LDPC_ERR_DIM;
            rows.push_back(int32_t(x - 1));
        }
        if (int64_t(rows.size()) != lines[2][size_t(j)] || int64_t(rows.size()) > maxc ||
            int64_t(L.size()) > std::max<int64_t>(maxc, int64_t(rows.size())))
            return LDPC_ERR_DIM;
        std::sort(rows.begin(), rows.end());
        auto want = col_rows[size_t(j)];
        std::sort(want.begin(), want.end());
        if (rows != want) return LDPC_ERR_DIM;
    }
    return ldpc_code_from_csr(int32_t(m), int32_t(n), row_ptr.data(), col_idx.empty() ? nullptr : col_idx.data(), out);
}

// Standard-form generator, Eq. 2-3; reading Q13.
// Bit-packed rows (64 columns per word); the pivot search is sequential, the
// elimination of column j from all other rows is split across host threads.
ldpc_status ldpc_make_G(ldpc_code *code) {
    if (!code) return LDPC_ERR_ARG;
    ldpc_code &c = *code;
    const int32_t n = c.n, m = c.m;
    const size_t W = (size_t(n) + 63) / 64;
    std::vector<uint64_t> M;
    try {
        M.assign(size_t(m) * W, 0);
    } catch (...) {
        return LDPC_ERR_NOMEM;
    }
    for (int32_t r = 0; r < m; ++r)
        for (int32_t e = c.row_ptr[r]; e < c.row_ptr[r + 1]; ++e) {
            int32_t v = c.col_idx[e];
            M[size_t(r) * W + size_t(v >> 6)] ^= uint64_t(1) << (v & 63);
        }
    std::vector<int32_t> pivot_row(static_cast<size_t>(n), -1);
    const unsigned T = worker_count();
    int32_t rank = 0;
    std::vector<int32_t> targets;
    targets.reserve(size_t(m));
    for (int32_t j = n - 1; j >= 0 && rank < m; --j) {
        const size_t w = size_t(j >> 6);
        const uint64_t bit = uint64_t(1) << (j & 63);
        int32_t p = -1;
        for (int32_t r = rank; r < m; ++r)
            if (M[size_t(r) * W + w] & bit) { p = r; break; }
        if (p < 0) continue;
        if (p != rank)
            std::swap_ranges(M.begin() + ptrdiff_t(size_t(p) * W), M.begin() + ptrdiff_t(size_t(p) * W + W),
                             M.begin() + ptrdiff_t(size_t(rank) * W));
        targets.clear();
        for (int32_t r = 0; r < m; ++r)
            if (r != rank && (M[size_t(r) * W + w] & bit)) targets.push_back(r);
        const uint64_t *src = M.data() + size_t(rank) * W;
        auto work = [&](size_t lo, size_t hi) {
            for (size_t t = lo; t < hi; ++t) {
                uint64_t *dst = M.data() + size_t(targets[t]) * W;
                for (size_t q = 0; q < W; ++q) dst[q] ^= src[q];
            }
        };
        const size_t ntar = targets.size();
        if (ntar * W < (size_t(1) << 16) || T == 1) {
            work(0, ntar);
        } else {
            std::vector<std::thread> pool;
            size_t chunk = (ntar + T - 1) / T;
            for (unsigned t = 0; t < T; ++t) {
                size_t lo = size_t(t) * chunk, hi = std::min(ntar, lo + chunk);
                if (lo < hi) pool.emplace_back(work, lo, hi);
            }
            for (auto &th : pool) th.join();
        }
        pivot_row[size_t(j)] = rank;
        ++rank;
    }
    const int32_t k = n - rank;
    if (k == 0) return LDPC_ERR_NO_INFO_BITS;
    try {
        c.perm.resize(size_t(n));
        int32_t nf = 0, np = 0;
        for (int32_t j = 0; j < n; ++j)
            if (pivot_row[size_t(j)] < 0) c.perm[size_t(nf++)] = j;
        for (int32_t j = 0; j < n; ++j)
            if (pivot_row[size_t(j)] >= 0) c.perm[size_t(k + np++)] = j;
        c.pinv.resize(size_t(n));
        for (int32_t t = 0; t < n; ++t) c.pinv[size_t(c.perm[size_t(t)])] = t;
        const size_t kw = (size_t(k) + 31) / 32;
        c.pcols.assign(size_t(n - k) * kw, 0u);
        for (int32_t b = 0; b < n - k; ++b) {
            const uint64_t *row = M.data() + size_t(pivot_row[size_t(c.perm[size_t(k + b)])]) * W;
            uint32_t *col = c.pcols.data() + size_t(b) * kw;
            for (int32_t a = 0; a < k; ++a) {
                int32_t fa = c.perm[size_t(a)];
                if ((row[fa >> 6] >> (fa & 63)) & 1u) col[a >> 5] |= 1u << (a & 31);
            }
        }
    } catch (...) {
        return LDPC_ERR_NOMEM;
    }
    c.rank = rank;
    c.k = k;
    c.has_G = true;
    c.bound_G = false;   // the device image (if any) predates G
    return LDPC_OK;
}

ldpc_status ldpc_code_query(const ldpc_code *code, ldpc_code_info *info) {
    if (!code || !info) return LDPC_ERR_ARG;
    info->n = code->n; info->m = code->m; info->k = code->k; info->rank = code->rank;
    info->nnz = code->nnz; info->max_row_deg = code->max_row_deg; info->max_col_deg = code->max_col_deg;
    info->wc = code->wc; info->wr = code->wr; info->gallager = code->gallager;
    info->design_rate = code->design_rate;
    info->device_bytes = ldpc::compute_layout(*code, code->has_G).total;
    return LDPC_OK;
}

ldpc_status ldpc_code_copy_H(const ldpc_code *code, uint8_t *dense) {
    if (!code || !dense) return LDPC_ERR_ARG;
    std::memset(dense, 0, size_t(code->m) * size_t(code->n));
    for (int32_t r = 0; r < code->m; ++r)
        for (int32_t e = code->row_ptr[r]; e < code->row_ptr[r + 1]; ++e)
            dense[size_t(r) * code->n + size_t(code->col_idx[e])] = 1;
    return LDPC_OK;
}

ldpc_status ldpc_code_copy_csr(const ldpc_code *code, int32_t *row_ptr, int32_t *col_idx) {
    if (!code || !row_ptr || (!col_idx && code->nnz)) return LDPC_ERR_ARG;
    std::copy(code->row_ptr.begin(), code->row_ptr.end(), row_ptr);
    std::copy(code->col_idx.begin(), code->col_idx.end(), col_idx);
    return LDPC_OK;
}

ldpc_status ldpc_code_copy_perm(const ldpc_code *code, int32_t *perm) {
    if (!code || !perm) return LDPC_ERR_ARG;
    if (!code->has_G) return LDPC_ERR_STATE;
    std::copy(code->perm.begin(), code->perm.end(), perm);
    return LDPC_OK;
}

ldpc_status ldpc_code_copy_P(const ldpc_code *code, uint32_t *p) {
    if (!code || !p) return LDPC_ERR_ARG;
    if (!code->has_G) return LDPC_ERR_STATE;
    std::copy(code->pcols.begin(), code->pcols.end(), p);
    return LDPC_OK;
}

ldpc_status ldpc_code_bind_device(ldpc_code *code, void *d_buf, size_t bytes, void *stream) {
    if (!code || !d_buf) return LDPC_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(d_buf) & 255u) return LDPC_ERR_ARG;
    ldpc::DeviceLayout L = ldpc::compute_layout(*code, code->has_G);
    if (bytes < L.total) return LDPC_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char *base = static_cast<char *>(d_buf);
    auto put = [&](size_t off, const void *src, size_t nbytes) -> bool {
        if (nbytes == 0) return true;
        return cudaMemcpyAsync(base + off, src, nbytes, cudaMemcpyHostToDevice, s) == cudaSuccess;
    };
    // P transposed for the encoder: pt[w][b] = word w of parity column b, columns
    // padded with zeros to a multiple of kEncColTile.
    std::vector<uint32_t> pt;
    auto put_pt = [&](size_t off) -> bool {
        const size_t kw = (size_t(code->k) + 31) / 32, npar = size_t(code->n - code->k);
        const size_t npp = (npar + ldpc::kEncColTile - 1) / ldpc::kEncColTile * ldpc::kEncColTile;
        pt.assign(kw * npp, 0u);
        for (size_t b = 0; b < npar; ++b)
            for (size_t w = 0; w < kw; ++w) pt[w * npp + b] = code->pcols[b * kw + w];
        return put(off, pt.data(), sizeof(uint32_t) * pt.size());
    };
    bool ok = put(L.row_ptr, code->row_ptr.data(), sizeof(int32_t) * code->row_ptr.size()) &&
              put(L.col_idx, code->col_idx.data(), sizeof(int32_t) * code->col_idx.size()) &&
              put(L.var_ptr, code->var_ptr.data(), sizeof(int32_t) * code->var_ptr.size()) &&
              put(L.var_edges, code->var_edges.data(), sizeof(int32_t) * code->var_edges.size());
    std::vector<int32_t> lidx, vpos;
    int32_t xcap = 0;      // exact exchange-region capacity (0: no exchange view)
    if (ok && code->gallager && code->wc >= 2) {
        // Band view: edge (band b >= 1, position p) of row b*mb + p/wr is CSR edge
        // b*n + p (ldpc_make_H orders rows band-major, slots in pi_b order).
        const int32_t n = code->n, wc = code->wc;
        const size_t lbase = ldpc::band_L_byte_offset(n, wc);
        lidx.resize(size_t(wc - 1) * size_t(n));
        vpos.resize(size_t(wc - 1) * size_t(n));
        // (row, element) order of every band >= 1: bank-balanced for the
        // check phase's gathers (ldpc::bank_balance_rows); E's check-major
        // slot (band_vpos) and both offset views follow that order
        std::vector<int32_t> rel(size_t(wc - 1) * size_t(n));
        for (int32_t b = 1; b < wc; ++b)
            for (int32_t p = 0; p < n; ++p) rel[size_t(b - 1) * n + p] = 4 * code->col_idx[size_t(b) * n + p];
        if (!std::getenv("LDPC_NO_BANKOPT")) ldpc::bank_balance_rows(n, wc, code->wr, rel);
        for (int32_t b = 1; b < wc; ++b)
            for (int32_t p = 0; p < n; ++p) {
                const int32_t x = rel[size_t(b - 1) * n + p];
                lidx[size_t(b - 1) * n + p] = int32_t(lbase) + x;
                vpos[size_t(x / 4) * (wc - 1) + (b - 1)] = int32_t(4 * (size_t(b - 1) * n + p));
            }
        ok = put(L.band_lidx, lidx.data(), sizeof(int32_t) * lidx.size()) &&
             put(L.band_vpos, vpos.data(), sizeof(int32_t) * vpos.size());
        std::vector<uint16_t> l16;
        if (ok && n <= 16383) {
            l16.resize(rel.size());
            for (size_t e = 0; e < rel.size(); ++e) l16[e] = uint16_t(rel[e]);
            ok = put(L.band_lidx16, l16.data(), sizeof(uint16_t) * l16.size());
        }
        const int C = ldpc::band_cluster_size(n, wc, code->wr);
        if (ok && C > 0) {
            // CTA q of a cluster owns band rows [q mbq, (q+1) mbq) of every band and
            // the variables [q nq, (q+1) nq) of its band-0 rows.  Its shared image:
            // E_hi [(b-1)][local row][j] then L [local variable].
            const int32_t wr = code->wr, mb = n / wr, mbq = mb / C, nq = n / C;
            const int32_t lbase_c = (wc - 1) * mbq * wr * 4;
            for (int32_t b = 1; b < wc; ++b)
                for (int32_t p = 0; p < n; ++p) {
                    const int32_t v = code->col_idx[size_t(b) * n + p];
                    const int32_t row_owner = (p / wr) / mbq, var_owner = v / nq;
                    lidx[size_t(b - 1) * n + p] =
                        row_owner == var_owner ? lbase_c + 4 * (v - var_owner * nq) : ~v;
                    const int32_t e_local = 4 * ((b - 1) * mbq * wr + (p - row_owner * mbq * wr));
                    vpos[size_t(v) * (wc - 1) + (b - 1)] =
                        row_owner == var_owner ? e_local : ~int32_t((b - 1) * n + p);
                }
            ok = put(L.cband_lidx, lidx.data(), sizeof(int32_t) * lidx.size()) &&
                 put(L.cband_vpos, vpos.data(), sizeof(int32_t) * vpos.size());
        }
        const int X = ldpc::xband_cluster_size(n, wc, code->wr);
        if (ok && X > 0) {
            std::vector<uint16_t> ridx, sidx;
            std::vector<int32_t> seg;
            xcap = ldpc::xband_tables(*code, X, ridx, sidx, seg);
            if (xcap <= ldpc::kXbandMaxCapacity)
                ok = put(L.xband_ridx, ridx.data(), sizeof(uint16_t) * ridx.size()) &&
                     put(L.xband_sidx, sidx.data(), sizeof(uint16_t) * sidx.size()) &&
                     put(L.xband_seg, seg.data(), sizeof(int32_t) * seg.size());
        }
    }
    bool asm_ok = false;
    if (ok && code->has_G) {
        std::vector<uint32_t> tab;
        asm_ok = ldpc::assemble_table(*code, tab);
        ok = put(L.perm, code->perm.data(), sizeof(int32_t) * code->perm.size()) &&
             put(L.pinv, code->pinv.data(), sizeof(int32_t) * code->pinv.size()) &&
             put_pt(L.pt) && (!asm_ok || put(L.asmtab, tab.data(), sizeof(uint32_t) * tab.size()));
    }
    // The host vectors are pageable: cudaMemcpyAsync from pageable memory is
    // staged synchronously, so they may be reused as soon as the call returns.
    if (!ok) return LDPC_ERR_CUDA;
    code->d_buf = d_buf;
    code->d_bytes = bytes;
    code->layout = L;
    code->bound_G = code->has_G;
    ldpc::DeviceCode &D = code->dev;
    D.n = code->n; D.m = code->m; D.k = code->has_G ? code->k : 0; D.nnz = code->nnz;
    D.max_row_deg = code->max_row_deg; D.max_col_deg = code->max_col_deg;
    D.regular_row = code->regular_row; D.regular_col = code->regular_col;
    D.kw = code->has_G ? (code->k + 31) / 32 : 0;
    D.nw = (code->n + 31) / 32;
    D.row_ptr = reinterpret_cast<const int32_t *>(base + L.row_ptr);
    D.col_idx = reinterpret_cast<const int32_t *>(base + L.col_idx);
    D.var_ptr = reinterpret_cast<const int32_t *>(base + L.var_ptr);
    D.var_edges = reinterpret_cast<const int32_t *>(base + L.var_edges);
    D.perm = code->has_G ? reinterpret_cast<const int32_t *>(base + L.perm) : nullptr;
    D.pinv = code->has_G ? reinterpret_cast<const int32_t *>(base + L.pinv) : nullptr;
    D.gallager = code->gallager; D.wc = code->wc; D.wr = code->wr;
    D.mb = code->gallager ? code->n / code->wr : 0;
    D.band_lidx = (code->gallager && code->wc >= 2) ? reinterpret_cast<const int32_t *>(base + L.band_lidx) : nullptr;
    D.band_vpos = (code->gallager && code->wc >= 2) ? reinterpret_cast<const int32_t *>(base + L.band_vpos) : nullptr;
    D.band_lidx16 = (code->gallager && code->wc >= 2 && code->n <= 16383)
                        ? reinterpret_cast<const uint16_t *>(base + L.band_lidx16) : nullptr;
    D.cluster = (code->gallager && code->wc >= 2) ? ldpc::band_cluster_size(code->n, code->wc, code->wr) : 0;
    D.cband_lidx = D.cluster ? reinterpret_cast<const int32_t *>(base + L.cband_lidx) : nullptr;
    D.cband_vpos = D.cluster ? reinterpret_cast<const int32_t *>(base + L.cband_vpos) : nullptr;
    D.xcluster = (code->gallager && code->wc >= 2 && xcap > 0 && xcap <= ldpc::kXbandMaxCapacity)
                     ? ldpc::xband_cluster_size(code->n, code->wc, code->wr) : 0;
    D.xcap = D.xcluster ? xcap : 0;
    D.xrows = D.xcluster ? ldpc::xband_rows_host(code->n / code->wr / D.xcluster) : 0;
    D.xslots = (D.xcluster == 16 && ldpc::xband2_fits(code->n, code->wc, code->wr) &&
                ldpc::xband2_smem_bytes(code->n, code->wc, code->wr, 16, D.xcap) + 1024 <= 227 * 1024) ? 2 : 1;
    D.xband_ridx = D.xcluster ? reinterpret_cast<const uint16_t *>(base + L.xband_ridx) : nullptr;
    D.xband_sidx = D.xcluster ? reinterpret_cast<const uint16_t *>(base + L.xband_sidx) : nullptr;
    D.xband_seg = D.xcluster ? reinterpret_cast<const int32_t *>(base + L.xband_seg) : nullptr;
    D.pt = code->has_G ? reinterpret_cast<const uint32_t *>(base + L.pt) : nullptr;
    D.asmtab = (code->has_G && asm_ok) ? reinterpret_cast<const uint32_t *>(base + L.asmtab) : nullptr;
    D.npar_pad = code->has_G ? (code->n - code->k + ldpc::kEncColTile - 1) / ldpc::kEncColTile * ldpc::kEncColTile : 0;
    return LDPC_OK;
}

void ldpc_code_free(ldpc_code *code) { delete code; }

// Eq. 9, corrected (reading Q6).
ldpc_status ldpc_partition(int64_t l, int32_t nproc, int64_t *counts, int64_t *displs) {
    if (l < 0 || nproc < 1 || !counts || !displs) return LDPC_ERR_ARG;
    const int64_t base = l / nproc, extra = l % nproc;
    int64_t off = 0;
    for (int32_t q = 0; q < nproc; ++q) {
        counts[q] = base + (q < extra ? 1 : 0);
        displs[q] = off;
        off += counts[q];
    }
    return LDPC_OK;
}

}  // extern "C"
