// ldpc_internal.h -- library-internal structures shared by the host code
// (host_code.cpp) and the CUDA kernels (*.cu).  Not part of the ABI; the
// oracle never includes it.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "../../include/ldpc.h"

namespace ldpc {

constexpr int kMaxCheckDegree = 32;   // generic-kernel limit (register arrays)
constexpr int kEncColTile = 128;      // parity columns per encoder CTA tile
constexpr float kLlrClamp = 30.0f;    // reading Q7: R and L_vc clamped to +-30
// reading Q7: |E_cv| <= 2 atanh(1 - 1e-12) = ln(2e12 - 1) = 28.32416830...
constexpr float kEMax = 28.3241683f;

// Offsets (bytes) of the arrays inside the caller's device buffer.
struct DeviceLayout {
    size_t row_ptr = 0;    // int32 [m+1]       check -> first edge (CSR)
    size_t col_idx = 0;    // int32 [nnz]       edge  -> variable
    size_t var_ptr = 0;    // int32 [n+1]       variable -> first slot in var_edges
    size_t var_edges = 0;  // int32 [nnz]       edges of each variable, ascending check
    size_t perm = 0;       // int32 [n]         (after make_G)
    size_t pinv = 0;       // int32 [n]         inverse of perm: position of column v in [m | mP]
    size_t pt = 0;         // uint32 [kw][npar_pad] P by message word: bit i of [w][b] = P[32w+i][b]
    size_t asmtab = 0;     // uint32 [nw][16] encoder assemble: per codeword word, its info/parity bit
                           // masks, the first info bit's index and the expand masks (host_code.cpp)
    // Gallager band view (ldpc_make_H codes only), used by the band kernel:
    size_t band_lidx = 0;  // int32 [(wc-1)*n]  edge (band b>=1, position p) -> byte offset of L[pi_b[p]]
    size_t band_vpos = 0;  // int32 [n*(wc-1)]  variable v, band b>=1 -> byte offset of its E in E_hi
    size_t band_lidx16 = 0; // uint16 [(wc-1)*n] 4*v (n <= 16383): band_lidx - L base, half the bytes
    // Cluster band view (frames too large for one SM: C CTAs share a frame):
    // value >= 0: byte offset in the owning CTA's shared memory; value < 0:
    // ~(element index) into the frame's global copy (Lg for lidx, Eg for vpos).
    size_t cband_lidx = 0; // int32 [(wc-1)*n]
    size_t cband_vpos = 0; // int32 [n*(wc-1)]
    // Exchange cluster view (spa_cluster.cu; C = xband_cluster_size CTAs per
    // frame exchange message segments with bulk DSMEM copies).  Slots are byte
    // offsets into the owning CTA's message buffer (see spa_cluster.cu):
    size_t xband_ridx = 0; // uint16 [(wc-1)*n]  band edge (b>=1, p) -> slot in its row owner's buffer
    size_t xband_sidx = 0; // uint16 [n*(wc-1)]  variable v, band b>=1 -> slot in its variable owner's buffer
    size_t xband_seg = 0;  // int32 [3][C C H (wc-1) H] var-region offset, row-region offset, bytes per segment
    size_t total = 0;
};

// Plain-old-data view of a bound code, passed by value to kernels.
struct DeviceCode {
    int32_t n, m, k, nnz;
    int32_t max_row_deg, max_col_deg;
    int32_t regular_row;   // every check has degree max_row_deg
    int32_t regular_col;   // every variable has degree max_col_deg
    int32_t kw, nw;        // ceil(k/32), ceil(n/32)
    const int32_t *row_ptr;
    const int32_t *col_idx;
    const int32_t *var_ptr;
    const int32_t *var_edges;
    const int32_t *perm;
    const int32_t *pinv;
    const uint32_t *pt;
    const uint32_t *asmtab;         // null unless both halves of perm ascend (every make_G here)
    int32_t npar_pad;               // n - k rounded up to kEncColTile
    int32_t gallager, wc, wr, mb;   // band structure (mb = n / wr rows per band)
    const int32_t *band_lidx;
    const int32_t *band_vpos;
    const uint16_t *band_lidx16;    // null when n > 16383
    int32_t cluster;               // C of the cluster band view (0: none)
    const int32_t *cband_lidx;
    const int32_t *cband_vpos;
    int32_t xcluster;              // C of the exchange cluster view (0: none)
    int32_t xslots;                // 2: the view serves the two-slot kernel (xband2_kernel)
    int32_t xrows;                 // rows per compute thread (H) the view's tables were built for
    int32_t xcap;                  // message region capacity (floats, multiple of 4)
    const uint16_t *xband_ridx;
    const uint16_t *xband_sidx;
    const int32_t *xband_seg;
};

// Cluster size for the cluster band kernel: the smallest power of two C <= 16
// with mb % C == 0 whose per-CTA share (E of bands >= 1 + L) fits 200 KB; 0
// when a frame fits one SM (or no such C exists).
inline int band_cluster_size(int32_t n, int32_t wc, int32_t wr) {
    const size_t one = size_t(wc) * size_t(n) * 4;
    if (one + 1024 <= 227 * 1024) return 0;
    for (int C = 2; C <= 16; C *= 2)
        if ((n / wr) % C == 0 && one / C <= 200 * 1024) return C;
    return 0;
}

// Exchange cluster kernel (spa_cluster.cu): C CTAs per frame, CTA q owns
// mbq = n / wr / C rows of every band and the nq = mbq wr variables of its
// band-0 rows.  Compute threads and rows per thread (= V-phase chunks H) of a
// CTA (the launch adds one producer warp):
constexpr int xband_rows_per_thread(int32_t mbq) {
    const int b0 = mbq > 0 ? (mbq + 1023) / 1024 : 1;
    return b0 == 3 ? 4 : b0;                      // instantiated: 1, 2, 4
}
constexpr int xband_threads(int32_t mbq) {
    const int b0 = xband_rows_per_thread(mbq);
    return ((mbq + b0 - 1) / b0 + 31) / 32 * 32;
}
// Host-side choice of rows per thread (LDPC_XBAND_H raises it: experiments;
// the compile-time-n kernels assume the default and are skipped then).
inline int xband_rows_host(int32_t mbq) {
    int h = xband_rows_per_thread(mbq);
    if (const char *e = std::getenv("LDPC_XBAND_H")) h = std::max(h, std::atoi(e));
    return h == 3 ? 4 : h;
}
inline int xband_threads_host(int32_t mbq) {
    const int b0 = xband_rows_host(mbq);
    return ((mbq + b0 - 1) / b0 + 31) / 32 * 32;
}
// Region capacity (floats): (wc-1) nq edge slots plus the 16-byte padding of
// its H x (wc-1) H x C segments -- worst case 3 floats each (shared-memory
// sizing), expected 1.5 (cluster-size choice).  The exact capacity comes
// from the tables at bind time (xband_tables); a code whose layout would
// overflow the 16-bit byte slots gets no exchange view.
inline int32_t xband_capacity_bound(int32_t n, int32_t wc, int32_t wr, int32_t C, int pad_x2 = 6) {
    const int32_t mbq = n / wr / C, nq = mbq * wr;
    const int32_t H = xband_rows_host(mbq);
    return ((wc - 1) * nq + (pad_x2 * H * H * (wc - 1) * C + 1) / 2 + 3) & ~3;
}
constexpr int32_t kXbandMaxCapacity = 16383;     // floats: byte slots < 65536
// Shared memory of the kernel for region capacity `cap`: two regions + the
// CTA's two 16-bit slot tables + barriers and flags.
inline size_t xband_smem_bytes(int32_t n, int32_t wc, int32_t wr, int32_t C, int32_t cap, int32_t rows = 0) {
    const size_t mbq = size_t(n / wr / C), nq = mbq * size_t(wr);
    const size_t H = size_t(rows > 0 ? rows : xband_rows_host(int32_t(mbq)));
    return 2 * size_t(cap) * 4 + 2 * size_t(wc - 1) * nq * 2 + 16 + 8 * (2 + H + size_t(wc - 1) * H) + 4 * size_t(C);
}
// Cluster size of a code's exchange view.  Frames larger than one SM: the
// smallest power of two C <= 16 with mb % C == 0 whose shared memory fits one
// CTA and whose expected region fits 16-bit byte slots (throughput: C5 -> 8).
// Frames that fit one SM: the C of least modelled stream latency (below)
// (latency: stream mode and small batches, C4 -> 9, C3 -> 6).  0: no view.
inline bool xband_fits(int32_t n, int32_t wc, int32_t wr, int C) {
    if ((n / wr) % C) return false;
    if (xband_capacity_bound(n, wc, wr, C, 3) > kXbandMaxCapacity) return false;
    if (xband_threads_host(n / wr / C) + 32 > 1024) return false;      // + the producer warp
    return xband_smem_bytes(n, wc, wr, C, xband_capacity_bound(n, wc, wr, C)) + 1024 <= 227 * 1024;
}
inline bool band_frame_fits_sm(int32_t n, int32_t wc) { return size_t(wc) * size_t(n) * 4 + 1024 <= 227 * 1024; }
// Two-slot exchange kernel (xband2_kernel): four regions + shared tables.
inline size_t xband2_smem_bytes(int32_t n, int32_t wc, int32_t wr, int32_t C, int32_t cap) {
    const size_t nq = size_t(n / wr / C) * size_t(wr);
    // four regions + the two slot tables as 32-bit offsets + barriers, flags
    return 4 * size_t(cap) * 4 + 2 * size_t(wc - 1) * nq * 4 + 16 + 2 * 8 * (3 + size_t(wc - 1)) + 2 * 4 * size_t(C);
}
// Frames larger than one SM whose 16-CTA view fits two frames per CTA with one
// row per thread use 16-CTA clusters and two frames in flight (the (3,6)
// instantiation; C5: 144 SMs instead of 120 and the exchange latency hidden).
inline bool xband2_fits(int32_t n, int32_t wc, int32_t wr) {
    constexpr int C = 16;
    if (wc != 3 || wr != 6 || (n / wr) % C) return false;
    const int32_t mbq = n / wr / C;
    if (xband_rows_host(mbq) != 1 || xband_threads_host(mbq) + 32 > 768) return false;
    return xband2_smem_bytes(n, wc, wr, C, xband_capacity_bound(n, wc, wr, C)) + 1024 <= 227 * 1024;
}
inline int xband_cluster_size(int32_t n, int32_t wc, int32_t wr) {
    if (wc < 2 || wr < 1 || n % wr) return 0;
    if (const char *e = std::getenv("LDPC_XBAND_C")) {          // experiments: force a cluster size
        const int C = std::atoi(e);
        return (C >= 2 && C <= 16 && xband_fits(n, wc, wr, C)) ? C : 0;
    }
    if (band_frame_fits_sm(n, wc)) {
        // latency view: the C dividing the band rows (<= 16, >= 32 rows per
        // CTA) minimising 0.32 us x rows per CTA + 10.4 us x C -- the stream-
        // mode latency model fitted on B200 (C4: C = 4 190 us, 6 145, 9 128,
        // 12 135, 15 145; C3 R1/2: C = 2 103 us, 3 87, 6 84, 9 98)
        const int32_t mb = n / wr;
        int best = 0;
        double best_cost = 1e30;
        for (int C : {2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16}) {      // instantiated sizes
            if (mb % C || mb / C < 32 || !xband_fits(n, wc, wr, C)) continue;
            const double cost = 0.32 * (mb / C) + 10.4 * C;
            if (cost < best_cost) {
                best_cost = cost;
                best = C;
            }
        }
        return best;
    }
    if (!std::getenv("LDPC_XBAND_1SLOT") && xband2_fits(n, wc, wr) && xband_fits(n, wc, wr, 16)) return 16;
    for (int C = 2; C <= 16; C *= 2)
        if (xband_fits(n, wc, wr, C)) return C;
    return 0;
}

// Shared-memory image of one frame in the band kernel (floats):
//   E_hi[(wc-1) n] (bands 1.., check-major: band b row r slot j at (b-1) n + r wr + j)
//   L[n]  (posterior, log2 units)      R[n] (channel LLR, log2 units; optional)
inline size_t band_L_byte_offset(int32_t n, int32_t wc) { return size_t(wc - 1) * size_t(n) * 4; }

}  // namespace ldpc

struct ldpc_code {
    int32_t n = 0, m = 0, k = -1, rank = -1, nnz = 0;
    int32_t max_row_deg = 0, max_col_deg = 0;
    int32_t wc = 0, wr = 0, gallager = 0;
    int32_t regular_row = 0, regular_col = 0;
    double design_rate = 0.0;
    std::vector<int32_t> row_ptr, col_idx;     // H as CSR, check-major edge ids
    std::vector<int32_t> var_ptr, var_edges;   // CSC view: edge ids per variable
    std::vector<int32_t> perm;                 // [free cols asc, pivot cols asc]
    std::vector<int32_t> pinv;                 // pinv[perm[t]] = t
    std::vector<uint32_t> pcols;               // (n-k) x kw
    bool has_G = false;
    // device binding
    void *d_buf = nullptr;
    size_t d_bytes = 0;
    bool bound_G = false;
    ldpc::DeviceLayout layout;
    ldpc::DeviceCode dev{};
};

namespace ldpc {
// Launch-configuration queries, cached per (device, kernel, block size,
// dynamic smem[, cluster size]) so that repeated ldpc_decode calls (stream
// mode issues one per frame) make no driver queries.  The dynamic
// shared-memory attribute of a kernel is only ever raised.  -1 on failure.
int device_attribute(int attr);                       // cudaDeviceAttr of the current device
bool ensure_smem_attribute(const void *kernel, size_t smem, bool nonportable_cluster = false);
int occupancy_blocks(const void *kernel, int threads, size_t smem);
int occupancy_clusters(const void *kernel, int threads, size_t smem, int cluster);

DeviceLayout compute_layout(const ldpc_code &c, bool with_G);
int32_t xband_tables(const ldpc_code &c, int C, std::vector<uint16_t> &ridx, std::vector<uint16_t> &sidx,
                     std::vector<int32_t> &seg);

// Launch plan of the Gallager band kernel (spa_band.cu).
struct BandPlan {
    void *kernel = nullptr;
    int threads = 0;
    int grid = 0;
    int64_t capacity = 0;       // frames decoded concurrently (SMs x CTAs per SM)
    size_t smem = 0;
    bool r_in_smem = false;
    bool vm = false;            // E of bands >= 1 stored variable-major
    int mode = 0;               // kernel MODE: 0 check-major, 1 VM, 2 VM + 16-bit offsets
    int lpr = 1;                // lanes per check row (2: lane-pair kernel, small batches)
    int b0 = 1;                 // band-0 rows per thread (threads = row stride)
    size_t ws_bytes = 0;
};
// false when the code is not eligible (not from ldpc_make_H, unsupported
// (wc, wr), n % 4 != 0, or the frame does not fit one SM's shared memory).
// variant: 0 auto, 3 check-major E, 4 variable-major E.
// lane_pairs: allow the LPR = 2 kernels (the fused simulate path has none).
bool band_plan(const ldpc_code &c, int64_t frames, bool et, int variant, BandPlan &p, int max_iter = 50,
               bool lane_pairs = true);
// band_kernel instantiation with n compiled in (spa_band_fixed.cu), or nullptr.
// lpr: lanes per check row (1, or 2 for the lane-pair instantiations).
void *pick_band_kernel_fixed(int n, int wr, int wc, int b0, bool et, int mode, int max_iter, int lpr = 1);
int band_fixed_b0(int n, int wr, int wc, int64_t frames, int sms);
bool band_fixed_vm(int n, int wr, int wc);
// Whether the band decoder runs without psi regime votes for this code and
// iteration count (few-iteration configs with a compile-time-n kernel).
inline bool band_novote(int n, int wr, int wc, int max_iter, bool et) {
    if (et || max_iter > 20 || std::getenv("LDPC_VOTES") || std::getenv("LDPC_NO_NFIX")) return false;
    return (n == 96 && wr == 6 && wc == 3) || (n == 1032 && wr == 12 && (wc == 3 || wc == 6 || wc == 9));
}
ldpc_status band_launch(const ldpc_code &c, const BandPlan &p, const float *llr, int64_t frames,
                        const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                        void *ws, size_t ws_bytes, void *stream);

// Launch plan of the lane-per-edge small-batch decoder (spa_edge.cu; variant 8).
struct EdgePlan {
    void *kernel = nullptr;
    int G = 0;                  // lanes per check row
    int kc = 0;                 // rows per lane group
    int threads = 0;
    int grid = 0;
    int64_t capacity = 0;       // frames decoded concurrently
    size_t smem = 0;
};
// false when the code has a row of degree > 32 or a frame's E, L, R do not fit
// one SM's shared memory.
bool edge_plan(const ldpc_code &c, int64_t frames, bool et, int max_iter, EdgePlan &p);
ldpc_status edge_launch(const ldpc_code &c, const EdgePlan &p, const float *llr, int64_t frames,
                        const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                        void *stream);

// Launch plan of the cluster band kernel (frames larger than one SM).
struct ClusterPlan {
    void *kernel = nullptr;
    int cluster = 0;
    int threads = 0;
    int grid = 0;
    size_t smem = 0;
    int64_t slot_floats = 0;
    size_t ws_bytes = 0;
};
bool cluster_plan(const ldpc_code &c, int64_t frames, bool et, ClusterPlan &p);

// Launch plan of the exchange cluster kernel (spa_cluster.cu; variant 7).
struct XClusterPlan {
    void *kernel = nullptr;
    int cluster = 0;
    int threads = 0;
    int grid = 0;
    int64_t capacity = 0;       // frames decoded concurrently (co-resident clusters)
    size_t smem = 0;
    size_t ws_bytes = 0;
    int slots = 1;              // frames in flight per cluster
    int64_t pairs_capacity() const { return slots == 2 ? capacity / 2 : 0; }
};
// Launch plan of the global-exchange kernel (spa_gexchange.cu; variant 9):
// groups of 16 co-resident CTAs (cooperative launch) on the 16-CTA exchange
// view, two frames in flight per group, segments through L2-resident staging.
struct GXPlan {
    void *kernel = nullptr;
    int threads = 0;
    int grid = 0;
    int groups = 0;
    int64_t capacity = 0;       // frames decoded concurrently
    size_t smem = 0;
    size_t ws_bytes = 0;
    size_t zero_bytes = 0;      // workspace prefix zeroed per launch (arrival / barrier counters)
    size_t off_arrivals = 0, off_gbar = 0, off_stage = 0, off_rws = 0, off_zbyte = 0, off_synd = 0;
};
// max_groups > 0 caps the groups (the tail on the SMs exchange clusters leave
// idle); dependent = launched as the programmatic dependent of the kernel
// before it on the stream (no cooperative attribute, no memset: the caller
// zeroes zero_bytes before the primary launch)
bool gx_plan(const ldpc_code &c, int64_t frames, bool et, GXPlan &p, int max_groups = 0);
ldpc_status gx_launch(const ldpc_code &c, const GXPlan &p, const float *llr, int64_t frames, const ldpc_decode_opts &o,
                      uint32_t *bits, uint8_t *syn, int32_t *iters, float *post, void *ws, size_t ws_bytes,
                      void *stream, bool dependent = false);

// The encoder's parity words on the tensor cores (encode_mma.cu); false when
// the code or batch stays on the INT-pipe kernel (LDPC_ENC_MMA=0/1 forces).
bool encode_parity_mma(const DeviceCode &D, const uint32_t *d_info, uint32_t *d_cw, int64_t frames,
                       cudaStream_t s, cudaError_t *err);

// false unless the bound code has an exchange cluster view, fixed iterations
// and an instantiated (wc, wr, rows-per-thread, C).
bool xcluster_plan(const ldpc_code &c, int64_t frames, bool et, XClusterPlan &p);
ldpc_status xcluster_launch(const ldpc_code &c, const XClusterPlan &p, const float *llr, int64_t frames,
                            const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                            void *ws, size_t ws_bytes, void *stream);
ldpc_status cluster_launch(const ldpc_code &c, const ClusterPlan &p, const float *llr, int64_t frames,
                           const ldpc_decode_opts &o, uint32_t *bits, uint8_t *syn, int32_t *iters, float *post,
                           void *ws, size_t ws_bytes, void *stream);
}  // namespace ldpc
