/*
 * ldpc.h -- C ABI of libldpc_b200.so: batched Sum-Product LDPC decoding on
 * NVIDIA B200 (sm_100a), after arXiv 2201.04265 ("distributed LDPC encoding
 * and Sum-Product decoding with MPI").  Citations: P:<line> = a line of the
 * paper text, S:<line> = a line of the CPU-program spec;
 * "reading Qn" = an interpretation listed in DESIGN.md.
 *
 * General contract
 *  - Every call returns ldpc_status; nothing throws or aborts across the ABI.
 *  - Bits are packed LSB-first into uint32 words.  A frame of b bits occupies
 *    ceil(b/32) words; pad bits are written 0 and ignored on input.
 *  - Every length-n vector is in H's column order (the variable-node order of
 *    the Tanner graph).  The k information bits of a codeword sit at
 *    positions perm[0..k) (ldpc_code_copy_perm), in message order.
 *  - LLRs are L = ln(p(bit=1)/p(bit=0)), positive favours 1 (Eq. 4, P:121-125,
 *    with the missing logarithm restored: reading Q1); z = 1 iff L >= 0
 *    (Eq. 8).
 *  - Device pointers (d_*) are caller-owned device memory (PyTorch allocates
 *    everything; the library never allocates device memory).  Host pointers
 *    are caller-owned host memory.  `stream` is a cudaStream_t passed as void*
 *    (NULL = the legacy default stream).
 *  - Device calls are asynchronous: argument errors and launch errors are
 *    returned synchronously (LDPC_ERR_ARG / LDPC_ERR_CUDA); device faults
 *    surface at the caller's next synchronisation of `stream`.
 *  - An ldpc_code is immutable after ldpc_make_G + ldpc_code_bind_device, and
 *    may then be used concurrently from several streams.
 */
#ifndef LDPC_B200_H
#define LDPC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LDPC_OK = 0,
    LDPC_ERR_ARG = 1,            /* bad argument (NULL, out of range, bad size)          */
    LDPC_ERR_NOT_DIVISIBLE = 2,  /* wr does not divide n (band construction)       */
    LDPC_ERR_NO_INFO_BITS = 3,   /* rank(H) == n, so k == 0                       */
    LDPC_ERR_DIM = 4,            /* dimension mismatch               */
    LDPC_ERR_STATE = 5,          /* call out of order (e.g. encode before make_G / bind)  */
    LDPC_ERR_UNSUPPORTED = 6,    /* e.g. a check degree > 32                               */
    LDPC_ERR_CUDA = 7,           /* a CUDA runtime call failed                             */
    LDPC_ERR_NOMEM = 8           /* host allocation failed                                 */
} ldpc_status;

typedef struct ldpc_code ldpc_code;   /* opaque; owns host memory only */

typedef struct {
    int32_t n;              /* code length (variable nodes)                        */
    int32_t m;              /* parity checks (rows of H, check nodes)              */
    int32_t k;              /* information bits = n - rank(H); -1 before make_G    */
    int32_t rank;           /* GF(2) rank of H; -1 before make_G                   */
    int32_t nnz;            /* Tanner-graph edges = ones of H                      */
    int32_t max_row_deg;    /* max check degree                                    */
    int32_t max_col_deg;    /* max variable degree                                 */
    int32_t wc, wr;         /* Gallager column/row weight, 0 for an external H     */
    int32_t gallager;       /* 1 if built by ldpc_make_H (band structure known)    */
    double design_rate;     /* 1 - wc/wr, or 1 - m/n for an external H      */
    size_t device_bytes;    /* bytes ldpc_code_bind_device needs                   */
} ldpc_code_info;

typedef struct {
    int32_t max_iter;       /* >= 1: SPA iterations ("predefined number")   */
    int32_t early_term;     /* 0: run exactly max_iter (paper); 1: stop after the  */
                            /* first iteration t >= 1 whose z^t has zero syndrome  */
                            /* (reading Q11 / c6)                                  */
    int32_t variant;        /* 0 = auto; see ldpc_decode                           */
    int32_t reserved;
} ldpc_decode_opts;

/* ---------------------------------------------------------------- codes */

/* Regular (wc, wr) Gallager parity-check matrix (band
 * construction S:52): wc bands of n/wr rows; band 0 row c has ones at columns
 * [c*wr, (c+1)*wr); band b >= 1 is the column permutation pi_b of band 0
 * drawn by Fisher-Yates (i = n-1..1, j = U(i+1), swap) from SplitMix64(seed),
 * U by rejection (reading Q12).  Requires 1 <= wc < wr, n > 0.
 * Errors: LDPC_ERR_NOT_DIVISIBLE if n % wr != 0; LDPC_ERR_ARG otherwise.
 * *out receives a new code (free with ldpc_code_free). */
ldpc_status ldpc_make_H(int32_t n, int32_t wc, int32_t wr, uint64_t seed, ldpc_code **out);

/* An external parity-check matrix given as CSR (P:4: "Any Binary Parity Check
 * matrix ... can be used"): row_ptr[m+1], col_idx[nnz] (host).  Duplicate
 * entries in a row are rejected (LDPC_ERR_ARG); rows may be empty; check
 * degrees must be <= 32 (LDPC_ERR_UNSUPPORTED). */
ldpc_status ldpc_code_from_csr(int32_t m, int32_t n, const int32_t *row_ptr,
                               const int32_t *col_idx, ldpc_code **out);

/* make_G on the GPU: the same elimination and result as
 * ldpc_make_G (rank, k, perm, P bit-identical: the reduced row echelon form is
 * unique), run as one cooperative kernel over H bit-packed in the caller's
 * device workspace (d_ws, >= ldpc_make_G_device_workspace_bytes, 256-byte
 * aligned; C5: ~1 GB).  Synchronises `stream`; the code's host image is
 * updated as by ldpc_make_G (bind_device again afterwards).  Errors as
 * ldpc_make_G, LDPC_ERR_CUDA on a device failure. */
ldpc_status ldpc_make_G_device_workspace_bytes(const ldpc_code *code, size_t *bytes);
ldpc_status ldpc_make_G_device(ldpc_code *code, void *d_ws, size_t ws_bytes, void *stream);

/* MacKay alist text (P:4): "n m", "max_col_weight
 * max_row_weight", the n column weights, the m row weights, n lines of 1-based
 * row indices per column and m lines of 1-based column indices per row, each
 * zero-padded to the maximum weight ('\n' line ends).
 * write: *len = text length (excluding the NUL).  buf == NULL only queries
 *   *len; otherwise cap must be >= *len + 1 (else LDPC_ERR_DIM).  Index lists
 *   are written in ascending order.
 * from_alist: text[len] (host, not NUL-terminated necessarily); the row lists
 *   define H (rows kept in file order), the column lists must describe the same
 *   matrix and every weight must match (LDPC_ERR_DIM); malformed text
 *   LDPC_ERR_ARG; then as ldpc_code_from_csr. */
ldpc_status ldpc_code_write_alist(const ldpc_code *code, char *buf, size_t cap, size_t *len);
ldpc_status ldpc_code_from_alist(const char *text, size_t len, ldpc_code **out);

/* Generator in standard form (Eq. 2-3): Gauss-Jordan
 * elimination of H over GF(2), columns scanned right to left, pivot = lowest
 * row index >= r (reading Q13).  Sets rank, k = n - rank, perm = [free
 * columns ascending, pivot columns ascending] and P (k x (n-k)) with
 * codeword = [m | m P] scattered by perm.  Host CPU, multi-threaded.
 * Errors: LDPC_ERR_NO_INFO_BITS if k == 0. */
ldpc_status ldpc_make_G(ldpc_code *code);

ldpc_status ldpc_code_query(const ldpc_code *code, ldpc_code_info *info);

/* Host copies for tests: dense H as m*n bytes (0/1, row-major); the column
 * permutation (n int32); P packed column-major by parity bit:
 * (n-k) * ceil(k/32) uint32, word [b][w] bit i = P[32w+i][b]. */
ldpc_status ldpc_code_copy_H(const ldpc_code *code, uint8_t *dense_mxn);
ldpc_status ldpc_code_copy_csr(const ldpc_code *code, int32_t *row_ptr, int32_t *col_idx);
ldpc_status ldpc_code_copy_perm(const ldpc_code *code, int32_t *perm_n);
ldpc_status ldpc_code_copy_P(const ldpc_code *code, uint32_t *p_packed);

/* Copy the code's device image (graph, permutation, packed P) into the
 * caller's device buffer d_buf (>= info.device_bytes, 256-byte aligned),
 * enqueued on `stream`.  d_buf must outlive every encode/decode that uses the
 * code.  Calling it again re-binds.  May be called before ldpc_make_G (then
 * only decoding is available) and again after it. */
ldpc_status ldpc_code_bind_device(ldpc_code *code, void *d_buf, size_t bytes, void *stream);

void ldpc_code_free(ldpc_code *code);
const char *ldpc_status_str(ldpc_status s);

/* ---------------------------------------------------------------- hot path */

/* Encode, Eq. 3 in standard form: for every frame,
 * c[perm[t]] = m_t (t < k) and c[perm[k+b]] = XOR_a m_a P[a][b].
 * d_info: frames * ceil(k/32) uint32 (packed message bits);
 * d_cw:   frames * ceil(n/32) uint32 (packed codeword, H column order).
 * Requires make_G and bind_device after it (else LDPC_ERR_STATE).
 * The parity product runs on the tensor cores (exact int32 dot products of
 * 0/1 bytes, parity = LSB) when ceil(k/32) >= 16 and the batch has at least
 * one 256 x 256 tile per SM, else as a binary GEMM on the INT pipe; the bits
 * are identical.  Launch errors return LDPC_ERR_CUDA. */
ldpc_status ldpc_encode(const ldpc_code *code, const uint32_t *d_info, uint32_t *d_cw,
                        int64_t frames, void *stream);

/* The decoder variant ldpc_decode would run for these arguments (opts->variant
 * 0 resolved): 1 generic on-chip, 2 generic global-state, 3/4 Gallager band
 * kernel (check-/variable-major E), 5 cluster band kernel, 6 band kernel with
 * 16-bit offsets, 7 exchange cluster kernel, 8 lane-per-edge small-batch
 * kernel, 9 global-exchange group kernel.  *variant = 0 and
 * LDPC_ERR_UNSUPPORTED when nothing fits. */
ldpc_status ldpc_decode_variant(const ldpc_code *code, int64_t frames, const ldpc_decode_opts *opts,
                                int32_t *variant);

/* Workspace the chosen decode variant needs for `frames` frames (0 for the
 * on-chip variants; the large-n variants keep per-frame message state in it).
 * When auto resolves to variant 8 for a code the band kernel can decode, the
 * band kernel's workspace is reported, so the same buffer serves
 * ldpc_decode_simulate. */
ldpc_status ldpc_decode_workspace_bytes(const ldpc_code *code, int64_t frames,
                                        const ldpc_decode_opts *opts, size_t *bytes);

/* Batched Sum-Product decoding (flooding schedule of Alg. 1,
 * P:351-369; batch processing P:542-544; stream processing = frames == 1).
 *   d_llr:       frames * n float32 channel LLRs R_v (Eq. 4), clamped to +-30
 *                on load (reading Q7).  16-byte aligned.
 *   d_bits:      frames * ceil(n/32) uint32: hard decisions z (Eq. 8).
 *   d_syndrome_ok: frames uint8: 1 iff H z^T = 0 (Eq. 1).
 *   d_iters:     frames int32: iterations run (max_iter unless early_term).
 *   d_posterior: nullable; frames * n float32 total LLRs L_v (Eq. 7).
 *   d_ws/ws_bytes: workspace, >= ldpc_decode_workspace_bytes().
 * Check update E_cv = (-1)^{d_c} prod sgn(L_v'c) * phi(sum phi(|L_v'c|)),
 * phi(x) = -ln tanh(x/2) (Eq. 5, reading Q2/Q3), L_v'c clamped to
 * +-30, |E_cv| <= E_MAX = 2 atanh(1 - 1e-12) (reading Q7).
 * opts->variant: 0 auto; 1 generic on-chip (team per frame); 2 generic
 * global-state (CTA per frame, any n); 3 Gallager band kernel, check-major E;
 * 4 Gallager band kernel, variable-major E (3 and 4 need an ldpc_make_H code
 * whose frame fits one SM; LDPC_ERR_UNSUPPORTED otherwise); 5 cluster band
 * kernel (ldpc_make_H codes too large for one SM, wr = 6; remote messages
 * through L2-resident global copies; the auto choice for such codes under
 * early termination); 6 = 4 with 16-bit
 * offsets (n <= 16383); 7 exchange cluster kernel (same codes as 5; a
 * cluster of C CTAs per frame trades message segments with bulk DSMEM copies;
 * fixed iterations, wr = 6; no workspace); 8 lane-per-edge kernel (any H with
 * row degree <= 32 whose E, L, R fit one SM's shared memory: a group of
 * 4/8/16/32 lanes per check row, one CTA per frame, no workspace; for batches
 * too small to fill the GPU with one thread per check row); 9 global-exchange
 * kernel (the codes of variant 7's 16-CTA two-frame view: groups of 16
 * co-resident CTAs, cooperative launch, trade segments through L2-resident
 * staging images instead of cluster shared memory, so 144 SMs instead of
 * 112; workspace: staging, counters and R', C5 ~43 MB).  Auto (0): a
 * frame that fits one SM runs the band kernel (one SM per frame) unless the
 * batch is too small to fill the GPU that way, in which case it runs variant
 * 7 with C SMs per frame when the code has that view (lower latency: stream
 * mode, small batches), else variant 8 when there are no more frames than
 * SMs; larger frames run 7, else 5; any other H runs 8 for such batches,
 * else 1 or 2.  Variant 7 on batches of many frame-pair rounds also runs the
 * last frames on variant 9's groups over the SMs its 16-CTA clusters leave
 * idle, launched as the clusters' programmatic dependent in the same call
 * (same results; its workspace is then variant 9's). */
ldpc_status ldpc_decode(const ldpc_code *code, const float *d_llr, int64_t frames,
                        const ldpc_decode_opts *opts, uint32_t *d_bits,
                        uint8_t *d_syndrome_ok, int32_t *d_iters, float *d_posterior,
                        void *d_ws, size_t ws_bytes, void *stream);

/* Fused simulate step (Eq. 4-8): for
 * frames frame0 .. frame0+frames-1 the decoder draws the channel LLRs in its
 * prologue exactly as ldpc_channel(code, seed, frame0, frames, d_cw, sigma)
 * would (same counters, same roundings), decodes them as ldpc_decode with
 * `opts`, and ADDS the frames' counters (as ldpc_count_errors) to
 * d_counters6 -- no frames*n*4-byte LLR buffer, one kernel launch.
 *   d_info: frames*ceil(k/32) uint32 info bits; d_cw: their codewords
 *   (ldpc_encode); d_bits / d_syndrome_ok / d_iters as ldpc_decode; no
 *   posterior.  Workspace: ldpc_decode_workspace_bytes for the same code,
 *   frames and opts.  Gallager (3,6) codes whose frame fits one SM, opts
 *   variant 0/3/4/6 (else LDPC_ERR_UNSUPPORTED); it always runs the band
 *   kernel (bit-identical to ldpc_decode with variant 3/4/6 as resolved for
 *   the same opts, also where ldpc_decode's auto choice is variant 8); needs make_G before
 *   bind_device (LDPC_ERR_STATE); sigma > 0. */
ldpc_status ldpc_decode_simulate(const ldpc_code *code, uint64_t seed, int64_t frame0, int64_t frames,
                                 double sigma, const uint32_t *d_info, const uint32_t *d_cw,
                                 const ldpc_decode_opts *opts, uint32_t *d_bits, uint8_t *d_syndrome_ok,
                                 int32_t *d_iters, int64_t *d_counters6, void *d_ws, size_t ws_bytes,
                                 void *stream);

/* ---------------------------------------------------------------- harness helpers */

/* Info bits (reading c4): word w of frame f = lane w%4 of Philox4x32-10 with
 * key (seed_lo, seed_hi), counter (w/4, f_lo, f_hi, 0); last word masked to k.
 * Frames frame0 .. frame0+frames-1; d_info: frames * ceil(k/32) uint32. */
ldpc_status ldpc_gen_info(uint64_t seed, int64_t frame0, int64_t frames, int32_t k,
                          uint32_t *d_info, void *stream);

/* BPSK (0 -> -1, 1 -> +1) over AWGN of std sigma and the
 * channel LLR R = fp32(clamp(2y/sigma^2, +-30)) (Eq. 4, reading Q1).  Noise:
 * Philox counter (v/4, f_lo, f_hi, 1), Box-Muller in fp64 (reading c4).
 * d_cw: frames * ceil(n/32) uint32; d_llr: frames * n float32. */
ldpc_status ldpc_channel(const ldpc_code *code, uint64_t seed, int64_t frame0, int64_t frames,
                         const uint32_t *d_cw, double sigma, float *d_llr, void *stream);

/* Error counters, ACCUMULATED (+=) into d_counters6 (int64[6]):
 * [0] info-bit errors (decoded bits at perm[0..k) vs d_info), [1] codeword-bit
 * errors (vs d_cw), [2] frame errors (any info-bit error), [3] undetected
 * errors (syndrome_ok but some codeword bit wrong), [4] sum of iterations,
 * [5] frames (SPEC run_ber S:522-530, reading Q14).  Requires make_G. */
ldpc_status ldpc_count_errors(const ldpc_code *code, const uint32_t *d_info,
                              const uint32_t *d_bits, const uint32_t *d_cw,
                              const uint8_t *d_syndrome_ok, const int32_t *d_iters,
                              int64_t frames, int64_t *d_counters6, void *stream);

/* Diagnostics: y[i] = phi(x[i]) with the GENERIC CSR decoder's device phi
 * (spa_decode.cu, variants 1 and 2 only), phi(x) = -ln tanh(x/2) for x >= 0
 * (the log-domain form of Eq. 5's tanh/atanh pair).  For the
 * exhaustive accuracy sweep in tests.  d_x, d_y: count float32 (device). */
ldpc_status ldpc_debug_phi(const float *d_x, float *d_y, int64_t count, void *stream);

/* Diagnostics: the throughput decoders' own phi (every band, exchange-cluster
 * and lane-per-edge kernel, variants 3-8), which works in log2 units:
 * psi(y) = log2(e) phi(y ln 2), phi as above (Eq. 5).
 * d_out[i] = the tier's value at d_y[i] (both count float32, device):
 *   tier 0 psi        (two regimes, split at y = 1.8033688, selected per element)
 *   tier 1 psi_small  (C1 - lg2 y + y^2 q(y^2); the regime y <= 1.8033688)
 *   tier 2 psi_large  (t h(t^2), t = 2^-y;      the regime y >  1.8033688)
 *   tier 3 psi_deep_large  (h0 2^-y;  voted for warps with every y >= 10)
 *   tier 4 psi_deep_small  (C1 - lg2 y; voted for warps with every y <= 2^-10)
 *   tier 5 / 6  the row evaluator with warp votes, first / second psi of a
 *          check row (the tier is chosen by the votes over each warp's inputs).
 * LDPC_ERR_ARG for a tier outside 0..6. */
ldpc_status ldpc_debug_psi(const float *d_y, float *d_out, int64_t count, int32_t tier, void *stream);

/* Diagnostics: the throughput decoders' check-node update (Eq. 5,
 * P:128-132, readings Q2/Q3/Q7) on `rows` independent rows of `degree`
 * inputs: d_x[r*degree + j] = L'_vc (log2 units, L' = L log2 e; clamped to
 * +-30 log2 e inside, as in the decoders); d_e[r*degree + j] = the new
 * E'_cv = (-1)^degree prod_{j'!=j} sgn(x_j') min(psi(sum_{j'!=j}
 * psi(|x_j'|)), E_MAX log2 e).  vote != 0 runs the warp-voted tiers
 * (deep, saturation and clamp) exactly as the fixed-iteration kernels do;
 * vote == 0 the plain two-regime form (early termination, <= 20 iterations).
 * degree in {2, 3, 4, 6, 12} (else LDPC_ERR_UNSUPPORTED). */
ldpc_status ldpc_debug_check_row(const float *d_x, float *d_e, int64_t rows, int32_t degree, int32_t vote,
                                 void *stream);

/* Work partition, Eq. 9 (corrected per S:336, reading Q6):
 * counts[q] = floor(l/N) + (q < l mod N), displs = exclusive prefix sum.
 * Used to shard frames across GPUs (one rank per GPU). Host. */
ldpc_status ldpc_partition(int64_t l, int32_t nproc, int64_t *counts, int64_t *displs);

#ifdef __cplusplus
}
#endif
#endif /* LDPC_B200_H */
