/*
 * ldpc_oracle.c -- the CPU ORACLE for batched Sum-Product LDPC decoding.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the C-ABI library
 * paper_2201_04265_b200/libldpc_b200.so and its Python binding) may include,
 * link, import or execute this file.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it.  It shares no code,
 * header, table or constant generator with the CUDA path.
 *
 * Plain, slow, obviously-correct C: each function follows the paper
 * (/root/reference/PAPER.md, cited as P:<line>) step by step, in the order and
 * notation the paper uses; where the paper is silent or garbled the reading
 * taken is the one listed in DESIGN.md ("Readings", Q1..Q20 of SURVEY.md §8c).
 * Floating point is `long double` (x87 80-bit) for the decoder, fp64 for the
 * channel (reading Q20).
 *
 * Parity pins (tests/test_oracle_pins.py) tie every function here to something
 * other than itself: the paper's worked examples (Fig. 1, Fig. 2), brute-force
 * bitwise-MAP on cycle-free Tanner graphs, closed forms, published PRNG
 * known-answer vectors, and algebraic invariants.  Decoding on graphs WITH
 * cycles is pinned to the brute-force MAP of the depth-T computation tree
 * (T <= 3) and to the ring's closed form (any T); no function here is
 * "parity unpinned".  For the configs' large codes at T = 50 no independent
 * value exists: the pin there is this same routine's.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* SplitMix64 (Steele, Lea, Flood 2014).  Used for the Gallager band          */
/* permutations (reading Q12).                                              */
/* ------------------------------------------------------------------------ */
uint64_t oracle_splitmix64_next(uint64_t *state)
{
    uint64_t z;
    *state += 0x9E3779B97F4A7C15ULL;
    z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Uniform integer in [0, s): draw r, reject if r >= 2^64 - (2^64 mod s). */
uint64_t oracle_uniform_below(uint64_t *state, uint64_t s)
{
    uint64_t rem = (0 - s) % s;          /* = 2^64 mod s */
    for (;;) {
        uint64_t r = oracle_splitmix64_next(state);
        if (rem == 0 || r < (0 - rem))   /* 0 - rem = 2^64 - rem */
            return r % s;
    }
}

/* ------------------------------------------------------------------------ */
/* Regular (wc, wr) Gallager parity-check matrix.                            */
/* P:37 (section II: (n_c, n_v) regular H), P:598 (section IV: "we design the  */
/* Parity Check matrix ... as shown in [gallager_ldpc]").  Band construction */
/* per SPEC S:52: wc stacked bands of n/wr rows; band 0 row c has ones at     */
/* columns [c*wr, (c+1)*wr); band b >= 1 is a random column permutation of   */
/* band 0, drawn by Fisher-Yates from SplitMix64(seed).                      */
/*                                                                          */
/* Output: cols[(b*mb + c)*wr + j] = column of the j-th one of row b*mb+c.   */
/* Returns 0 ok, 1 if wr does not divide n, 2 on other bad arguments.        */
/* ------------------------------------------------------------------------ */
int oracle_make_H(int32_t n, int32_t wc, int32_t wr, uint64_t seed, int32_t *cols)
{
    if (n <= 0 || wc < 1 || wr < 2 || wc >= wr)
        return 2;
    if (n % wr != 0)
        return 1;
    int32_t mb = n / wr;
    int32_t *a = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    uint64_t state = seed;
    for (int32_t c = 0; c < mb; c++)
        for (int32_t j = 0; j < wr; j++)
            cols[(size_t)c * wr + j] = c * wr + j;
    for (int32_t b = 1; b < wc; b++) {
        for (int32_t i = 0; i < n; i++)
            a[i] = i;
        for (int32_t i = n - 1; i >= 1; i--) {
            int32_t j = (int32_t)oracle_uniform_below(&state, (uint64_t)i + 1);
            int32_t t = a[i]; a[i] = a[j]; a[j] = t;
        }
        for (int32_t c = 0; c < mb; c++)
            for (int32_t j = 0; j < wr; j++)
                cols[((size_t)b * mb + c) * wr + j] = a[c * wr + j];
    }
    free(a);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Generator in standard form.  P:47-53 (Eq. 2, H G^T = 0: G spans the null   */
/* space of H), P:329 (G converted to [I_k : P] by column permutations).      */
/* Gauss-Jordan elimination of H over GF(2), scanning columns RIGHT TO LEFT  */
/* (reading Q13): for j = n-1..0 the pivot is the lowest-index row >= r with */
/* bit j set; swap it to row r, XOR it into every other row having bit j,   */
/* r++.  rank = r.  F = free columns ascending, Piv = pivot columns           */
/* ascending, perm = [F, Piv], P[a][b] = RREF[row(Piv_b)][F_a], k = n - rank. */
/* Rows are stored one bit per uint64 lane (a representation, not blocking). */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t n, k, rank;
    int32_t *perm;      /* n */
    uint8_t *P;         /* k x (n-k), row-major, one byte per bit */
} oracle_G;

oracle_G *oracle_make_G(int32_t m, int32_t n, const int32_t *row_ptr, const int32_t *col_idx)
{
    size_t W = ((size_t)n + 63) / 64;
    uint64_t *rows = (uint64_t *)calloc((size_t)m * W, sizeof(uint64_t));
    for (int32_t i = 0; i < m; i++)
        for (int32_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
            int32_t j = col_idx[e];
            rows[(size_t)i * W + j / 64] ^= (uint64_t)1 << (j % 64); /* GF(2): repeated entry cancels */
        }
    int32_t *pivot_row_of_col = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int32_t j = 0; j < n; j++)
        pivot_row_of_col[j] = -1;
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * W);
    int32_t r = 0;
    for (int32_t j = n - 1; j >= 0 && r < m; j--) {
        size_t w = (size_t)j / 64;
        uint64_t bit = (uint64_t)1 << (j % 64);
        int32_t p = -1;
        for (int32_t i = r; i < m; i++)
            if (rows[(size_t)i * W + w] & bit) { p = i; break; }
        if (p < 0)
            continue;
        if (p != r) {
            memcpy(tmp, rows + (size_t)p * W, W * 8);
            memcpy(rows + (size_t)p * W, rows + (size_t)r * W, W * 8);
            memcpy(rows + (size_t)r * W, tmp, W * 8);
        }
        for (int32_t i = 0; i < m; i++) {
            if (i != r && (rows[(size_t)i * W + w] & bit)) {
                for (size_t q = 0; q < W; q++)
                    rows[(size_t)i * W + q] ^= rows[(size_t)r * W + q];
            }
        }
        pivot_row_of_col[j] = r;
        r++;
    }
    oracle_G *g = (oracle_G *)calloc(1, sizeof(oracle_G));
    g->n = n;
    g->rank = r;
    g->k = n - r;
    g->perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t nf = 0, np = 0;
    for (int32_t j = 0; j < n; j++)
        if (pivot_row_of_col[j] < 0) g->perm[nf++] = j;
    for (int32_t j = 0; j < n; j++)
        if (pivot_row_of_col[j] >= 0) { g->perm[g->k + np] = j; np++; }
    g->P = (uint8_t *)calloc((size_t)g->k * (size_t)(n - g->k) + 1, 1);
    for (int32_t a = 0; a < g->k; a++) {
        int32_t fa = g->perm[a];
        for (int32_t b = 0; b < n - g->k; b++) {
            int32_t row = pivot_row_of_col[g->perm[g->k + b]];
            g->P[(size_t)a * (n - g->k) + b] =
                (uint8_t)((rows[(size_t)row * W + fa / 64] >> (fa % 64)) & 1);
        }
    }
    free(tmp);
    free(pivot_row_of_col);
    free(rows);
    return g;
}
int32_t oracle_G_k(const oracle_G *g) { return g->k; }
int32_t oracle_G_rank(const oracle_G *g) { return g->rank; }
void oracle_G_perm(const oracle_G *g, int32_t *out) { memcpy(out, g->perm, sizeof(int32_t) * (size_t)g->n); }
void oracle_G_P(const oracle_G *g, uint8_t *out) { memcpy(out, g->P, (size_t)g->k * (size_t)(g->n - g->k)); }
void oracle_G_free(oracle_G *g)
{
    if (!g) return;
    free(g->perm); free(g->P); free(g);
}

/* ------------------------------------------------------------------------ */
/* Encoding, Eq. 3 in the standard form of P:329: the k info bits  */
/* are copied, then each parity bit b is sum_a m_a P[a][b] over GF(2).  The  */
/* permuted codeword is scattered back to H column order: c[perm[t]] = cp[t]. */
/* m: frames x k bytes (0/1); c: frames x n bytes (0/1).                    */
/* ------------------------------------------------------------------------ */
void oracle_encode(int32_t k, int32_t n, const int32_t *perm, const uint8_t *P,
                   const uint8_t *m, int64_t frames, uint8_t *c)
{
    for (int64_t f = 0; f < frames; f++) {
        const uint8_t *mf = m + f * k;
        uint8_t *cf = c + f * n;
        for (int32_t t = 0; t < k; t++)
            cf[perm[t]] = mf[t] & 1;
        for (int32_t b = 0; b < n - k; b++) {
            uint8_t s = 0;
            for (int32_t a = 0; a < k; a++)
                s ^= (uint8_t)(mf[a] & P[(size_t)a * (n - k) + b]);
            cf[perm[k + b]] = s;
        }
    }
}

/* Syndrome H z^T over GF(2), Eq. 1.  Returns 1 iff all zero. */
int oracle_syndrome_zero(int32_t m, const int32_t *row_ptr, const int32_t *col_idx, const uint8_t *z)
{
    for (int32_t c = 0; c < m; c++) {
        uint8_t s = 0;
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; e++)
            s ^= z[col_idx[e]] & 1;
        if (s)
            return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).                        */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Info bits (reading c4): word w of frame f is lane w%4 of                  */
/* Philox(key=(seed_lo, seed_hi), ctr=(w/4, f_lo, f_hi, 0)); bit t of the    */
/* frame is bit t%32 (LSB first) of word t/32.  Output one byte per bit.     */
void oracle_gen_info(uint64_t seed, int64_t frame0, int64_t frames, int32_t k, uint8_t *bits)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t i = 0; i < frames; i++) {
        uint64_t f = (uint64_t)(frame0 + i);
        for (int32_t t = 0; t < k; t++) {
            int32_t w = t / 32;
            uint32_t ctr[4] = {(uint32_t)(w / 4), (uint32_t)f, (uint32_t)(f >> 32), 0u};
            uint32_t out[4];
            oracle_philox4x32_10(ctr, key, out);
            bits[i * k + t] = (uint8_t)((out[w % 4] >> (t % 32)) & 1u);
        }
    }
}

/* BPSK over AWGN, P:329 ("we convert the 0 bits to -1 and 1 bits remain as */
/* 1") and P:125 (AWGN of power sigma^2).  Noise (reading c4): counter      */
/* (j, f_lo, f_hi, 1) gives x0..x3; Box-Muller with u1 = (x0+1) 2^-32,       */
/* u2 = x1 2^-32 gives z_{4j}, z_{4j+1}; x2, x3 likewise give z_{4j+2},      */
/* z_{4j+3}.  y = (2c - 1) + sigma z, in fp64.                               */
void oracle_channel_y(uint64_t seed, int64_t frame0, int64_t frames, int32_t n,
                      const uint8_t *c, double sigma, double *y)
{
    const double two_pi = 6.283185307179586476925286766559;
    const double inv32 = 1.0 / 4294967296.0;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t i = 0; i < frames; i++) {
        uint64_t f = (uint64_t)(frame0 + i);
        for (int32_t v = 0; v < n; v++) {
            int32_t j = v / 4, lane = v % 4;
            uint32_t ctr[4] = {(uint32_t)j, (uint32_t)f, (uint32_t)(f >> 32), 1u};
            uint32_t x[4];
            oracle_philox4x32_10(ctr, key, x);
            uint32_t xa = (lane < 2) ? x[0] : x[2];
            uint32_t xb = (lane < 2) ? x[1] : x[3];
            double u1 = ((double)xa + 1.0) * inv32;
            double u2 = (double)xb * inv32;
            double rad = sqrt(-2.0 * log(u1));
            double z = (lane % 2 == 0) ? rad * cos(two_pi * u2) : rad * sin(two_pi * u2);
            double x_bpsk = c[i * n + v] ? 1.0 : -1.0;
            y[i * n + v] = x_bpsk + sigma * z;
        }
    }
}

/* Channel LLR, Eq. 4 read as R = ln(p1/p0) = 2 y / sigma^2      */
/* (reading Q1), clamped to +-30 (reading Q7), rounded once to fp32.         */
void oracle_llr(const double *y, int64_t count, double sigma, float *R)
{
    for (int64_t i = 0; i < count; i++) {
        double llr = 2.0 * y[i] / (sigma * sigma);
        if (llr > 30.0) llr = 30.0;
        if (llr < -30.0) llr = -30.0;
        R[i] = (float)llr;
    }
}

/* The two composed: codeword bits -> fp32 channel LLRs. */
void oracle_channel(uint64_t seed, int64_t frame0, int64_t frames, int32_t n,
                    const uint8_t *c, double sigma, float *R)
{
    double *y = (double *)malloc(sizeof(double) * (size_t)(frames * n + 1));
    oracle_channel_y(seed, frame0, frames, n, c, sigma, y);
    oracle_llr(y, frames * n, sigma, R);
    free(y);
}

/* ------------------------------------------------------------------------ */
/* Sum-Product decoding, P:118-155 (Eqs. 4-8) with the flooding schedule of  */
/* Alg. 1 (all checks, then all variables).                       */
/*   Eq. 5 (garbled; reading Q2/Q3):                               */
/*      E_cv = (-1)^{d_c} 2 atanh( prod_{v' != v} tanh(L_{v'c}/2) )           */
/*   Eq. 6:  L_vc = R_v + sum_{c' != c} E_{c'v}                  */
/*   Eq. 7:  L_v  = R_v + sum_c E_cv                              */
/*   Eq. 8:  z_v  = [L_v >= 0]                                    */
/* Clamps (reading Q7): R and every L_vc to +-30, the atanh argument to       */
/* +-(1 - 1e-12).  The exclusive products are prefix/suffix products (SPEC   */
/* S:240).  Early termination (reading Q11 / c6): after iteration t >= 1,    */
/* stop if H z^t = 0.                                                         */
/* One frame; E, Lvc, th, pre, suf are scratch of size nnz / max degree.     */
/* ------------------------------------------------------------------------ */
typedef long double ld;

static ld clampl(ld x, ld lim)
{
    if (x > lim) return lim;
    if (x < -lim) return -lim;
    return x;
}

void oracle_spa_decode(int32_t m, int32_t n, const int32_t *row_ptr, const int32_t *col_idx,
                       const float *R_in, int32_t max_iter, int32_t early_term,
                       double *L_out, uint8_t *z_out, int32_t *iters_out, uint8_t *syn_ok_out)
{
    int32_t nnz = row_ptr[m];
    int32_t maxd = 0;
    for (int32_t c = 0; c < m; c++)
        if (row_ptr[c + 1] - row_ptr[c] > maxd) maxd = row_ptr[c + 1] - row_ptr[c];
    /* variable -> list of edge ids in ascending check order (the Tanner graph) */
    int32_t *vdeg = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    for (int32_t e = 0; e < nnz; e++) vdeg[col_idx[e] + 1]++;
    for (int32_t v = 0; v < n; v++) vdeg[v + 1] += vdeg[v];
    int32_t *vptr = vdeg;
    int32_t *vedges = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nnz + 1));
    int32_t *fill = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    for (int32_t c = 0; c < m; c++)
        for (int32_t e = row_ptr[c]; e < row_ptr[c + 1]; e++) {
            int32_t v = col_idx[e];
            vedges[vptr[v] + fill[v]++] = e;
        }
    ld *R = (ld *)malloc(sizeof(ld) * (size_t)n);
    ld *L = (ld *)malloc(sizeof(ld) * (size_t)n);
    ld *E = (ld *)calloc((size_t)nnz + 1, sizeof(ld));
    ld *Enew = (ld *)calloc((size_t)nnz + 1, sizeof(ld));
    ld *th = (ld *)malloc(sizeof(ld) * ((size_t)maxd + 1));
    ld *pre = (ld *)malloc(sizeof(ld) * ((size_t)maxd + 2));
    ld *suf = (ld *)malloc(sizeof(ld) * ((size_t)maxd + 2));
    uint8_t *z = (uint8_t *)malloc((size_t)n + 1);
    const ld pmax = 1.0L - 1e-12L;

    for (int32_t v = 0; v < n; v++) {
        R[v] = clampl((ld)R_in[v], 30.0L);
        L[v] = R[v];                       /* L_v = R_v sent to all checks */
        z[v] = (L[v] >= 0.0L) ? 1 : 0;
    }
    int32_t iters = max_iter;
    int32_t stopped = 0;
    for (int32_t t = 1; t <= max_iter; t++) {
        /* check-node update, Eq. 5, using L_vc of Eq. 6 from the previous E */
        for (int32_t c = 0; c < m; c++) {
            int32_t d = row_ptr[c + 1] - row_ptr[c];
            for (int32_t j = 0; j < d; j++) {
                int32_t e = row_ptr[c] + j;
                int32_t v = col_idx[e];
                ld s = R[v];
                for (int32_t q = vptr[v]; q < vptr[v + 1]; q++)
                    if (vedges[q] != e) s += E[vedges[q]];
                ld Lvc = clampl(s, 30.0L);
                th[j] = tanhl(Lvc / 2.0L);
            }
            pre[0] = 1.0L;
            for (int32_t j = 0; j < d; j++) pre[j + 1] = pre[j] * th[j];
            suf[d] = 1.0L;
            for (int32_t j = d - 1; j >= 0; j--) suf[j] = suf[j + 1] * th[j];
            ld sign_d = (d % 2 == 0) ? 1.0L : -1.0L;
            for (int32_t j = 0; j < d; j++) {
                ld p = clampl(pre[j] * suf[j + 1], pmax);
                Enew[row_ptr[c] + j] = sign_d * 2.0L * atanhl(p);
            }
        }
        ld *sw = E; E = Enew; Enew = sw;
        /* total LLR, Eq. 7, and hard decision, Eq. 8 */
        for (int32_t v = 0; v < n; v++) {
            ld s = R[v];
            for (int32_t q = vptr[v]; q < vptr[v + 1]; q++) s += E[vedges[q]];
            L[v] = s;
            z[v] = (s >= 0.0L) ? 1 : 0;
        }
        if (early_term && oracle_syndrome_zero(m, row_ptr, col_idx, z)) {
            iters = t;
            stopped = 1;
            break;
        }
    }
    for (int32_t v = 0; v < n; v++) {
        if (L_out) L_out[v] = (double)L[v];
        if (z_out) z_out[v] = z[v];
    }
    if (iters_out) *iters_out = iters;
    if (syn_ok_out) *syn_ok_out = stopped ? 1 : (uint8_t)oracle_syndrome_zero(m, row_ptr, col_idx, z);
    free(vdeg); free(vedges); free(fill); free(R); free(L); free(E); free(Enew);
    free(th); free(pre); free(suf); free(z);
}

/* Batch decode: "Sum-Product decoding ... on the batch of n      */
/* length vectors in a serial manner".                                        */
void oracle_spa_decode_batch(int32_t m, int32_t n, const int32_t *row_ptr, const int32_t *col_idx,
                             const float *R, int64_t frames, int32_t max_iter, int32_t early_term,
                             double *L_out, uint8_t *z_out, int32_t *iters_out, uint8_t *syn_ok_out)
{
    for (int64_t f = 0; f < frames; f++)
        oracle_spa_decode(m, n, row_ptr, col_idx, R + f * n, max_iter, early_term,
                          L_out ? L_out + f * n : 0, z_out ? z_out + f * n : 0,
                          iters_out ? iters_out + f : 0, syn_ok_out ? syn_ok_out + f : 0);
}

/* ------------------------------------------------------------------------ */
/* Work partition, Eq. 9 (garbled; reading Q6 = SPEC S:336):      */
/* counts[q] = floor(l/N) + [q < l mod N], displs = exclusive prefix sum.    */
/* ------------------------------------------------------------------------ */
void oracle_partition(int64_t l, int32_t N, int64_t *counts, int64_t *displs)
{
    int64_t acc = 0;
    for (int32_t q = 0; q < N; q++) {
        counts[q] = l / N + ((q < l % N) ? 1 : 0);
        displs[q] = acc;
        acc += counts[q];
    }
}

/* ------------------------------------------------------------------------ */
/* Error counters (SPEC run_ber S:522-530; reading Q14):                     */
/* out[0] info-bit errors at positions perm[0..k), out[1] codeword-bit errors,*/
/* out[2] frame errors (any info-bit error), out[3] undetected errors        */
/* (syndrome zero but some codeword bit wrong), out[4] sum of iterations,    */
/* out[5] frames.  z, c: frames x n bytes; info: frames x k bytes.           */
/* ------------------------------------------------------------------------ */
void oracle_count_errors(int32_t k, int32_t n, const int32_t *perm, const uint8_t *info,
                         const uint8_t *z, const uint8_t *c, const uint8_t *syn_ok,
                         const int32_t *iters, int64_t frames, int64_t out[6])
{
    for (int q = 0; q < 6; q++) out[q] = 0;
    for (int64_t f = 0; f < frames; f++) {
        int64_t ie = 0, ce = 0;
        for (int32_t t = 0; t < k; t++)
            ie += (z[f * n + perm[t]] ^ info[f * k + t]) & 1;
        for (int32_t v = 0; v < n; v++)
            ce += (z[f * n + v] ^ c[f * n + v]) & 1;
        out[0] += ie;
        out[1] += ce;
        out[2] += ie > 0;
        out[3] += (syn_ok[f] && ce > 0);
        out[4] += iters[f];
        out[5] += 1;
    }
}
