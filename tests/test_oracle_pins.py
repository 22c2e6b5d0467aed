"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test names the passage (P:<line> of PAPER.md, S:<line> of SPEC.md) or the
closed form it relies on.  None re-types the oracle's own formula: the expected
values come from the paper's worked examples, published known-answer vectors,
brute-force enumeration, or algebraic invariants.
"""
import math

import numpy as np
import pytest

from tests import helpers as hp


# ----------------------------------------------------------------- PRNG KATs
def test_philox_known_answers(oracle):
    rows = [r for r in hp.golden_lines("prng_kat.txt") if r[0] == "philox"]
    assert len(rows) == 3
    for r in rows:
        ctr = [int(x, 16) for x in r[1:5]]
        key = [int(x, 16) for x in r[5:7]]
        want = [int(x, 16) for x in r[7:11]]
        assert oracle.philox4x32_10(ctr, key) == want


def test_splitmix64_known_answers(oracle):
    r = [r for r in hp.golden_lines("prng_kat.txt") if r[0] == "splitmix64"][0]
    seed = int(r[1])
    want = [int(x) for x in r[2:]]
    assert oracle.splitmix64_stream(seed, len(want)) == want


def test_uniform_below_matches_modulo_when_no_rejection(oracle):
    # s = 2^j: 2^64 mod s = 0, so no draw is rejected and U(s) = r mod s.
    raw = oracle.splitmix64_stream(77, 200)
    for j in (1, 5, 32, 63):
        assert oracle.uniform_below_stream(77, 1 << j, 200) == [x % (1 << j) for x in raw]
    # s = 3: only r = 2^64 - 1 is rejected, so U(3) = r mod 3 on these draws.
    assert oracle.uniform_below_stream(77, 3, 200) == [x % 3 for x in raw]


def test_uniform_below_rejects_above_threshold(oracle):
    # s = 2^63 + 1: 2^64 mod s = 2^63 - 1, so the threshold 2^64 - (2^64 mod s)
    # is s itself: every draw >= s is skipped (about half of them).
    s = (1 << 63) + 1
    raw = oracle.splitmix64_stream(5, 400)
    kept = [x % s for x in raw if x < s]
    got = oracle.uniform_below_stream(5, s, len(kept) - 5)
    assert got == kept[: len(got)]
    assert len(kept) < len(raw)  # some were rejected


# ----------------------------------------------------------------- make_H
@pytest.mark.parametrize("n,wc,wr", [(96, 3, 6), (1008, 3, 6), (3996, 3, 4), (3996, 3, 12),
                                     (1032, 9, 12), (8, 2, 4)])
def test_make_H_weights_and_bands(oracle, n, wc, wr):
    """(n_c, n_v) regular H; exact row weight wr, column
    weight wc, band 0 contiguous, each band a permutation of the columns."""
    code = oracle.make_H(n, wc, wr, seed=1)
    H = code.dense()
    mb = n // wr
    assert H.shape == (n * wc // wr, n)
    assert np.all(H.sum(axis=1) == wr)
    assert np.all(H.sum(axis=0) == wc)
    for c in range(mb):
        assert list(np.nonzero(H[c])[0]) == list(range(c * wr, (c + 1) * wr))
    for b in range(wc):
        band = H[b * mb:(b + 1) * mb]
        assert np.all(band.sum(axis=0) == 1)


def test_make_H_deterministic_and_seed_sensitive(oracle):
    a = oracle.make_H(1008, 3, 6, 1).dense()
    b = oracle.make_H(1008, 3, 6, 1).dense()
    c = oracle.make_H(1008, 3, 6, 2).dense()
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


def test_make_H_rejects_bad_args(oracle):
    with pytest.raises(ValueError, match="divide"):
        oracle.make_H(4000, 3, 6, 1)           # reading Q16: 4000 % 6 != 0
    with pytest.raises(ValueError):
        oracle.make_H(12, 6, 6, 1)             # wc >= wr


def test_fisher_yates_is_uniform(oracle):
    """Band-1 permutation of n = 3 (wr = 3 -> band 1 is one row; use the row
    order of a (2,3) code with n = 3... instead use the permutation itself via
    n = 3, wr = 3: band 1 row 0 lists pi_1[0..3))."""
    counts = {}
    trials = 6000
    for s in range(trials):
        code = oracle.make_H(3, 2, 3, s)
        key = tuple(code.col_idx[3:6])
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 6
    exp = trials / 6
    chi2 = sum((v - exp) ** 2 / exp for v in counts.values())
    assert chi2 < 20.5  # chi^2_5, p = 0.001


# ----------------------------------------------------------------- make_G
def test_fig1_rank_and_graph(oracle):
    """Fig. 1: rank 3, k = 5; its Tanner graph edges
    equal the drawn ones."""
    H = hp.golden_matrix("fig1_H.txt")
    code = oracle.Code.from_dense(H).make_G()
    assert code.rank == 3 == hp.gf2_rank(H)
    assert code.k == 5
    G = code.G_dense()
    assert not np.any((H.astype(int) @ G.T.astype(int)) % 2)
    drawn = {(int(v) - 1, int(c) - 1) for v, c in hp.golden_lines("fig1_edges.txt")}
    graph = {(int(code.col_idx[e]), c) for c in range(code.m)
             for e in range(code.row_ptr[c], code.row_ptr[c + 1])}
    assert drawn == graph


def test_fig2_generator_reproduced_from_its_parity_check(oracle):
    """Fig. 2 prints G = [I_4 : P].  From H = [P^T : I_4] the
    right-to-left elimination (reading Q13) must return exactly that G with the
    identity permutation, and the H is a tree (cycle-free Tanner graph)."""
    G = hp.golden_matrix("fig2_G.txt")
    P = G[:, 4:]
    H = np.concatenate([P.T, np.eye(4, dtype=np.uint8)], axis=1)
    assert hp.is_tree(H)
    code = oracle.Code.from_dense(H).make_G()
    assert code.k == 4
    assert list(code.perm) == list(range(8))
    assert np.array_equal(code.P, P)
    assert np.array_equal(code.G_dense(), G)


def test_hamming74(oracle):
    """Textbook Hamming(7,4) (reading Q18: not in the paper): k = 4, 16
    codewords, minimum distance 3, every codeword has zero syndrome."""
    H = hp.hamming74_H()
    code = oracle.Code.from_dense(H).make_G()
    assert code.k == 4 and code.rank == 3
    msgs = ((np.arange(16)[:, None] >> np.arange(4)[None, :]) & 1).astype(np.uint8)
    cws = oracle.encode(code, msgs)
    assert len({tuple(c) for c in cws}) == 16
    assert {tuple(c) for c in cws} == {tuple(c) for c in hp.codewords(H)}
    w = cws.sum(axis=1)
    assert w[w > 0].min() == 3


@pytest.mark.parametrize("n,wc,wr", [(96, 3, 6), (1008, 3, 6), (1032, 9, 12), (1032, 6, 12),
                                     (1032, 3, 12), (3996, 3, 12)])
def test_make_G_null_space(oracle, n, wc, wr):
    """Eq. 2: H G^T = 0; rows(G) = n - rank(H); the standard
    form has I_k on perm[0..k); rank agrees with an independent
    left-to-right elimination; rank <= m - (wc - 1) since every band sums to
    the all-ones row."""
    code = oracle.make_H(n, wc, wr, 1).make_G()
    H = code.dense()
    rank = hp.gf2_rank(H)
    assert code.rank == rank
    assert code.k == n - rank
    assert rank <= code.m - (wc - 1)
    G = code.G_dense()
    assert G.shape == (code.k, n)
    assert not np.any((H.astype(np.int64) @ G.T.astype(np.int64)) % 2)
    assert np.array_equal(G[:, code.perm[:code.k]], np.eye(code.k, dtype=np.uint8))
    assert hp.gf2_rank(G) == code.k
    assert sorted(code.perm) == list(range(n))


# ----------------------------------------------------------------- encode
def test_fig2_encode_example(oracle):
    """Fig. 2: m = [1,0,1,1] -> p = [1,0,1,1,1,0,0,1]."""
    G = hp.golden_matrix("fig2_G.txt")
    rows = {r[0]: [int(x) for x in r[1:]] for r in hp.golden_lines("fig2_encode.txt")}
    code = oracle.Code.from_dense(np.concatenate([G[:, 4:].T, np.eye(4, dtype=np.uint8)], 1)).make_G()
    p = oracle.encode(code, np.array([rows["m"]], dtype=np.uint8))
    assert list(p[0]) == rows["p"]


@pytest.mark.parametrize("n,wc,wr", [(96, 3, 6), (1008, 3, 6), (3996, 3, 4)])
def test_encode_codewords_linear(oracle, n, wc, wr):
    """Eq. 1: every encoded word has zero syndrome; encoding is
    linear over GF(2); m = 0 -> 0; systematic bits sit at perm[0..k)."""
    code = oracle.make_H(n, wc, wr, 1).make_G()
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2, (20, code.k), dtype=np.uint8)
    b = rng.integers(0, 2, (20, code.k), dtype=np.uint8)
    ca, cb, cab = oracle.encode(code, a), oracle.encode(code, b), oracle.encode(code, a ^ b)
    H = code.dense().astype(np.int64)
    assert not np.any((ca.astype(np.int64) @ H.T) % 2)
    assert np.array_equal(ca ^ cb, cab)
    assert not oracle.encode(code, np.zeros((1, code.k), np.uint8)).any()
    assert np.array_equal(ca[:, code.perm[:code.k]], a)
    for f in range(3):
        assert oracle.syndrome_zero(code, ca[f])


def test_syndrome_zero_pinned(oracle):
    """Eq. 1: syndrome_zero(z) is 1 exactly when H z^T = 0 over
    GF(2).  Against numpy's integer product and brute-force enumeration: every
    weight-1 word is rejected (no H here has an all-zero column), every
    codeword of Fig. 1 and Hamming(7,4) is accepted, and random
    words of a Gallager code agree with (H z) mod 2 -- so an always-true (or
    always-false) syndrome fails."""
    mats = [hp.golden_matrix("fig1_H.txt"), hp.hamming74_H()]
    for H in mats:
        code = oracle.Code.from_dense(H)
        n = H.shape[1]
        for v in range(n):
            e = np.zeros(n, np.uint8)
            e[v] = 1
            assert not oracle.syndrome_zero(code, e)
        cws = hp.codewords(H)
        assert len(cws) > 1
        for c in cws:
            assert oracle.syndrome_zero(code, c)
        words = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1).astype(np.uint8)
        want = np.all((words.astype(np.int64) @ H.T.astype(np.int64)) % 2 == 0, axis=1)
        got = np.array([oracle.syndrome_zero(code, w) for w in words])
        assert np.array_equal(got, want)
        assert 0 < want.sum() < len(words)
    code = oracle.make_H(96, 3, 6, 1)
    H = code.dense().astype(np.int64)
    rng = np.random.default_rng(5)
    z = rng.integers(0, 2, (200, 96), dtype=np.uint8)
    for f in range(200):
        assert oracle.syndrome_zero(code, z[f]) == (not np.any((H @ z[f].astype(np.int64)) % 2))
    assert not any(oracle.syndrome_zero(code, z[f]) for f in range(200))     # random words fail


# ----------------------------------------------------------------- channel
def test_llr_spec_examples(oracle):
    """Eq. 4: R = 2y/sigma^2; SPEC S:289-291 examples."""
    for r in hp.golden_lines("spec_examples.txt"):
        if r[0] == "llr":
            y, s, want = float(r[1]), float(r[2]), float(r[3])
            assert oracle.llr(np.array([y]), s)[0] == pytest.approx(want, abs=0)


def test_llr_clamp_odd_monotone(oracle):
    y = np.linspace(-40, 40, 2001)
    R = oracle.llr(y, 1.0)
    assert R.max() == 30.0 and R.min() == -30.0
    assert np.array_equal(oracle.llr(-y, 1.0), -R)
    assert np.all(np.diff(R) >= 0)


def test_channel_statistics(oracle):
    """BPSK 0 -> -1, 1 -> +1 plus N(0, sigma^2): the noise
    y - x is Gaussian (KS test), mean/variance within sampling bounds,
    and the uncoded hard-decision BER is Q(1/sigma) within 4 s.e.."""
    from scipy import stats
    sigma = 0.8
    rng = np.random.default_rng(1)
    F, n = 50, 2000
    c = rng.integers(0, 2, (F, n), dtype=np.uint8)
    y = oracle.channel_y(501, 0, c, sigma)
    noise = (y - (2.0 * c - 1.0)).ravel() / sigma
    N = noise.size
    assert abs(noise.mean()) < 4 / math.sqrt(N)
    assert abs(noise.var() - 1.0) < 0.02
    assert stats.kstest(noise, "norm").pvalue > 1e-3
    R = oracle.channel(501, 0, c, sigma)
    assert np.array_equal(R, oracle.llr(y, sigma))
    ber = np.mean((R >= 0).astype(np.uint8) != c)
    p = hp.q_function(1.0 / sigma)
    assert abs(ber - p) < 4 * math.sqrt(p * (1 - p) / N)


def test_channel_noiseless_identity_and_frame_independence(oracle):
    rng = np.random.default_rng(2)
    c = rng.integers(0, 2, (4, 96), dtype=np.uint8)
    R = oracle.channel(9, 0, c, 1e-9)
    assert np.array_equal((R >= 0).astype(np.uint8), c)
    assert np.all(np.abs(R) == 30.0)
    # frame f depends only on (seed, f): a shifted window reproduces it
    R_all = oracle.channel(9, 10, c, 0.7)
    R_one = oracle.channel(9, 12, c[2:3], 0.7)
    assert np.array_equal(R_all[2:3], R_one)


def test_gen_info_bit_layout(oracle):
    """Info word w of frame f is Philox lane w%4 at counter (w/4, f, 0, 0)."""
    k = 70
    bits = oracle.gen_info(123, 5, 2, k)
    key = [123, 0]
    for i, f in enumerate((5, 6)):
        for w in range(3):
            word = oracle.philox4x32_10([w // 4, f, 0, 0], key)[w % 4]
            for b in range(32):
                t = 32 * w + b
                if t < k:
                    assert bits[i, t] == (word >> b) & 1


# ----------------------------------------------------------------- SPA decode
def _tree_R(rng, H, sigma):
    cw = hp.codewords(H)
    x = cw[rng.integers(0, len(cw))]
    y = (2.0 * x - 1.0) + sigma * rng.standard_normal(H.shape[1])
    return (2.0 * y / sigma ** 2).astype(np.float32)


def test_spa_equals_map_on_fig2_tree(oracle):
    """Cycle-free Tanner graph (Fig. 2's H = [P^T : I_4], odd-degree checks):
    SPA posteriors equal brute-force bitwise-MAP marginals."""
    G = hp.golden_matrix("fig2_G.txt")
    H = np.concatenate([G[:, 4:].T, np.eye(4, dtype=np.uint8)], axis=1)
    code = oracle.Code.from_dense(H)
    rng = np.random.default_rng(3)
    for _ in range(50):
        R = _tree_R(rng, H, 1.2)
        L, z, it, so = oracle.spa_decode(code, R, max_iter=20)
        want = hp.map_llr(H, R)
        assert np.max(np.abs(L[0] - want)) < 1e-9


def test_spa_equals_map_on_random_trees(oracle):
    rng = np.random.default_rng(4)
    done = 0
    odd = 0
    while done < 60:
        H = hp.random_tree_H(rng, n_max=int(rng.integers(4, 17)))
        if H.shape[0] == 0:
            continue
        assert hp.is_tree(H)
        R = _tree_R(rng, H, 1.5)
        want = hp.map_llr(H, R)
        if np.max(np.abs(want)) > 25:        # keep clear of the +-30 clamps (reading Q7)
            continue
        code = oracle.Code.from_dense(H)
        L, *_ = oracle.spa_decode(code, R, max_iter=2 * H.shape[1] + 2)
        assert np.max(np.abs(L[0] - want)) < 1e-9
        odd += int(np.any(H.sum(axis=1) % 2 == 1))
        done += 1
    assert odd > 10   # odd check degrees exercised the (-1)^{d_c} rule (reading Q3)


def test_spa_single_parity_check_closed_form(oracle):
    """SPC of length 7 after one iteration:
    L_v = R_v + (-1)^7 * 2 atanh(prod_{u != v} tanh(R_u / 2)), which is also
    the exact MAP (a one-check tree)."""
    rng = np.random.default_rng(5)
    H = np.ones((1, 7), dtype=np.uint8)
    code = oracle.Code.from_dense(H)
    for _ in range(20):
        R = rng.normal(0, 2, 7).astype(np.float32)
        L, *_ = oracle.spa_decode(code, R, max_iter=1)
        Rd = R.astype(np.float64)
        for v in range(7):
            prod = np.prod(np.tanh(np.delete(Rd, v) / 2))
            assert L[0, v] == pytest.approx(Rd[v] - 2 * math.atanh(prod), abs=1e-12)
        assert np.max(np.abs(L[0] - hp.map_llr(H, R))) < 1e-9


def test_spa_repetition_chain_closed_form(oracle):
    """Checks x_i + x_{i+1} = 0 on a path: the code is {0^n, 1^n}, whose MAP
    posterior is sum_u R_u for every bit; SPA reaches it after n - 1 iterations."""
    n = 9
    H = np.zeros((n - 1, n), dtype=np.uint8)
    for i in range(n - 1):
        H[i, i] = H[i, i + 1] = 1
    code = oracle.Code.from_dense(H)
    rng = np.random.default_rng(6)
    for _ in range(10):
        R = rng.normal(0.5, 1.0, n).astype(np.float32)
        L, *_ = oracle.spa_decode(code, R, max_iter=n)
        assert np.max(np.abs(L[0] - float(np.sum(R.astype(np.float64))))) < 1e-9


def test_spa_spec_scalar_examples(oracle):
    """S:180-182 degree-3 check (corrected value, reading Q19), degree-2
    pass-through, zero-message annihilation (reading Q9),
    degree-1 check forcing bit 0 with E_MAX (reading Q9)."""
    row = [r for r in hp.golden_lines("spec_examples.txt") if r[0] == "check3"][0]
    a, b, want = float(row[1]), float(row[2]), float(row[3])
    code = oracle.Code.from_dense(np.ones((1, 3), np.uint8))
    L, *_ = oracle.spa_decode(code, np.array([0.0, a, b], np.float32), max_iter=1)
    assert L[0, 0] == pytest.approx(want, abs=1e-10)
    # degree 2: the check passes the other variable's LLR through
    code2 = oracle.Code.from_dense(np.ones((1, 2), np.uint8))
    L, *_ = oracle.spa_decode(code2, np.array([0.75, -2.5], np.float32), max_iter=1)
    assert L[0, 0] == pytest.approx(0.75 - 2.5, abs=1e-12)
    # a zero incoming message makes every other extrinsic exactly zero
    L, *_ = oracle.spa_decode(code, np.array([1.5, 0.0, 3.0], np.float32), max_iter=1)
    assert L[0, 0] == 1.5 and L[0, 2] == 3.0
    # degree-1 check: E = -2 atanh(1 - 1e-12) = -ln((2 - 1e-12) / 1e-12)
    # = -ln(2e12 - 1) = -28.32416830... (closed form; 2e12 - 1 is exact in fp64)
    code1 = oracle.Code.from_dense(np.ones((1, 1), np.uint8))
    L, z, *_ = oracle.spa_decode(code1, np.array([5.0], np.float32), max_iter=1)
    # (1 - 1e-12 rounds to long double with 1 - p off by 4e-21 = 4e-9 relative,
    # hence the 1e-8 tolerance)
    assert L[0, 0] == pytest.approx(5.0 - math.log(2e12 - 1), abs=1e-8)
    assert z[0, 0] == 0
    # tie: L = 0 decides bit 1 (Eq. 8)
    L, z, *_ = oracle.spa_decode(code, np.array([0.0, 0.0, 0.0], np.float32), max_iter=1)
    assert np.all(L[0] == 0.0) and np.all(z[0] == 1)


def test_spa_sign_equivariance_even_degree(oracle):
    """Negating every channel LLR of an even-degree code negates every message
    and posterior exactly."""
    code = oracle.make_H(96, 3, 6, 1)
    rng = np.random.default_rng(7)
    R = rng.normal(0.3, 2.0, (3, 96)).astype(np.float32)
    L1, *_ = oracle.spa_decode(code, R, 10)
    L2, *_ = oracle.spa_decode(code, -R, 10)
    assert np.array_equal(L1, -L2)


def test_spa_noiseless_codeword_fixed_point(oracle):
    """clamp-strength LLRs of a codeword decode to that codeword."""
    code = oracle.make_H(1008, 3, 6, 1).make_G()
    rng = np.random.default_rng(8)
    c = oracle.encode(code, rng.integers(0, 2, (2, code.k), dtype=np.uint8))
    R = (30.0 * (2.0 * c - 1.0)).astype(np.float32)
    L, z, it, so = oracle.spa_decode(code, R, 5)
    assert np.array_equal(z, c) and np.all(so == 1)
    assert np.all(np.sign(L) == 2.0 * c - 1.0)


def test_spa_fig1_agrees_with_ml(oracle):
    """S:573 acceptance #4: on Fig. 1's (2,4) n = 8 code at sigma = 0.4, the
    SPA hard decision equals the exhaustive ML codeword in >= 95% of 500 trials."""
    H = hp.golden_matrix("fig1_H.txt")
    code = oracle.Code.from_dense(H).make_G()
    rng = np.random.default_rng(9)
    cws = hp.codewords(H)
    agree = 0
    for _ in range(500):
        x = cws[rng.integers(0, len(cws))]
        y = (2.0 * x - 1.0) + 0.4 * rng.standard_normal(8)
        R = (2 * y / 0.16).astype(np.float32)
        _, z, *_ = oracle.spa_decode(code, R, 10)
        agree += int(np.array_equal(z[0], hp.ml_decode(H, R)))
    assert agree >= 475


def test_spa_coding_gain(oracle):
    """S:574 acceptance #5: at uncoded BER ~ 1e-2 the (3,6) n = 1008 code's
    decoded info BER is at least 5x lower."""
    code = oracle.make_H(1008, 3, 6, 1).make_G()
    sigma = 1.0 / 2.3263          # Q(1/sigma) = 0.01
    F = 30
    info = oracle.gen_info(11, 0, F, code.k)
    c = oracle.encode(code, info)
    R = oracle.channel(12, 0, c, sigma)
    uncoded = np.mean((R >= 0).astype(np.uint8) != c)
    _, z, it, so = oracle.spa_decode(code, R, 50, early_term=True)
    coded = np.mean(z[:, code.perm[:code.k]] != info)
    assert 0.005 < uncoded < 0.02
    assert coded * 5 <= uncoded


def test_spa_early_termination_consistent_with_fixed_trace(oracle):
    """Reading c6: the early-termination count is the first t whose hard
    decision has zero syndrome in the fixed-iteration trace, and the outputs
    equal the fixed-mode outputs at that t."""
    code = oracle.make_H(96, 3, 6, 1).make_G()
    H = code.dense().astype(np.int64)
    info = oracle.gen_info(21, 0, 6, code.k)
    R = oracle.channel(22, 0, oracle.encode(code, info), 0.85)
    Le, ze, ite, soe = oracle.spa_decode(code, R, 30, early_term=True)
    for f in range(R.shape[0]):
        first = None
        for t in range(1, 31):
            L, z, it, so = oracle.spa_decode(code, R[f], t)
            if not np.any((H @ z[0].astype(np.int64)) % 2):      # Eq. 1 by numpy, not the oracle
                first = t
                assert np.array_equal(L[0], Le[f]) and np.array_equal(z[0], ze[f])
                break
        if first is None:
            assert ite[f] == 30 and soe[f] == 0
        else:
            assert ite[f] == first and soe[f] == 1


# ----------------------------------------------------------------- partition
def test_partition_eq9(oracle):
    """Eq. 9, corrected per S:336: S:339-341 examples and the
    invariants of S:380-384 over (l, N) in [0, 1000] x [1, 64]."""
    c, d = oracle.partition(10, 4)
    assert list(c) == [3, 3, 2, 2] and list(d) == [0, 3, 6, 8]
    c, d = oracle.partition(4, 4)
    assert list(c) == [1, 1, 1, 1]
    c, d = oracle.partition(0, 3)
    assert list(c) == [0, 0, 0]
    for l in range(0, 1001, 7):
        for N in range(1, 65):
            c, d = oracle.partition(l, N)
            assert c.sum() == l and c.max() - c.min() <= 1
            assert np.all(np.diff(c) <= 0)
            assert d[0] == 0 and np.array_equal(d[1:], np.cumsum(c)[:-1])


def test_count_errors_hand_example(oracle):
    H = hp.hamming74_H()
    code = oracle.Code.from_dense(H).make_G()
    info = np.array([[1, 0, 1, 1], [0, 0, 0, 0]], np.uint8)
    c = oracle.encode(code, info)
    z = c.copy()
    z[0, code.perm[1]] ^= 1       # one info-bit error in frame 0
    z[1, code.perm[5]] ^= 1       # one parity-bit error in frame 1
    out = oracle.count_errors(code, info, z, c, np.array([0, 1], np.uint8), np.array([3, 7], np.int32))
    assert list(out) == [1, 2, 1, 1, 10, 2]


# ---------------------------------------------------------------------------
# SPA on graphs WITH cycles (Alg. 1): T flooding
# iterations give, at every variable, the exact bitwise MAP of the depth-T
# computation tree (the graph unwrapped from that variable, every copy of a
# variable observed through its own copy of R).  The trees are enumerated by
# brute force (tests/helpers.py), nothing of the oracle is reused.

def _k4_edge_vertex_H():
    """Variables = the 6 edges of K4, checks = its 4 vertices: variable degree
    2, check degree 3 (odd: exercises the (-1)^d rule, reading Q3), girth 6."""
    edges = [(a, b) for a in range(4) for b in range(a + 1, 4)]
    H = np.zeros((4, 6), dtype=np.uint8)
    for j, (a, b) in enumerate(edges):
        H[a, j] = H[b, j] = 1
    return H


@pytest.mark.parametrize("name", ["k4", "hamming74", "fig1"])
def test_spa_on_cyclic_graphs_equals_map_on_computation_tree(oracle, name):
    H = {"k4": _k4_edge_vertex_H, "hamming74": hp.hamming74_H, "fig1": lambda: hp.golden_matrix("fig1_H.txt")}[name]()
    assert not hp.is_tree(H)
    code = oracle.Code.from_dense(H)
    rng = np.random.default_rng(41)
    n = H.shape[1]
    checked = {1: 0, 2: 0, 3: 0}
    wrapped = 0
    for _ in range(12):
        R = rng.normal(0.0, 1.6, n).astype(np.float32)
        for T in (1, 2, 3):
            L, *_ = oracle.spa_decode(code, R, max_iter=T)
            for v in range(n):
                var_of, par, kids = hp.computation_tree(H, v, T)
                want = hp.tree_root_map_llr(var_of, par, kids, R, max_free=17)
                if want is None:
                    continue
                assert abs(L[0, v] - want) < 1e-9, (name, T, v, L[0, v], want)
                checked[T] += 1
                wrapped += int(len(set(var_of)) < len(var_of))     # some variable appears more than once
    assert checked[1] >= 12 * n and checked[2] > 0
    assert wrapped > 0          # the trees really unwrapped a cycle (replicated variables)
    if name == "k4":
        assert checked[3] == 12 * n
        # and the result is NOT the code's MAP: cycles over-count evidence
        L, *_ = oracle.spa_decode(code, R, max_iter=3)
        assert np.max(np.abs(L[0] - hp.map_llr(H, R))) > 1e-3


def test_spa_ring_closed_form(oracle):
    """A single cycle: checks x_i + x_{i+1 mod n} = 0.  Degree-2 checks pass the
    other input through unchanged (2 atanh(tanh(x/2)) = x), so T iterations
    give L_v = R_v + sum_{d=1..T} (R_{v+d} + R_{v-d}) with indices mod n --
    evidence counted again on every lap, unlike the MAP sum_u R_u."""
    n = 5
    H = np.zeros((n, n), dtype=np.uint8)
    for i in range(n):
        H[i, i] = H[i, (i + 1) % n] = 1
    code = oracle.Code.from_dense(H)
    rng = np.random.default_rng(42)
    for _ in range(10):
        R = rng.normal(0.0, 0.4, n).astype(np.float32)
        Rd = R.astype(np.float64)
        for T in (1, 2, 3, 7, 12):
            L, *_ = oracle.spa_decode(code, R, max_iter=T)
            want = np.array([Rd[v] + sum(Rd[(v + d) % n] + Rd[(v - d) % n] for d in range(1, T + 1)) for v in range(n)])
            assert np.max(np.abs(L[0] - want)) < 1e-9


def test_tree_marginaliser_equals_codeword_enumeration():
    """tests/helpers.py computation_tree_map_llr (the tree code marginalised
    check by check in the probability domain) against the enumeration of ALL
    codewords of the same computation tree: K4's edge-vertex graph,
    Hamming(7,4), Fig. 1; T = 1..3."""
    rng = np.random.default_rng(44)
    for H in (_k4_edge_vertex_H(), hp.hamming74_H(), hp.golden_matrix("fig1_H.txt")):
        for _ in range(4):
            R = rng.normal(0.0, 1.6, H.shape[1]).astype(np.float32)
            done = 0
            for T in (1, 2, 3):
                dp = hp.computation_tree_map_llr(H, R, T)
                for v in range(H.shape[1]):
                    want = hp.tree_root_map_llr(*hp.computation_tree(H, v, T), R, max_free=17)
                    if want is not None:
                        assert abs(dp[v] - want) < 1e-10
                        done += 1
            assert done > H.shape[1]


@pytest.mark.parametrize("n,wc,wr,ebn0,Ts,nroots", [(96, 3, 6, 2.0, (1, 2, 3, 4, 6), None), (1008, 3, 6, 1.5, (1, 2, 3, 5), None),
                                                     (3996, 3, 4, 2.5, (1, 2, 4), 300), (3996, 3, 6, 2.5, (1, 3), 300),
                                                     (1032, 3, 12, 2.5, (1, 2), 12), (1032, 9, 12, 2.5, (1,), 6),
                                                     (3996, 3, 12, 2.5, (1, 2), 10), (16200, 3, 6, 1.5, (1, 2, 3), 150),
                                                     (64800, 3, 6, 1.2, (1, 2), 100)])
def test_spa_on_config_codes_equals_computation_tree_map(oracle, n, wc, wr, ebn0, Ts, nroots):
    """The configs' own Gallager codes (C1, C2, C3, Table I, C4, C5; all with
    cycles) at the configs' noise: T flooding iterations of the oracle
    equal the exact MAP of the depth-T computation tree within 1e-9 at every
    (sampled) variable.  (Beyond ~6 iterations the two fp precisions drift
    apart on these graphs -- DESIGN.md §4 rule 2 -- so the pin stops there.)"""
    code = oracle.make_H(n, wc, wr, 1)
    H = (code.n, code.row_ptr, code.col_idx)        # CSR: n = 64800 does not fit densely
    rng = np.random.default_rng(45)
    sigma = math.sqrt(1.0 / (2.0 * (1.0 - wc / wr) * 10 ** (ebn0 / 10)))
    y = -1.0 + sigma * rng.standard_normal((2, n))
    R = np.clip(2.0 * y / sigma ** 2, -20, 20).astype(np.float32)
    roots = None if nroots is None else rng.choice(n, nroots, replace=False)
    compared = 0
    for T in Ts:
        L, *_ = oracle.spa_decode(code, R, max_iter=T)
        for f in range(R.shape[0]):
            want = hp.computation_tree_map_llr(H, R[f], T, roots)
            sel = ~np.isnan(want)
            assert sel.sum() == (n if roots is None else nroots)
            if np.max(np.abs(want[sel])) > 25:          # keep clear of the clamps (reading Q7)
                continue
            assert np.max(np.abs(L[f][sel] - want[sel])) < 1e-9, (T, f)
            compared += 1
    assert compared >= len(Ts)                  # at most half the (T, frame) cases may sit near the clamps


def test_early_termination_equals_first_zero_syndrome_of_computation_tree(oracle):
    """C2's code at 3.0 dB: the oracle's early-terminated decode stops at the
    first T whose exact T-iteration posteriors (tree marginaliser, not the
    oracle) decide a codeword, with those decisions and a set syndrome flag
    (Eqs. 1, 8; reading Q11)."""
    code = oracle.make_H(1008, 3, 6, 1)
    csr = (code.n, code.row_ptr, code.col_idx)
    rng = np.random.default_rng(47)
    sigma = math.sqrt(1.0 / (2.0 * 0.5 * 10 ** 0.3))
    y = -1.0 + sigma * rng.standard_normal((4, 1008))
    R = np.clip(2.0 * y / sigma ** 2, -20, 20).astype(np.float32)
    L, z, it, so = oracle.spa_decode(code, R, max_iter=50, early_term=True)
    stops = set()
    for f in range(4):
        T, Lt, zt = hp.computation_tree_first_zero_syndrome(csr, R[f], 8)
        assert T is not None and np.min(np.abs(Lt)) > 1e-3      # decisions are not near ties
        assert int(it[f]) == T and int(so[f]) == 1
        assert np.array_equal(z[f], zt)
        assert np.max(np.abs(L[f] - Lt)) < 1e-5
        stops.add(T)
    assert len(stops) > 1       # different stopping iterations were exercised
