"""CPU tests of the library's host side (no GPU): H/G construction is
bit-exact with the oracle, the C ABI exports every declared symbol, argument
errors are reported, and the product package never touches oracle/."""
import os
import re

import numpy as np
import pytest

from tests import helpers as hp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import paper_2201_04265_b200 as L
    return L


def _pack_P_columns(P: np.ndarray) -> np.ndarray:
    """oracle P (k x (n-k) bytes) -> the ABI layout uint32 [(n-k), ceil(k/32)]."""
    k, npar = P.shape
    kw = (k + 31) // 32
    out = np.zeros((npar, kw), dtype=np.uint64)
    for a in range(k):
        out[:, a // 32] |= (P[a].astype(np.uint64) << np.uint64(a % 32))
    return out.astype(np.uint32)


def test_header_symbols_exported(L):
    hdr = open(os.path.join(ROOT, "include", "ldpc.h")).read()
    declared = set(re.findall(r"\b(ldpc_[a-zA-Z0-9_]+)\s*\(", hdr))
    assert declared == set(L._lib.EXPORTED)
    lib = L._lib.lib()
    for name in declared:
        assert hasattr(lib, name), name


def test_product_package_does_not_use_oracle():
    pkg = os.path.join(ROOT, "paper_2201_04265_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", "Makefile")):
                txt = open(os.path.join(dirpath, f)).read()
                bad = re.findall(r"(import\s+oracle|from\s+oracle|#include\s+[<\"].*oracle|liboracle|ldpc_oracle)", txt)
                assert not bad, (f, bad)


@pytest.mark.parametrize("n,wc,wr,seed", [(96, 3, 6, 1), (1008, 3, 6, 1), (3996, 3, 4, 1), (3996, 3, 6, 1),
                                          (3996, 3, 12, 1), (1032, 9, 12, 1), (1032, 6, 12, 7), (16200, 3, 6, 1)])
def test_make_H_bit_exact(L, oracle, n, wc, wr, seed):
    lib_code = L.ldpc_make_H(n, wc, wr, seed)
    ora = oracle.make_H(n, wc, wr, seed)
    rp, ci = L.ldpc_code_copy_csr(lib_code)
    assert np.array_equal(rp, ora.row_ptr)
    assert np.array_equal(ci, ora.col_idx)
    info = lib_code.info
    assert (info.n, info.m, info.nnz, info.wc, info.wr) == (n, n * wc // wr, n * wc, wc, wr)
    assert info.max_row_deg == wr and info.max_col_deg == wc


@pytest.mark.parametrize("n,wc,wr", [(96, 3, 6), (1008, 3, 6), (3996, 3, 4), (3996, 3, 6), (3996, 3, 12),
                                     (1032, 9, 12), (1032, 6, 12), (1032, 3, 12), (16200, 3, 6)])
def test_make_G_bit_exact(L, oracle, n, wc, wr):
    lib_code = L.ldpc_make_G(L.ldpc_make_H(n, wc, wr, 1))
    ora = oracle.make_H(n, wc, wr, 1).make_G()
    info = lib_code.info
    assert info.k == ora.k and info.rank == ora.rank
    assert np.array_equal(L.ldpc_code_copy_perm(lib_code), ora.perm)
    assert np.array_equal(L.ldpc_code_copy_P(lib_code), _pack_P_columns(ora.P))


def test_make_G_small_codes_bit_exact(L, oracle):
    G2 = hp.golden_matrix("fig2_G.txt")
    mats = [hp.golden_matrix("fig1_H.txt"), hp.hamming74_H(),
            np.concatenate([G2[:, 4:].T, np.eye(4, dtype=np.uint8)], axis=1)]
    rng = np.random.default_rng(0)
    for _ in range(20):
        mats.append(hp.random_tree_H(rng, 14))
        mats.append((rng.random((int(rng.integers(2, 9)), int(rng.integers(9, 40)))) < 0.3).astype(np.uint8))
    for H in mats:
        ora = oracle.Code.from_dense(H)
        lib_code = L.ldpc_code_from_csr(ora.m, ora.n, ora.row_ptr, ora.col_idx)
        assert np.array_equal(L.ldpc_code_copy_H(lib_code), H)
        if hp.gf2_rank(H) == H.shape[1]:
            with pytest.raises(L.LdpcError):
                L.ldpc_make_G(lib_code)
            continue
        L.ldpc_make_G(lib_code)
        ora.make_G()
        assert lib_code.info.k == ora.k
        assert np.array_equal(L.ldpc_code_copy_perm(lib_code), ora.perm)
        assert np.array_equal(L.ldpc_code_copy_P(lib_code), _pack_P_columns(ora.P))


def test_argument_errors(L):
    with pytest.raises(L.LdpcError) as e:
        L.ldpc_make_H(4000, 3, 6, 1)
    assert e.value.status == 2   # LDPC_ERR_NOT_DIVISIBLE (reading Q16)
    with pytest.raises(L.LdpcError):
        L.ldpc_make_H(96, 6, 6, 1)
    with pytest.raises(L.LdpcError):   # duplicate column in a row
        L.ldpc_code_from_csr(1, 4, [0, 2], [1, 1])
    with pytest.raises(L.LdpcError) as e:   # degree 33 > 32
        L.ldpc_code_from_csr(1, 40, [0, 33], list(range(33)))
    assert e.value.status == 6
    c = L.ldpc_make_H(96, 3, 6, 1)
    with pytest.raises(L.LdpcError) as e:   # perm before make_G
        L.ldpc_code_copy_perm(c)
    assert e.value.status == 5


def test_partition_matches_oracle(L, oracle):
    for l in (0, 1, 7, 10, 999, 1000000):
        for N in (1, 2, 3, 4, 8, 64):
            c1, d1 = L.ldpc_partition(l, N)
            c2, d2 = oracle.partition(l, N)
            assert np.array_equal(c1, c2) and np.array_equal(d1, d2)
