"""MacKay alist import/export (acceptance 9 at S:578; the
paper's demo claim that any binary parity-check matrix can be used, P:4).
The Fig. 1 alist under tests/golden/ was written by hand from the paper's
matrix, independently of the library."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def L():
    import paper_2201_04265_b200 as L
    return L


def _fig1_H():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "fig1_H.txt")) if l.strip() and not l.startswith("#")]
    return np.array([[int(x) for x in r] for r in rows], dtype=np.uint8)


def _code_from_dense(L, H):
    m, n = H.shape
    rp = np.zeros(m + 1, np.int32)
    ci = []
    for r in range(m):
        cols = np.nonzero(H[r])[0]
        ci.extend(cols.tolist())
        rp[r + 1] = len(ci)
    return L.ldpc_code_from_csr(m, n, rp, np.array(ci, np.int32))


def test_fig1_alist_matches_golden(L):
    want = open(os.path.join(GOLDEN, "fig1.alist")).read()
    code = _code_from_dense(L, _fig1_H())
    assert L.ldpc_code_write_alist(code) == want
    back = L.ldpc_code_from_alist(want)
    assert np.array_equal(L.ldpc_code_copy_H(back), _fig1_H())


@pytest.mark.parametrize("n,wc,wr", [(96, 3, 6), (1032, 9, 12), (3996, 3, 4), (16200, 3, 6)])
def test_round_trip_constructed_codes(L, n, wc, wr):
    """write -> read -> write is identical text, the matrix is bit-identical,
    and make_G of the re-imported H gives the same k, perm and P (the
    standard form depends only on H, reading Q13)."""
    code = L.ldpc_make_H(n, wc, wr, 1)
    text = L.ldpc_code_write_alist(code)
    lines = text.splitlines()
    assert lines[0] == f"{n} {n * wc // wr}" and lines[1] == f"{wc} {wr}"
    assert len(lines) == 4 + n + n * wc // wr
    back = L.ldpc_code_from_alist(text)
    assert L.ldpc_code_write_alist(back) == text
    if n <= 4000:
        assert np.array_equal(L.ldpc_code_copy_H(back), L.ldpc_code_copy_H(code))
    else:
        # CSR rows may list columns in another order: compare sorted rows
        rp0, ci0 = L.ldpc_code_copy_csr(code)
        rp1, ci1 = L.ldpc_code_copy_csr(back)
        assert np.array_equal(rp0, rp1)
        for r in range(0, len(rp0) - 1, 97):
            assert sorted(ci0[rp0[r]:rp0[r + 1]]) == sorted(ci1[rp1[r]:rp1[r + 1]])
    if n <= 1032:
        L.ldpc_make_G(code)
        L.ldpc_make_G(back)
        assert code.info.k == back.info.k
        assert np.array_equal(L.ldpc_code_copy_perm(code), L.ldpc_code_copy_perm(back))
        assert np.array_equal(L.ldpc_code_copy_P(code), L.ldpc_code_copy_P(back))


def test_irregular_code_zero_padding(L):
    """Rows and columns below the maximum weight are padded with literal 0s."""
    H = np.array([[1, 1, 1, 0, 0],
                  [0, 1, 0, 1, 0],
                  [0, 0, 0, 0, 1]], np.uint8)
    text = L.ldpc_code_write_alist(_code_from_dense(L, H))
    assert text.splitlines() == ["5 3", "2 3", "1 2 1 1 1", "3 2 1",
                                 "1 0", "1 2", "1 0", "2 0", "3 0",
                                 "1 2 3", "2 4 0", "5 0 0"]
    assert np.array_equal(L.ldpc_code_copy_H(L.ldpc_code_from_alist(text)), H)
    # unpadded lists are accepted too
    unpadded = "\n".join(["5 3", "2 3", "1 2 1 1 1", "3 2 1", "1", "1 2", "1", "2", "3", "1 2 3", "2 4", "5"])
    assert np.array_equal(L.ldpc_code_copy_H(L.ldpc_code_from_alist(unpadded)), H)


@pytest.mark.parametrize("bad,status", [
    ("8 4\n2 4\n", 1),                                               # truncated header
    ("8 4\n2 x\n", 1),                                               # not a number
])
def test_malformed_rejected(L, bad, status):
    with pytest.raises(L._lib.LdpcError) as e:
        L.ldpc_code_from_alist(bad)
    assert e.value.status == status


def test_inconsistent_lists_rejected(L):
    good = open(os.path.join(GOLDEN, "fig1.alist")).read().splitlines()
    for i, repl in [(4, "1 2"),          # column 1 lists row 2 instead of 3
                    (12, "1 2 6 6"),     # row 1 repeats a column (weight mismatch)
                    (2, "2 2 2 2 2 2 2 1"),   # column weight disagrees with its list
                    (15, "3 4 5 9")]:    # column index out of range
        bad = list(good)
        bad[i] = repl
        with pytest.raises(L._lib.LdpcError) as e:
            L.ldpc_code_from_alist("\n".join(bad) + "\n")
        assert e.value.status in (1, 4), (i, e.value.status)
