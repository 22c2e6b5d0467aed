"""Independent test helpers: golden-file readers, brute-force GF(2) and MAP.

Nothing here calls the oracle or the CUDA library; these are the "something
other than itself" that the oracle's pins compare against.
"""
from __future__ import annotations

import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_lines(name: str) -> list[list[str]]:
    out = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                out.append(line.split())
    return out


def golden_matrix(name: str) -> np.ndarray:
    return np.array([[int(x) for x in row] for row in golden_lines(name)], dtype=np.uint8)


def hamming74_H() -> np.ndarray:
    """Textbook Hamming(7,4): column j (1-based) is the binary expansion of j."""
    return np.array([[(j >> b) & 1 for j in range(1, 8)] for b in range(3)], dtype=np.uint8)


def gf2_rank(H: np.ndarray) -> int:
    """GF(2) rank by left-to-right elimination on Python-int rows (independent
    of the oracle's right-to-left bit-packed Gauss-Jordan)."""
    rows = [int("".join(str(int(b)) for b in r[::-1]) or "0", 2) for r in np.asarray(H)]
    rank = 0
    ncols = H.shape[1]
    for col in range(ncols):
        bit = 1 << col
        piv = None
        for i in range(rank, len(rows)):
            if rows[i] & bit:
                piv = i
                break
        if piv is None:
            continue
        rows[rank], rows[piv] = rows[piv], rows[rank]
        for i in range(len(rows)):
            if i != rank and rows[i] & bit:
                rows[i] ^= rows[rank]
        rank += 1
    return rank


def codewords(H: np.ndarray) -> np.ndarray:
    """All x in GF(2)^n with H x = 0, by enumeration (n <= 20)."""
    H = np.asarray(H, dtype=np.int64)
    m, n = H.shape
    assert n <= 20
    xs = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1).astype(np.int64)
    s = (xs @ H.T) % 2
    return xs[np.all(s == 0, axis=1)].astype(np.uint8)


def map_llr(H: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Exact bitwise-MAP posterior LLRs ln(P(x_v=1|y)/P(x_v=0|y)) for LLR inputs
    R = ln(p1/p0) of independent bits, uniform prior over the code:
    P(x) ~ prod_u exp(x_u R_u).  Brute force over all codewords."""
    cw = codewords(H).astype(np.float64)
    R = np.asarray(R, dtype=np.float64)
    score = cw @ R
    out = np.zeros(H.shape[1])
    for v in range(H.shape[1]):
        s1 = score[cw[:, v] == 1]
        s0 = score[cw[:, v] == 0]
        out[v] = _lse(s1) - _lse(s0)
    return out


def _lse(a: np.ndarray) -> float:
    if a.size == 0:
        return -math.inf
    mx = a.max()
    return float(mx + np.log(np.exp(a - mx).sum()))


def ml_decode(H: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Block ML codeword: argmax_x sum_u x_u R_u over the code."""
    cw = codewords(H)
    return cw[np.argmax(cw.astype(np.float64) @ np.asarray(R, dtype=np.float64))]


def random_tree_H(rng: np.random.Generator, n_max: int = 16) -> np.ndarray:
    """A random cycle-free Tanner graph whose checks all have degree >= 2:
    grow from one variable; each new check attaches to one existing variable
    and 1..3 new ones."""
    nv = 1
    checks = []
    while True:
        add = int(rng.integers(1, 4))
        if nv + add > n_max:
            break
        anchor = int(rng.integers(0, nv))
        checks.append([anchor] + list(range(nv, nv + add)))
        nv += add
    H = np.zeros((len(checks), nv), dtype=np.uint8)
    for c, vs in enumerate(checks):
        H[c, vs] = 1
    # random relabelling of variables and checks keeps it a tree
    H = H[rng.permutation(H.shape[0])][:, rng.permutation(nv)]
    return H


def is_tree(H: np.ndarray) -> bool:
    """Connected and |E| = |V| + |C| - 1."""
    m, n = H.shape
    edges = int(H.sum())
    if edges != m + n - 1:
        return False
    seen = {("v", 0)}
    stack = [("v", 0)]
    while stack:
        kind, i = stack.pop()
        nbrs = [("c", c) for c in np.nonzero(H[:, i])[0]] if kind == "v" else \
               [("v", v) for v in np.nonzero(H[i])[0]]
        for nb in nbrs:
            if nb not in seen:
                seen.add(nb)
                stack.append(nb)
    return len(seen) == m + n


def q_function(x: float) -> float:
    return 0.5 * math.erfc(x / math.sqrt(2.0))


def computation_tree(H: np.ndarray, root: int, depth: int):
    """The computation tree of flooding SPA (Wiberg 1996; Richardson & Urbanke,
    Modern Coding Theory §3): the Tanner graph of H unwrapped from variable
    `root` for `depth` check hops.  A variable copy reached through check c
    expands through its other checks only; copies `depth` check hops from the
    root are leaves.  Returns (var_of, parent_of, children_of): var_of[i] is the
    original variable of tree variable i (0 = the root), children_of[j] the
    tree variables below tree check j, parent_of[j] the tree variable above
    it."""
    H = np.asarray(H)
    var_of, var_depth, var_from = [root], [0], [-1]
    parent_of, children_of = [], []
    i = 0
    while i < len(var_of):
        if var_depth[i] < depth:
            for c in np.flatnonzero(H[:, var_of[i]]):
                if c == var_from[i]:
                    continue
                kids = []
                for u in np.flatnonzero(H[c]):
                    if u == var_of[i]:
                        continue
                    var_of.append(int(u))
                    var_depth.append(var_depth[i] + 1)
                    var_from.append(int(c))
                    kids.append(len(var_of) - 1)
                parent_of.append(i)
                children_of.append(kids)
        i += 1
    return var_of, parent_of, children_of


def tree_root_map_llr(var_of, parent_of, children_of, R, max_free: int = 20):
    """Exact bitwise-MAP LLR ln(P(x_root = 1 | y) / P(x_root = 0 | y)) of the
    tree code defined by computation_tree(), every tree variable i observed
    through its own copy of R[var_of[i]]: brute force over ALL codewords of the
    tree code.  A codeword is fixed by the root, and per check by all but the
    last of its children (the last child closes the check's parity); checks
    appear in breadth-first order, so a check's parent is set before it.
    Returns None if the code has more than 2^max_free codewords."""
    free = 1 + sum(max(len(k) - 1, 0) for k in children_of)
    if free > max_free:
        return None
    N = 1 << free
    idx = np.arange(N, dtype=np.int64)
    x = np.zeros((len(var_of), N), dtype=np.int8)
    x[0] = idx & 1
    b = 1
    for p, kids in zip(parent_of, children_of):
        if not kids:                 # a degree-1 check forces its variable to 0
            return None
        acc = x[p].copy()
        for k in kids[:-1]:
            x[k] = (idx >> b) & 1
            b += 1
            acc ^= x[k]
        x[kids[-1]] = acc
    Rt = np.asarray(R, dtype=np.float64)[np.asarray(var_of)]
    score = Rt @ x.astype(np.float64)
    return _lse(score[x[0] == 1]) - _lse(score[x[0] == 0])


def computation_tree_map_llr(H: np.ndarray, R, depth: int, roots=None) -> np.ndarray:
    """Root MAP LLRs of the depth-`depth` computation trees of the variables in
    `roots` (default: all; other entries are NaN),
    by marginalising the tree code directly in the (log-)probability domain:
    a subtree's likelihood given its top variable's bit is the product over
    the checks below it of the sum, over every assignment of the check's other
    variables with the right parity (enumerated explicitly, 2^(d-1) terms), of
    the product of those variables' subtree likelihoods.  Subtrees depend only
    on (variable, check it hangs from, remaining depth), so they are shared
    between roots.  No tanh rule, no sign rule, no LLR messages: it is the
    definition of the marginal on a tree, and is itself checked against the
    enumeration of all tree codewords (tree_root_map_llr) in the CPU tests."""
    import functools
    import itertools
    Rd = np.asarray(R, dtype=np.float64)
    if isinstance(H, tuple):                    # (n, row_ptr, col_idx): CSR of a matrix too large to hold densely
        nvar, rp, ci = H
        rows = [[int(u) for u in ci[rp[c]:rp[c + 1]]] for c in range(len(rp) - 1)]
        cols = [[] for _ in range(nvar)]
        for c, r in enumerate(rows):
            for u in r:
                cols[u].append(c)
    else:
        H = np.asarray(H)
        nvar = H.shape[1]
        rows = [np.flatnonzero(H[c]).tolist() for c in range(H.shape[0])]
        cols = [np.flatnonzero(H[:, v]).tolist() for v in range(H.shape[1])]

    @functools.lru_cache(maxsize=None)
    def below_var(v, from_c, left):
        """(log P(subtree obs | x_v = 0), ... = 1) of the copy of v hanging from check from_c."""
        lp = [0.0, float(Rd[v])]
        if left > 0:
            for c in cols[v]:
                if c != from_c:
                    m = below_check(c, v, left)
                    lp[0] += m[0]
                    lp[1] += m[1]
        return tuple(lp)

    @functools.lru_cache(maxsize=None)
    def below_check(c, v, left):
        kids = [below_var(u, c, left - 1) for u in rows[c] if u != v]
        terms = ([], [])
        for bits in itertools.product((0, 1), repeat=len(kids)):
            terms[sum(bits) & 1].append(sum(k[b] for k, b in zip(kids, bits)))
        return (_lse(np.array(terms[0])), _lse(np.array(terms[1])))

    out = np.full(nvar, np.nan)
    for v in (range(nvar) if roots is None else roots):
        lp = below_var(int(v), -1, depth)
        out[v] = lp[1] - lp[0]
    return out


def computation_tree_first_zero_syndrome(csr, R, max_T: int):
    """Early termination from the definition (Eq. 8 hard decisions with ties to
    1, Eq. 1 syndrome; reading Q11: stop at the first iteration whose decisions
    satisfy every check): the smallest T <= max_T whose exact T-iteration
    posteriors (computation_tree_map_llr, every variable) decide a codeword.
    Returns (T, posteriors, decisions), or (None, None, None)."""
    n, rp, ci = csr
    for T in range(1, max_T + 1):
        L = computation_tree_map_llr(csr, R, T)
        z = (L >= 0).astype(np.int64)
        syn = np.add.reduceat(z[np.asarray(ci)], np.asarray(rp[:-1])) & 1
        if not syn.any():
            return T, L, z.astype(np.uint8)
    return None, None, None
