"""ctypes wrapper around oracle/liboracle.so -- the CPU ORACLE.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs.  The product package
``paper_2201_04265_b200`` never imports this module (a test asserts it).

Every function forwards to the plain C implementation in ldpc_oracle.c, which
cites the paper passage it follows.  Marshalling only: bits travel as one
uint8 per bit, LLRs as float32 (inputs) / float64 (posteriors).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ldpc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile ldpc_oracle.c with plain gcc (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.POINTER
        L.oracle_splitmix64_next.restype = C.c_uint64
        L.oracle_splitmix64_next.argtypes = [P(C.c_uint64)]
        L.oracle_uniform_below.restype = C.c_uint64
        L.oracle_uniform_below.argtypes = [P(C.c_uint64), C.c_uint64]
        L.oracle_make_H.restype = C.c_int
        L.oracle_make_H.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]
        L.oracle_make_G.restype = C.c_void_p
        L.oracle_make_G.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]
        L.oracle_G_k.restype = C.c_int32
        L.oracle_G_k.argtypes = [C.c_void_p]
        L.oracle_G_rank.restype = C.c_int32
        L.oracle_G_rank.argtypes = [C.c_void_p]
        L.oracle_G_perm.argtypes = [C.c_void_p, C.c_void_p]
        L.oracle_G_P.argtypes = [C.c_void_p, C.c_void_p]
        L.oracle_G_free.argtypes = [C.c_void_p]
        L.oracle_encode.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int64, C.c_void_p]
        L.oracle_syndrome_zero.restype = C.c_int
        L.oracle_syndrome_zero.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_philox4x32_10.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_gen_info.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p]
        L.oracle_channel.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                     C.c_double, C.c_void_p]
        L.oracle_channel_y.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                       C.c_double, C.c_void_p]
        L.oracle_llr.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p]
        L.oracle_spa_decode_batch.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_partition.argtypes = [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.oracle_count_errors.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- PRNGs
def splitmix64_stream(seed: int, count: int) -> list[int]:
    st = C.c_uint64(seed)
    return [lib().oracle_splitmix64_next(C.byref(st)) for _ in range(count)]


def uniform_below_stream(seed: int, bound: int, count: int) -> list[int]:
    st = C.c_uint64(seed)
    return [lib().oracle_uniform_below(C.byref(st), bound) for _ in range(count)]


def philox4x32_10(ctr, key) -> list[int]:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(o))
    return [int(x) for x in o]


# ---------------------------------------------------------------- codes
class Code:
    """A parity-check matrix as CSR (rows = checks), plus (optionally) G."""

    def __init__(self, m: int, n: int, row_ptr, col_idx):
        self.m, self.n = int(m), int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.k = None
        self.rank = None
        self.perm = None
        self.P = None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def dense(self) -> np.ndarray:
        H = np.zeros((self.m, self.n), dtype=np.uint8)
        for c in range(self.m):
            for e in range(self.row_ptr[c], self.row_ptr[c + 1]):
                H[c, self.col_idx[e]] ^= 1
        return H

    @staticmethod
    def from_dense(H) -> "Code":
        H = np.asarray(H, dtype=np.uint8)
        m, n = H.shape
        rp = [0]
        ci = []
        for c in range(m):
            cols = np.nonzero(H[c])[0]
            ci.extend(int(x) for x in cols)
            rp.append(len(ci))
        return Code(m, n, np.array(rp, np.int32), np.array(ci, np.int32))

    def make_G(self) -> "Code":
        L = lib()
        g = L.oracle_make_G(self.m, self.n, _p(self.row_ptr), _p(self.col_idx))
        try:
            self.k = L.oracle_G_k(g)
            self.rank = L.oracle_G_rank(g)
            self.perm = np.zeros(self.n, dtype=np.int32)
            L.oracle_G_perm(g, _p(self.perm))
            self.P = np.zeros((self.k, self.n - self.k), dtype=np.uint8)
            if self.P.size:
                L.oracle_G_P(g, _p(self.P))
        finally:
            L.oracle_G_free(g)
        return self

    def G_dense(self) -> np.ndarray:
        """G in H column order: row a is the codeword of unit message e_a."""
        Gp = np.concatenate([np.eye(self.k, dtype=np.uint8), self.P], axis=1)
        G = np.zeros_like(Gp)
        G[:, self.perm] = Gp
        return G


def make_H(n: int, wc: int, wr: int, seed: int) -> Code:
    """Gallager (wc, wr) band construction; raises ValueError on bad args."""
    m = n * wc // wr if wr else 0
    cols = np.zeros(max(m * wr, 1), dtype=np.int32)
    rc = lib().oracle_make_H(n, wc, wr, seed, _p(cols))
    if rc == 1:
        raise ValueError("wr does not divide n")
    if rc != 0:
        raise ValueError("bad (n, wc, wr)")
    rp = np.arange(0, m * wr + 1, wr, dtype=np.int32)
    return Code(m, n, rp, cols[: m * wr])


def encode(code: Code, m_bits: np.ndarray) -> np.ndarray:
    m_bits = np.ascontiguousarray(m_bits, dtype=np.uint8).reshape(-1, code.k)
    F = m_bits.shape[0]
    c = np.zeros((F, code.n), dtype=np.uint8)
    P = np.ascontiguousarray(code.P, dtype=np.uint8)
    lib().oracle_encode(code.k, code.n, _p(code.perm), _p(P), _p(m_bits), F, _p(c))
    return c


def syndrome_zero(code: Code, z: np.ndarray) -> bool:
    z = np.ascontiguousarray(z, dtype=np.uint8)
    return bool(lib().oracle_syndrome_zero(code.m, _p(code.row_ptr), _p(code.col_idx), _p(z)))


def gen_info(seed: int, frame0: int, frames: int, k: int) -> np.ndarray:
    out = np.zeros((frames, k), dtype=np.uint8)
    lib().oracle_gen_info(seed, frame0, frames, k, _p(out))
    return out


def channel(seed: int, frame0: int, c: np.ndarray, sigma: float) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.uint8)
    F, n = c.shape
    R = np.zeros((F, n), dtype=np.float32)
    lib().oracle_channel(seed, frame0, F, n, _p(c), float(sigma), _p(R))
    return R


def channel_y(seed: int, frame0: int, c: np.ndarray, sigma: float) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.uint8)
    F, n = c.shape
    y = np.zeros((F, n), dtype=np.float64)
    lib().oracle_channel_y(seed, frame0, F, n, _p(c), float(sigma), _p(y))
    return y


def llr(y: np.ndarray, sigma: float) -> np.ndarray:
    y = np.ascontiguousarray(y, dtype=np.float64)
    R = np.zeros(y.shape, dtype=np.float32)
    lib().oracle_llr(_p(y), y.size, float(sigma), _p(R))
    return R


def spa_decode(code: Code, R: np.ndarray, max_iter: int, early_term: bool = False):
    """Returns (L float64 [F,n], z uint8 [F,n], iters int32 [F], syn_ok uint8 [F])."""
    R = np.ascontiguousarray(R, dtype=np.float32).reshape(-1, code.n)
    F = R.shape[0]
    L = np.zeros((F, code.n), dtype=np.float64)
    z = np.zeros((F, code.n), dtype=np.uint8)
    it = np.zeros(F, dtype=np.int32)
    so = np.zeros(F, dtype=np.uint8)
    lib().oracle_spa_decode_batch(code.m, code.n, _p(code.row_ptr), _p(code.col_idx), _p(R), F,
                                  int(max_iter), int(bool(early_term)), _p(L), _p(z), _p(it), _p(so))
    return L, z, it, so


def partition(l: int, N: int):
    counts = np.zeros(N, dtype=np.int64)
    displs = np.zeros(N, dtype=np.int64)
    lib().oracle_partition(l, N, _p(counts), _p(displs))
    return counts, displs


def count_errors(code: Code, info, z, c, syn_ok, iters) -> np.ndarray:
    info = np.ascontiguousarray(info, dtype=np.uint8)
    z = np.ascontiguousarray(z, dtype=np.uint8)
    c = np.ascontiguousarray(c, dtype=np.uint8)
    syn_ok = np.ascontiguousarray(syn_ok, dtype=np.uint8)
    iters = np.ascontiguousarray(iters, dtype=np.int32)
    out = np.zeros(6, dtype=np.int64)
    lib().oracle_count_errors(code.k, code.n, _p(code.perm), _p(info), _p(z), _p(c), _p(syn_ok),
                              _p(iters), z.shape[0], _p(out))
    return out
