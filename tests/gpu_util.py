"""GPU-test helpers: build the same code on both sides, generate frames with
the ORACLE (CPU), upload them, and download GPU results."""
from __future__ import annotations

import numpy as np


def torch():
    import torch as t
    return t


def lib():
    import paper_2201_04265_b200 as L
    return L


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """uint8 [F, b] 0/1 -> uint32 [F, ceil(b/32)] LSB-first (test-side packing)."""
    F, b = bits.shape
    w = (b + 31) // 32
    padded = np.zeros((F, w * 32), dtype=np.uint64)
    padded[:, :b] = bits
    shifts = np.arange(32, dtype=np.uint64)[None, None, :]
    return (padded.reshape(F, w, 32) << shifts).sum(axis=2).astype(np.uint32)


def unpack_bits(words: np.ndarray, b: int) -> np.ndarray:
    w = np.ascontiguousarray(words).view(np.uint32)
    bits = ((w[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1).astype(np.uint8)
    return bits.reshape(w.shape[0], -1)[:, :b]


class Pair:
    """The same code on the library (GPU-bound) and oracle side."""

    def __init__(self, O, n=None, wc=None, wr=None, seed=1, H=None, with_G=True):
        L = lib()
        if H is not None:
            self.ora = O.Code.from_dense(H)
            self.lib = L.ldpc_code_from_csr(self.ora.m, self.ora.n, self.ora.row_ptr, self.ora.col_idx)
        else:
            self.ora = O.make_H(n, wc, wr, seed)
            self.lib = L.ldpc_make_H(n, wc, wr, seed)
        self.with_G = with_G
        if with_G:
            self.ora.make_G()
            L.ldpc_make_G(self.lib)
        L.ldpc_code_bind_device(self.lib)
        self.n = self.ora.n
        self.k = self.ora.k if with_G else None

    def frames(self, O, seed: int, frame0: int, F: int, sigma: float, zero_codeword: bool = False):
        """Oracle-generated info bits, codewords and fp32 LLRs (numpy)."""
        if zero_codeword or not self.with_G:
            info = None
            c = np.zeros((F, self.n), dtype=np.uint8)
        else:
            info = O.gen_info(seed, frame0, F, self.k)
            c = O.encode(self.ora, info)
        R = O.channel(seed, frame0, c, sigma)
        return info, c, R

    def decode(self, R: np.ndarray, max_iter: int, early_term: bool = False, variant: int = 0):
        t = torch()
        L = lib()
        llr = t.from_numpy(np.ascontiguousarray(R, dtype=np.float32)).cuda()
        out = L.decode(self.lib, llr, max_iter=max_iter, early_term=early_term, posterior=True, variant=variant)
        t.cuda.synchronize()
        bits = unpack_bits(out.bits.cpu().numpy(), self.n)
        return (out.posterior.cpu().numpy(), bits, out.syndrome_ok.cpu().numpy(), out.iters.cpu().numpy())
