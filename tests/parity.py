"""Decode-parity comparator: the acceptance rule of DESIGN.md "Parity"
(SURVEY.md §8c), applied frame by frame between the CUDA decoder and the
oracle, with the oracle run in parallel host threads (ctypes releases the GIL).

Rule:
 1. The oracle decodes the exact fp32 LLR buffer the GPU decoded, and again
    with every LLR moved by one fp32 ulp in a random direction (fixed seed),
    a relative perturbation of 2^-24..2^-23.
 2. A frame is ILL-CONDITIONED if the oracle's two posteriors (clipped to
    +-30) differ by more than 1e-4 anywhere.  `exempt=False` disables this.
 3. On well-conditioned frames: posteriors clipped to +-30 agree within
    1e-3 absolute or 1e-4 relative; hard decisions agree except where
    |L_oracle| < 1e-3; syndrome flags agree; iteration counts agree.
 4. Ill-conditioned frames are counted and reported; their hard decisions
    are gated only on STABLE bits: both oracle runs agree in sign and |L|
    exceeds max(1e-3, 10 s_f), s_f = the frame's measured sensitivity
    max|L1 - L2| (a bit whose margin is within the frame's own chaos scale is
    not decided by the algorithm but by rounding).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

ABS_TOL = 1e-3
REL_TOL = 1e-4
PROBE_TOL = 1e-4
CLIP = 30.0


def oracle_decode_parallel(O, code, R: np.ndarray, max_iter: int, early_term: bool, threads: int | None = None):
    R = np.ascontiguousarray(R, dtype=np.float32)
    F = R.shape[0]
    threads = threads or max(1, min(os.cpu_count() or 1, 64))
    chunks = np.array_split(np.arange(F), min(threads, max(F, 1)))
    outs = [None] * len(chunks)

    def run(i):
        idx = chunks[i]
        if len(idx):
            outs[i] = O.spa_decode(code, R[idx], max_iter, early_term)

    with ThreadPoolExecutor(len(chunks)) as ex:
        list(ex.map(run, range(len(chunks))))
    outs = [o for o in outs if o is not None]
    return tuple(np.concatenate([o[j] for o in outs]) for j in range(4))


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    w = np.ascontiguousarray(words).view(np.uint32)
    bits = ((w[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1).astype(np.uint8)
    return bits.reshape(w.shape[0], -1)[:, :n]


@dataclass
class ParityReport:
    frames: int
    exempt: int
    max_abs_err_ok: float
    max_abs_err_exempt: float
    failures: list

    def __str__(self):
        return (f"frames={self.frames} exempt={self.exempt} max|dL|={self.max_abs_err_ok:.3g} "
                f"(exempt max {self.max_abs_err_exempt:.3g}) failures={len(self.failures)}")


def compare(O, code, R: np.ndarray, gpu_L: np.ndarray, gpu_z: np.ndarray, gpu_syn: np.ndarray,
            gpu_it: np.ndarray, max_iter: int, early_term: bool, exempt: bool = True,
            seed: int = 12345) -> ParityReport:
    R = np.ascontiguousarray(R, dtype=np.float32)
    L1, z1, it1, so1 = oracle_decode_parallel(O, code, R, max_iter, early_term)
    if exempt:
        rng = np.random.default_rng(seed)
        direction = np.where(rng.random(R.shape) < 0.5, np.float32(-np.inf), np.float32(np.inf))
        R2 = np.nextafter(R, direction).astype(np.float32)
        L2, *_ = oracle_decode_parallel(O, code, R2, max_iter, early_term)
        ill = np.max(np.abs(np.clip(L1, -CLIP, CLIP) - np.clip(L2, -CLIP, CLIP)), axis=1) > PROBE_TOL
    else:
        L2 = L1
        ill = np.zeros(R.shape[0], dtype=bool)
    a = np.clip(gpu_L.astype(np.float64), -CLIP, CLIP)
    b = np.clip(L1, -CLIP, CLIP)
    err = np.abs(a - b)
    bad_val = (err > ABS_TOL) & (err > REL_TOL * np.abs(b))
    z_diff = (gpu_z != z1) & (np.abs(L1) >= 1e-3)
    failures = []
    max_ok, max_ex = 0.0, 0.0
    for f in range(R.shape[0]):
        if ill[f]:
            max_ex = max(max_ex, float(err[f].max()))
            s_f = float(np.max(np.abs(np.clip(L1[f], -CLIP, CLIP) - np.clip(L2[f], -CLIP, CLIP))))
            margin = max(1e-3, 10.0 * s_f)
            stable = (np.sign(L1[f]) == np.sign(L2[f])) & (np.abs(L1[f]) >= margin) & (np.abs(L2[f]) >= margin)
            if np.any(z_diff[f] & stable):
                failures.append((f, "hard decision (ill-conditioned, stable bits)"))
            continue
        max_ok = max(max_ok, float(err[f].max()))
        if bad_val[f].any():
            failures.append((f, f"posterior max err {err[f].max():.3g}"))
        if z_diff[f].any():
            failures.append((f, "hard decision"))
        if int(gpu_syn[f]) != int(so1[f]):
            failures.append((f, f"syndrome flag gpu={int(gpu_syn[f])} oracle={int(so1[f])}"))
        if int(gpu_it[f]) != int(it1[f]):
            failures.append((f, f"iterations gpu={int(gpu_it[f])} oracle={int(it1[f])}"))
    return ParityReport(R.shape[0], int(ill.sum()), max_ok, max_ex, failures)
