"""Decode-parity comparator: the acceptance rule of DESIGN.md "Parity"
(SURVEY.md §8c), applied frame by frame between the CUDA decoder and the
oracle, with the oracle run in parallel host threads (ctypes releases the GIL).

Rule (SURVEY.md §8c "Acceptance rule for decode parity"):
 1. The oracle decodes the exact fp32 LLR buffer the GPU decoded, and again
    with every LLR moved by one fp32 ulp in a random direction (fixed seed),
    a relative perturbation of 2^-24..2^-23.
 2. A frame is ILL-CONDITIONED if the oracle's two posteriors (clipped to
    +-30) differ by more than 1e-4 anywhere.  `exempt=False` disables this.
 3. Every frame is gated: posteriors clipped to +-30 agree within 1e-3
    absolute or 1e-4 relative; hard decisions agree except where
    |L_oracle| < 1e-3; syndrome flags agree; iteration counts agree.
 4. A frame that fails 3 AND is ill-conditioned is EXEMPT from the posterior
    gate only.  Its hard decisions are still gated on the bits where both
    oracle runs agree in sign with |L| >= 1e-3, and its syndrome flag and
    iteration count wherever the two oracle runs agree on them.
 5. The exempt fraction is reported and gated (`max_exempt_frac`).
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
    ill: int = 0           # ill-conditioned frames (rule 2), whether or not they needed the exemption

    def __str__(self):
        return (f"frames={self.frames} ill={self.ill} exempt={self.exempt} max|dL|={self.max_abs_err_ok:.3g} "
                f"(exempt max {self.max_abs_err_exempt:.3g}) failures={len(self.failures)}")


def compare(O, code, R: np.ndarray, gpu_L: np.ndarray, gpu_z: np.ndarray, gpu_syn: np.ndarray,
            gpu_it: np.ndarray, max_iter: int, early_term: bool, exempt: bool = True,
            seed: int = 12345, max_exempt_frac: float = 0.02) -> ParityReport:
    R = np.ascontiguousarray(R, dtype=np.float32)
    F = R.shape[0]
    L1, z1, it1, so1 = oracle_decode_parallel(O, code, R, max_iter, early_term)
    if exempt:
        rng = np.random.default_rng(seed)
        direction = np.where(rng.random(R.shape) < 0.5, np.float32(-np.inf), np.float32(np.inf))
        R2 = np.nextafter(R, direction).astype(np.float32)
        L2, _, it2, so2 = oracle_decode_parallel(O, code, R2, max_iter, early_term)
        ill = np.max(np.abs(np.clip(L1, -CLIP, CLIP) - np.clip(L2, -CLIP, CLIP)), axis=1) > PROBE_TOL
    else:
        L2, it2, so2 = L1, it1, so1
        ill = np.zeros(F, dtype=bool)
    a = np.clip(gpu_L.astype(np.float64), -CLIP, CLIP)
    b = np.clip(L1, -CLIP, CLIP)
    err = np.abs(a - b)
    bad_val = (err > ABS_TOL) & (err > REL_TOL * np.abs(b))
    z_diff = (gpu_z != z1) & (np.abs(L1) >= 1e-3)
    stable = (np.sign(L1) == np.sign(L2)) & (np.abs(L1) >= 1e-3) & (np.abs(L2) >= 1e-3)
    failures = []
    max_ok, max_ex = 0.0, 0.0
    n_exempt = 0
    for f in range(F):
        syn_bad = int(gpu_syn[f]) != int(so1[f])
        it_bad = int(gpu_it[f]) != int(it1[f])
        passes = not (bad_val[f].any() or z_diff[f].any() or syn_bad or it_bad)
        if passes:
            max_ok = max(max_ok, float(err[f].max()))
            continue
        if ill[f]:
            n_exempt += 1
            max_ex = max(max_ex, float(err[f].max()))
            if np.any(z_diff[f] & stable[f]):
                failures.append((f, "hard decision (ill-conditioned, stable bits)"))
            if syn_bad and int(so1[f]) == int(so2[f]):
                failures.append((f, f"syndrome flag (ill-conditioned, oracle runs agree) gpu={int(gpu_syn[f])} "
                                    f"oracle={int(so1[f])}"))
            if it_bad and int(it1[f]) == int(it2[f]):
                failures.append((f, f"iterations (ill-conditioned, oracle runs agree) gpu={int(gpu_it[f])} "
                                    f"oracle={int(it1[f])}"))
            continue
        max_ok = max(max_ok, float(err[f].max()))
        if bad_val[f].any():
            failures.append((f, f"posterior max err {err[f].max():.3g}"))
        if z_diff[f].any():
            failures.append((f, "hard decision"))
        if syn_bad:
            failures.append((f, f"syndrome flag gpu={int(gpu_syn[f])} oracle={int(so1[f])}"))
        if it_bad:
            failures.append((f, f"iterations gpu={int(gpu_it[f])} oracle={int(it1[f])}"))
    if F and n_exempt > max_exempt_frac * F:
        failures.append((-1, f"exempt fraction {n_exempt}/{F} above {max_exempt_frac}"))
    return ParityReport(F, n_exempt, max_ok, max_ex, failures, int(ill.sum()))


@dataclass
class DecisionReport:
    frames: int
    exempt: np.ndarray          # bool [F]: frames whose decisions needed rule 4
    oracle: tuple               # (L, z, iters, syndrome_ok) of the oracle's run on R
    failures: list

    def __str__(self):
        return f"frames={self.frames} exempt={int(self.exempt.sum())} failures={len(self.failures)}"


def compare_decisions(O, code, R: np.ndarray, gpu_z: np.ndarray, gpu_syn: np.ndarray, gpu_it: np.ndarray,
                      max_iter: int, early_term: bool, seed: int = 12345,
                      max_exempt_frac: float = 0.02) -> DecisionReport:
    """Rules 1-5 for a decoder that returns no posteriors (the fused simulate
    path): hard decisions, syndrome flags and iteration counts only.  R is the
    ORACLE's channel output for the same (seed, frame) counters; the device
    draws its own, equal to within one fp32 ulp on <= 0.01% of the LLRs
    (reading c4), a difference the rule-1 probe measures the frame's
    sensitivity to."""
    R = np.ascontiguousarray(R, dtype=np.float32)
    F = R.shape[0]
    L1, z1, it1, so1 = oracle_decode_parallel(O, code, R, max_iter, early_term)
    rng = np.random.default_rng(seed)
    direction = np.where(rng.random(R.shape) < 0.5, np.float32(-np.inf), np.float32(np.inf))
    L2, z2, it2, so2 = oracle_decode_parallel(O, code, np.nextafter(R, direction).astype(np.float32),
                                              max_iter, early_term)
    ill = np.max(np.abs(np.clip(L1, -CLIP, CLIP) - np.clip(L2, -CLIP, CLIP)), axis=1) > PROBE_TOL
    z_diff = (gpu_z != z1) & (np.abs(L1) >= 1e-3)
    stable = (np.sign(L1) == np.sign(L2)) & (np.abs(L1) >= 1e-3) & (np.abs(L2) >= 1e-3)
    exempt = np.zeros(F, dtype=bool)
    failures = []
    for f in range(F):
        syn_bad = int(gpu_syn[f]) != int(so1[f])
        it_bad = int(gpu_it[f]) != int(it1[f])
        if not (z_diff[f].any() or syn_bad or it_bad):
            continue
        if not ill[f]:
            failures.append((f, f"decisions differ (well-conditioned): bits {int(z_diff[f].sum())} "
                                f"syn {syn_bad} iters {int(gpu_it[f])}/{int(it1[f])}"))
            continue
        exempt[f] = True
        if np.any(z_diff[f] & stable[f]):
            failures.append((f, "hard decision (ill-conditioned, stable bits)"))
        if syn_bad and int(so1[f]) == int(so2[f]):
            failures.append((f, "syndrome flag (ill-conditioned, oracle runs agree)"))
        if it_bad and int(it1[f]) == int(it2[f]):
            failures.append((f, "iterations (ill-conditioned, oracle runs agree)"))
    if F and exempt.sum() > max_exempt_frac * F:
        failures.append((-1, f"exempt fraction {int(exempt.sum())}/{F} above {max_exempt_frac}"))
    return DecisionReport(F, exempt, (L1, z1, it1, so1), failures)
