"""Seeded synthetic workloads -- shared by tests, bench
and smoke.  Holds none of the method's arithmetic: only the configuration
table of BASELINE.json's configs and the Eb/N0 -> sigma parameterisation of
the channel (reading Q15).  Both the oracle and the CUDA path implement the
same counter-based generators (SplitMix64 for H, Philox4x32-10 for frames)
from these seeds.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

CODE_SEED = 1


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    wc: int
    wr: int
    frames: int
    max_iter: int
    early_term: bool
    ebn0_db: tuple
    frame_seeds: tuple
    note: str = ""
    n_requested: int = 0

    @property
    def design_rate(self) -> float:
        return 1.0 - self.wc / self.wr

    def sigma(self, i: int = 0) -> float:
        """sigma^2 = 1 / (2 R 10^(Eb/N0 / 10)), R = design rate (reading Q15)."""
        ebn0 = 10.0 ** (self.ebn0_db[i] / 10.0)
        return math.sqrt(1.0 / (2.0 * self.design_rate * ebn0))

    @property
    def edges(self) -> int:
        return self.n * self.wc


# BASELINE.json configs[0..4]; C3's n = 4000 is not divisible by 6 or 12, so
# the nearest length divisible by 4, 6 and 12 is used (reading Q16).
C1 = Workload("C1", 96, 3, 6, 1000, 20, False, (2.0,), (101,), "batch + stream(1)")
C2 = Workload("C2", 1008, 3, 6, 10000, 50, True, (1.0, 1.5, 2.0, 2.5, 3.0), (201, 202, 203, 204, 205),
              "early termination, Eb/N0 sweep")
C3_R14 = Workload("C3-R1/4", 3996, 3, 4, 100000, 50, False, (2.5,), (301,), "rate 1/4", 4000)
C3_R12 = Workload("C3-R1/2", 3996, 3, 6, 100000, 50, False, (2.5,), (302,), "rate 1/2", 4000)
C3_R34 = Workload("C3-R3/4", 3996, 3, 12, 100000, 50, False, (2.5,), (303,), "rate 3/4", 4000)
C4 = Workload("C4", 16200, 3, 6, 200000, 50, False, (1.5,), (401,), "with bit-packed encode of all frames")
C5 = Workload("C5", 64800, 3, 6, 1000000, 50, False, (1.2,), (501,), "sharded over 1/2/4/8 GPUs")

ALL = {w.name: w for w in (C1, C2, C3_R14, C3_R12, C3_R34, C4, C5)}

# The paper's own experiment, Table I: n = 1032, 12 ones per row,
# 9/6/3 per column (design rates 1/4, 1/2, 3/4), 10 decoding iterations, 1000
# vectors.  The paper states no SNR; Eb/N0 = 2.5 dB (as C3) is this build's
# choice.
T1_R14 = Workload("T1-R1/4", 1032, 9, 12, 1000, 10, False, (2.5,), (601,), "Table I, wc = 9")
T1_R12 = Workload("T1-R1/2", 1032, 6, 12, 1000, 10, False, (2.5,), (602,), "Table I, wc = 6")
T1_R34 = Workload("T1-R3/4", 1032, 3, 12, 1000, 10, False, (2.5,), (603,), "Table I, wc = 3")
TABLE_I = {w.name: w for w in (T1_R14, T1_R12, T1_R34)}
ALL.update(TABLE_I)
