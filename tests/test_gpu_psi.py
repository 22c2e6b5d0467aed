"""Exhaustive device pins of the throughput decoders' phi (SURVEY.md §8c,
"GPU-side numerics"): every band, exchange-cluster and lane-per-edge kernel
evaluates Eq. 5 through band_common.cuh's psi in log2 units,
psi(y) = log2(e) phi(y ln 2), phi(x) = -ln tanh(x/2) = log1p(2/expm1(x)).

Gate (§8c): relative error <= 2e-6, or absolute error <= 1e-6 where
phi < 1e-6 -- applied in phi units (phi = psi ln 2) against fp64.

Domains swept (every positive normal fp32 value in them):
  * the first psi of a row sees |L'_vc| <= the clamp 30 log2 e = 43.28;
  * the second psi sees exclusive sums of up to 11 first-psi values, each
    <= psi(2^-126) = 127.5, so up to 1403: the sweep runs to 2048;
  * each tier over the whole domain its warp vote admits it to.
"""
import math

import numpy as np
import pytest

from tests.gpu_util import lib, torch

pytestmark = pytest.mark.gpu

LOG2E = 1.0 / math.log(2.0)
CLAMP_B = float(np.float32(43.2808512))
SPLIT_B = float(np.float32(1.8033688))
EMAX_B = float(np.float32(40.86313714))
REL_GATE = 2e-6
ABS_GATE = 1e-6          # where phi < 1e-6


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    t = torch()
    if not t.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    lib()._lib.lib()


def psi64(y):
    """fp64 psi(y) = log2(e) phi(y ln 2), phi(x) = log1p(2 / expm1(x))."""
    t = torch()
    return t.log1p(2.0 / t.expm1(y.double() * math.log(2.0))) * LOG2E


def _bits(v: float) -> int:
    return int(np.float32(v).view(np.int32))


def _sweep(tier: int, lo: float, hi: float, lo_open: bool = False, hi_open: bool = False):
    """Run ldpc_debug_psi(tier) on every fp32 y in [lo, hi] (positive, normal);
    return (worst relative error where phi >= 1e-6, worst absolute error where
    phi < 1e-6, number of gate failures, first failing y)."""
    t = torch()
    L = lib()
    a = _bits(lo) + (1 if lo_open else 0)
    b = _bits(hi) - (1 if hi_open else 0)
    chunk = 1 << 25
    worst_rel, worst_abs, fails, first_bad = 0.0, 0.0, 0, None
    for start in range(a, b + 1, chunk):
        stop = min(start + chunk, b + 1)
        yi = t.arange(start, stop, dtype=t.int32, device="cuda")
        y = yi.view(t.float32)
        out = t.empty_like(y)
        L.ldpc_debug_psi(y, out, y.numel(), tier)
        ref = psi64(y) * math.log(2.0)             # phi units
        got = out.double() * math.log(2.0)
        err = (got - ref).abs()
        small = ref < 1e-6
        rel = t.where(small, t.zeros_like(err), err / ref)
        ok = (rel <= REL_GATE) | (small & (err <= ABS_GATE))
        worst_rel = max(worst_rel, float(rel.max()))
        if bool(small.any()):
            worst_abs = max(worst_abs, float(err[small].max()))
        nbad = int((~ok).sum())
        if nbad and first_bad is None:
            first_bad = float(y[~ok][0])
        fails += nbad
    return worst_rel, worst_abs, fails, first_bad


TINY = float(np.finfo(np.float32).tiny)

# (tier, name, lo, hi, lo_open, hi_open): every tier over its whole domain
SWEEPS = [
    (0, "psi (first psi: y <= clamp)", TINY, CLAMP_B, False, False),
    (0, "psi (second psi: sums up to 2048)", CLAMP_B, 2048.0, True, False),
    (1, "psi_small (y <= split)", TINY, SPLIT_B, False, False),
    (2, "psi_large (split < y <= 2048)", SPLIT_B, 2048.0, True, False),
    (3, "psi_deep_large (10 <= y <= 2048)", 10.0, 2048.0, False, False),
    (4, "psi_deep_small (y <= 2^-10)", TINY, 2.0 ** -10, False, False),
    (5, "psi_row votes, first psi (y <= 2048)", TINY, 2048.0, False, False),
    (6, "psi_row votes, second psi (y <= 2048)", TINY, 2048.0, False, False),
]


@pytest.mark.parametrize("tier,name,lo,hi,lo_open,hi_open", SWEEPS, ids=[s[1] for s in SWEEPS])
def test_psi_tier_exhaustive(tier, name, lo, hi, lo_open, hi_open):
    worst_rel, worst_abs, fails, first_bad = _sweep(tier, lo, hi, lo_open, hi_open)
    print(f"{name}: max rel err {worst_rel:.3g} (phi >= 1e-6), max abs err {worst_abs:.3g} (phi < 1e-6), "
          f"fails {fails}")
    assert fails == 0, (name, fails, first_bad, worst_rel, worst_abs)


def test_psi_special_values():
    """psi(0) = +inf (a zero message, reading Q9), psi(+inf) = 0; a subnormal
    y is flushed to zero by the approx instructions (.ftz) and gives +inf
    where the truth is >= 127.5: downstream that makes the row's other
    exclusive sums +inf, whose psi is 0 against a truth < h0 2^-127 (< 1e-38):
    accepted."""
    t = torch()
    L = lib()
    ys = t.tensor([0.0, float("inf"), 1e-45, 1e-39], device="cuda")
    for tier in (0, 1, 5, 6):
        out = t.empty_like(ys)
        L.ldpc_debug_psi(ys, out, ys.numel(), tier)
        o = out.cpu().tolist()
        assert o[0] == math.inf and o[2] == math.inf and o[3] == math.inf, (tier, o)
        if tier in (0, 5, 6):
            assert o[1] == 0.0, (tier, o)
    with pytest.raises(L.LdpcError):
        L.ldpc_debug_psi(ys, ys, 4, 7)


def test_generic_phi_exhaustive_sweep():
    """The generic CSR kernels' phi (spa_decode.cu, variants 1/2; natural-log
    domain) over every positive normal fp32 x <= 60 against fp64
    log1p(2/expm1(x)), at the §8c gate (relative <= 2e-6, or absolute <= 1e-6
    where phi < 1e-6)."""
    t = torch()
    L = lib()
    lo = _bits(TINY)
    hi = _bits(60.0)
    chunk = 1 << 25
    fails, worst = 0, 0.0
    for start in range(lo, hi + 1, chunk):
        stop = min(start + chunk, hi + 1)
        xi = t.arange(start, stop, dtype=t.int32, device="cuda")
        x = xi.view(t.float32)
        y = t.empty_like(x)
        L.ldpc_debug_phi(x, y, x.numel())
        ref = t.log1p(2.0 / t.expm1(x.double()))
        err = (y.double() - ref).abs()
        small = ref < 1e-6
        rel = t.where(small, t.zeros_like(err), err / ref)
        worst = max(worst, float(rel.max()))
        fails += int((~((rel <= REL_GATE) | (small & (err <= ABS_GATE)))).sum())
    print(f"generic phi: max rel err {worst:.3g} where phi >= 1e-6; gate failures {fails}")
    assert fails == 0
    xs = t.tensor([0.0, float("inf"), 1e-45], device="cuda")
    ys = t.empty_like(xs)
    L.ldpc_debug_phi(xs, ys, 3)
    assert ys[0].item() == math.inf and ys[1].item() == 0.0 and ys[2].item() > 87


# ---------------------------------------------------------------- check rows
def check_row64(x: np.ndarray) -> np.ndarray:
    """Eq. 5 in log2 units, fp64, written out (readings Q2/Q3/Q7): for each
    edge j, E'_j = (-1)^D prod_{k != j} sgn(x_k) min(psi(sum_{k != j}
    psi(min(|x_k|, clamp))), E_MAX log2 e)."""
    t = torch()
    X = t.from_numpy(x).double().cuda()
    R, D = X.shape
    ax = X.abs().clamp(max=CLAMP_B)
    f = psi64(ax)
    E = t.empty_like(X)
    neg = t.signbit(X)
    for j in range(D):
        others = [k for k in range(D) if k != j]
        s = f[:, others].sum(dim=1)
        mag = psi64(s).clamp(max=EMAX_B)
        nneg = neg[:, others].sum(dim=1) + D
        E[:, j] = t.where(nneg % 2 == 1, -mag, mag)
    return E.cpu().numpy()


def _rows(rng, D: int, R: int) -> dict:
    """Rows of D fp32 inputs in every regime the kernels meet."""
    sgn = lambda shape: np.where(rng.random(shape) < 0.5, -1.0, 1.0)
    out = {}
    # channel-like messages, several scales (log2 units)
    for sc in (0.3, 3.0, 15.0):
        out[f"gauss{sc}"] = rng.normal(0.0, sc, (R, D))
    # log-uniform magnitudes over the whole range, random signs
    out["loguniform"] = sgn((R, D)) * np.exp2(rng.uniform(-30, 7, (R, D)))
    # converged rows: every input at or above the saturation / clamp tiers
    out["saturated"] = sgn((R, D)) * rng.uniform(43.0, 80.0, (R, D))
    out["clamped"] = sgn((R, D)) * rng.uniform(CLAMP_B, 90.0, (R, D))
    # deep tiers: all inputs large (>= 10) or all tiny (<= 2^-10)
    out["deep_large"] = sgn((R, D)) * rng.uniform(10.0, 43.0, (R, D))
    out["deep_small"] = sgn((R, D)) * np.exp2(rng.uniform(-40, -10, (R, D)))
    # one unreliable input among confident ones (the exclusive sums straddle)
    m = sgn((R, D)) * rng.uniform(10.0, 43.0, (R, D))
    m[np.arange(R), rng.integers(0, D, R)] = rng.normal(0, 0.5, R)
    out["one_weak"] = m
    return {k: v.astype(np.float32) for k, v in out.items()}


@pytest.mark.parametrize("D", [2, 3, 4, 6, 12])
@pytest.mark.parametrize("vote", [True, False])
def test_check_row_against_fp64(D, vote):
    """check_row<D, VOTE> (the decoders' Eq. 5 update, every tier) against the
    fp64 formula on rows in every regime.  Bound derived from the arithmetic:
    each psi is within 2e-6 relative (sweeps above) and the exclusive sums add
    <= D 2^-24 relative, so the relative error of a sum is <= 3e-6; the
    second psi turns that into <= 3e-6 / ln 2 = 4.3e-6 absolute where psi is
    small-regime and <= s ln2 3e-6 relative (s <= 43: 9e-5) where it is
    large-regime -- plus 2e-6 relative of its own.  Gate: |dE| <= 1e-5 or
    <= 1e-4 |E| (log2 units)."""
    t = torch()
    L = lib()
    rng = np.random.default_rng(1000 + D)
    for name, x in _rows(rng, D, 20000).items():
        dx = t.from_numpy(x).cuda()
        de = t.empty_like(dx)
        L.ldpc_debug_check_row(dx, de, x.shape[0], D, vote)
        got = de.cpu().numpy().astype(np.float64)
        want = check_row64(x)
        err = np.abs(got - want)
        bad = (err > 1e-5) & (err > 1e-4 * np.abs(want))
        print(f"D={D} vote={vote} {name}: max |dE| {err.max():.3g}, bad {int(bad.sum())}")
        assert not bad.any(), (name, x[bad.any(axis=1)][:3], got[bad.any(axis=1)][:3], want[bad.any(axis=1)][:3])
        assert np.all(np.signbit(got) == np.signbit(want)), name


@pytest.mark.parametrize("D", [2, 3, 4, 6])
def test_saturation_tier_bit_exact(D):
    """Saturation tier (D <= 6): rows whose every |x| is at or above the
    saturation bound return +-E_MAX bit for bit -- with the votes (the
    shortcut) and without them (the full two-regime evaluation), so the
    shortcut changes no output."""
    t = torch()
    L = lib()
    rng = np.random.default_rng(7 + D)
    x = (np.where(rng.random((5000, D)) < 0.5, -1.0, 1.0) * rng.uniform(43.21, 100.0, (5000, D))).astype(np.float32)
    outs = []
    for vote in (True, False):
        dx = t.from_numpy(x).cuda()
        de = t.empty_like(dx)
        L.ldpc_debug_check_row(dx, de, x.shape[0], D, vote)
        outs.append(de.cpu().numpy())
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.all(np.abs(outs[0]) == np.float32(EMAX_B))


def test_check_row_probe_rejects_degree():
    t = torch()
    L = lib()
    x = t.zeros(10, device="cuda")
    with pytest.raises(L.LdpcError):
        L.ldpc_debug_check_row(x, x, 1, 5, True)
