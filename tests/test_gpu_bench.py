"""bench.py's multi-GPU work split on the device: the per-rank
work of a strong-scaling step (Eq. 9 shards; C5's chunked
launches) gives the same summed counters for N = 1 and for the two ranks of
N = 2.  The ranks' shares run one after the other on the one GPU: they share
nothing (no data-path collective), so this is each rank's own work, not a
stand-in for ranks that wait on one another."""
import pytest

import ldpc_workloads as W
from tests.gpu_util import lib, torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    t = torch()
    if not t.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    lib()._lib.lib()


def _counters(bench, L, code, wl, total, rank, world, chunk, budget):
    t = torch()
    f0, count = bench.rank_share(total, rank, world, "strong")
    work = bench.RankWork(L, code, wl, 0, f0, count, chunk, t.device("cuda"), 0, budget_bytes=budget)
    s = t.cuda.current_stream()
    work.device_work(s)
    t.cuda.synchronize()
    return work, work.d_ctr.cpu().tolist()


@pytest.mark.parametrize("cfg,total,chunk", [("C5", 33000, 16384), ("C4", 5001, 2048)])
def test_strong_split_matches_single_rank(cfg, total, chunk):
    import bench
    L = lib()
    wl = W.ALL[cfg]
    code = L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)
    L.ldpc_make_G_device(code)
    L.ldpc_code_bind_device(code)
    one, c1 = _counters(bench, L, code, wl, total, 0, 1, chunk, 40e9)        # resident, one launch
    assert one.resident and c1[5] == total
    parts = []
    for r in range(2):
        w, c = _counters(bench, L, code, wl, total, r, 2, chunk, 0)           # chunked launches
        assert not w.resident and len(w.spans) == -(-w.count // chunk)
        parts.append(c)
    summed = [a + b for a, b in zip(*parts)]
    assert summed == c1, (summed, c1)
    assert c1[4] == 50 * total                                                  # fixed iterations


def test_sweep_one_launch_counters_equal_the_points():
    """C2's five Eb/N0 points decoded as one batch in one ldpc_decode call
    (bench.py `sweep_one_launch`) give, per point slice, exactly the counters
    of the points decoded one launch each: frames are independent,
    and the iteration counts (early termination) are part of the counters."""
    import argparse

    import bench
    L = lib()
    t = torch()
    wl = W.ALL["C2"]
    code = L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)
    L.ldpc_make_G_device(code)
    L.ldpc_code_bind_device(code)
    args = argparse.Namespace(frames=1500, scaling="strong", chunk=16384, variant=0, eager=False, warmup=1, steps=2,
                              ebn0=None)
    dev = t.device("cuda", t.cuda.current_device())
    props = t.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    points = list(range(len(wl.ebn0_db)))
    results = [bench.measure_point(args, L, code, wl, p, dev, 0, 1, False, sms, props) for p in points]
    one = bench.measure_sweep_one_launch(args, L, code, wl, points, results, dev, 0, 1, False, sms, props)
    assert one["frames_per_step"] == 1500 * len(points)
    assert one["counters_match_points"], one
    its = [r["counters"][4] / r["counters"][5] for r in results]
    assert its == sorted(its, reverse=True)          # ascending Eb/N0 = longest-running frames first
    assert one["value"] > 0 and one["decode_ms_per_step"] > 0
