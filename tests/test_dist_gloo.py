"""Multi-process (world_size 2, gloo, CPU) tests of the sharding, chunking
and reduction logic the multi-GPU bench uses -- bench.py's own functions
(rank_share, chunk_spans, reduce_step): Eq. 9 shards cover the step's frames
exactly once, chunks cover each shard, and the all-reduced error counters of
the shards equal the single-process counters (results
independent of world size); the reduced time is the max over ranks.  The
per-chunk decode here is the oracle (CPU): the GPU kernels are covered by the
-m gpu tests; this file checks the host-side distribution only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, scaling, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import ldpc_workloads as W
        from oracle import oracle as O
        w = W.C1
        frame0, count = bench.rank_share(total, rank, world, scaling)
        code = O.make_H(w.n, w.wc, w.wr, W.CODE_SEED).make_G()
        ctr = torch.zeros(6, dtype=torch.int64)
        spans = bench.chunk_spans(frame0, count, 7)          # ragged chunks, as C5's 16,384-frame launches
        for f0, m in spans:
            info = O.gen_info(w.frame_seeds[0], f0, m, code.k)
            c = O.encode(code, info)
            R = O.channel(w.frame_seeds[0], f0, c, 1.0)
            _, z, it, so = O.spa_decode(code, R, w.max_iter)
            ctr += torch.from_numpy(O.count_errors(code, info, z, c, so, it))
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        bench.reduce_step(ctr, t)
        shards = [None] * world
        dist.all_gather_object(shards, (frame0, count, spans))
        if rank == 0:
            q.put((ctr.numpy().tolist(), shards, float(t)))
    finally:
        dist.destroy_process_group()


def _single(oracle, frame0, total):
    import ldpc_workloads as W
    w = W.C1
    code = oracle.make_H(w.n, w.wc, w.wr, W.CODE_SEED).make_G()
    info = oracle.gen_info(w.frame_seeds[0], frame0, total, code.k)
    c = oracle.encode(code, info)
    R = oracle.channel(w.frame_seeds[0], frame0, c, 1.0)
    _, z, it, so = oracle.spa_decode(code, R, w.max_iter)
    return list(oracle.count_errors(code, info, z, c, so, it))


def _run(world, total, scaling):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, scaling, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return q.get()


@pytest.mark.parametrize("world", [2])
def test_strong_split_counters_equal_single_process(oracle, world):
    """Strong scaling (bench default): the step's 37 frames split 19 + 18 by
    Eq. 9, each shard in ragged 7-frame chunks; the reduced counters equal one
    process decoding all 37."""
    total = 37
    ctr, shards, tmax = _run(world, total, "strong")
    assert tmax == float(world)
    covered = sorted((f0, c) for f0, c, _ in shards)
    assert covered[0][0] == 0 and sum(c for _, c in covered) == total
    for (a0, ac), (b0, _) in zip(covered, covered[1:]):
        assert a0 + ac == b0
    assert max(c for _, c in covered) - min(c for _, c in covered) <= 1
    for f0, c, spans in shards:                   # chunks tile the shard in order
        assert spans[0][0] == f0 and sum(m for _, m in spans) == c
        assert all(a + m == b for (a, m), (b, _) in zip(spans, spans[1:]))
    want = _single(oracle, 0, total)
    assert ctr == want and want[5] == total


def test_weak_split_counters(oracle):
    """Weak scaling: each rank decodes its own 9 frames at global indices
    r*9 .. r*9+8; the reduced counters equal one process decoding 18."""
    ctr, shards, tmax = _run(2, 9, "weak")
    assert sorted((f0, c) for f0, c, _ in shards) == [(0, 9), (9, 9)]
    assert ctr == _single(oracle, 0, 18)


def test_shard_helpers():
    from paper_2201_04265_b200 import dist as D
    assert D.shard(10, 0, 4) == (0, 3) and D.shard(10, 3, 4) == (8, 2)
    assert D.weak_shard(200000, 3) == (600000, 200000)
    assert sum(D.shard(1000000, r, 8)[1] for r in range(8)) == 1000000
    import bench
    assert bench.chunk_spans(5, 40000, 16384) == [(5, 16384), (16389, 16384), (32773, 7232)]
    assert bench.chunk_spans(0, 0, 16384) == []
    # C5 at N = 8: 125,000 frames per rank, 8 chunks (7 x 16384 + 10312)
    f0, c = bench.rank_share(1000000, 7, 8, "strong")
    assert (f0, c) == (875000, 125000) and len(bench.chunk_spans(f0, c, 16384)) == 8


def test_sweep_fit_recovers_line():
    """bench.sweep_fit (the C2 sweep's fixed + per-iteration decode-time fit)
    recovers a known line t = a + b x iterations exactly."""
    import bench
    import ldpc_workloads as W
    a, b = 0.14, 0.046
    iters = [42.1, 23.2, 11.0, 6.9, 5.2]
    frames = 10000
    res = [{"counters": [0, 0, 0, 0, int(round(x * frames)), frames], "dec_ms": (a + b * (round(x * frames) / frames)) * 3,
            "roofline": {"peak": 1163.28, "frac": 0.5}} for x in iters]
    fit = bench.sweep_fit(W.C2, res, 3)
    assert abs(fit["decode_ms_per_iteration_of_all_frames"] - b) < 1e-9
    assert abs(fit["decode_ms_fixed_per_step"] - a) < 1e-9
    assert abs(fit["fixed_cost_in_iterations_per_frame"] - a / b) < 1e-6
    assert abs(fit["per_iteration_gedge_updates_per_s"] - frames * W.C2.edges / (b / 1e3) / 1e9) < 1e-6
