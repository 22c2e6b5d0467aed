"""Multi-process (world_size 2, gloo, CPU) tests of the sharding and
reduction logic the multi-GPU bench uses: Eq. 9 shards cover the batch
exactly once, and the all-reduced error counters of the shards equal the
single-process counters (results independent of world size).
The per-shard decode here is the oracle (CPU): the GPU kernels are covered by
the -m gpu tests; this file checks the host-side distribution only."""
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


def _worker(rank, world, port, total, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ldpc_workloads as W
        from oracle import oracle as O
        from paper_2201_04265_b200 import dist as D
        w = W.C1
        frame0, count = D.shard(total, rank, world)
        code = O.make_H(w.n, w.wc, w.wr, W.CODE_SEED).make_G()
        info = O.gen_info(w.frame_seeds[0], frame0, count, code.k)
        c = O.encode(code, info)
        R = O.channel(w.frame_seeds[0], frame0, c, 1.0)
        _, z, it, so = O.spa_decode(code, R, w.max_iter)
        ctr = torch.from_numpy(O.count_errors(code, info, z, c, so, it))
        D.all_reduce_counters(ctr)
        spans = [None] * world
        dist.all_gather_object(spans, (frame0, count))
        t = torch.tensor([float(rank + 1)])
        D.max_over_ranks(t)
        if rank == 0:
            q.put((ctr.numpy().tolist(), spans, float(t)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_counters_equal_single_process(oracle, world):
    import ldpc_workloads as W
    total = 37                      # ragged: 37 = 19 + 18
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ctr, spans, tmax = q.get()
    assert tmax == float(world)
    covered = sorted(spans)
    assert covered[0][0] == 0 and sum(c for _, c in covered) == total
    for (a0, ac), (b0, _) in zip(covered, covered[1:]):
        assert a0 + ac == b0
    assert max(c for _, c in covered) - min(c for _, c in covered) <= 1
    # single process, same frames
    w = W.C1
    code = oracle.make_H(w.n, w.wc, w.wr, W.CODE_SEED).make_G()
    info = oracle.gen_info(w.frame_seeds[0], 0, total, code.k)
    c = oracle.encode(code, info)
    R = oracle.channel(w.frame_seeds[0], 0, c, 1.0)
    _, z, it, so = oracle.spa_decode(code, R, w.max_iter)
    want = oracle.count_errors(code, info, z, c, so, it)
    assert ctr == list(want)
    assert want[5] == total


def test_shard_helpers():
    from paper_2201_04265_b200 import dist as D
    assert D.shard(10, 0, 4) == (0, 3) and D.shard(10, 3, 4) == (8, 2)
    assert D.weak_shard(200000, 3) == (600000, 200000)
    assert sum(D.shard(1000000, r, 8)[1] for r in range(8)) == 1000000
