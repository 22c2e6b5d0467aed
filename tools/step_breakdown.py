#!/usr/bin/env python3
"""Where a small bench step's time goes: the step's graph (memset, encode,
decode, count) against graphs of each launch alone, every replay preceded by
the bench's untimed L2 flush, CUDA events on the replaying stream, median of
`--reps`.  Diagnostic only (not a bench line).

    python tools/step_breakdown.py --config T1-R3/4 --frames 1000
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ldpc_workloads as W  # noqa: E402
import bench as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="T1-R3/4")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    import torch
    import paper_2201_04265_b200 as L
    dev = torch.device("cuda", 0)
    wl = W.ALL[a.config]
    F = a.frames or wl.frames
    code = L.ldpc_code_bind_device(L.ldpc_make_G(L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)))
    work = B.RankWork(L, code, wl, 0, 0, F, F, dev, 0)
    s = torch.cuda.Stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(l2, dtype=torch.int32, device=dev)

    def enc(st):
        L.ldpc_encode(code, work.d_info, work.d_cw, F, stream=st)

    def dec(st):
        L.ldpc_decode(code, work.d_llr, F, work.d_bits, work.d_syn, work.d_it, None, work.d_ws, wl.max_iter,
                      wl.early_term, 0, stream=st)

    def cnt(st):
        L.ldpc_count_errors(code, work.d_info, work.d_bits, work.d_cw, work.d_syn, work.d_it, F, work.d_ctr,
                            stream=st)

    def step(st):
        B.memset_async(work.d_ctr, st)
        enc(st)
        dec(st)
        cnt(st)

    parts = {"step": step, "encode": enc, "decode": dec, "count": cnt,
             "memset": lambda st: B.memset_async(work.d_ctr, st)}
    with torch.cuda.stream(s):
        step(s)
    torch.cuda.synchronize()
    for name, fn in parts.items():
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn(s)
        torch.cuda.synchronize()
        ts = []
        with torch.cuda.stream(s):
            for r in range(a.reps + 3):
                flush.add_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                g.replay()
                e1.record(s)
                e1.synchronize()
                if r >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"{a.config} F={F} {name:7s} median {statistics.median(ts):8.1f} us  min {min(ts):8.1f} us",
              flush=True)


if __name__ == "__main__":
    main()
