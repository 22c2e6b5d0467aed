#!/usr/bin/env python3
"""Run ldpc_decode on a config's frames (device-generated) `--reps` times; a
driver for ncu captures of one decode launch (not a benchmark).

    python tools/decode_once.py --config C5 --frames 64 --variant 7 --reps 2
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ldpc_workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--iters", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_2201_04265_b200 as L
    wl = W.ALL[a.config]
    code = L.ldpc_code_bind_device(L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED))
    n = code.info.n
    F = a.frames
    llr = (torch.randn((F, n), device="cuda") * 2.0 + 2.0).contiguous()
    it = a.iters or wl.max_iter
    print("variant", L.ldpc_decode_variant(code, F, it, wl.early_term, a.variant))
    for r in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = L.decode(code, llr, max_iter=it, early_term=wl.early_term, variant=a.variant)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        eu = F * wl.wc * n * it
        print(f"rep {r}: {dt*1e3:.2f} ms  {eu/dt/1e9:.1f} G edge-updates/s")


if __name__ == "__main__":
    main()
