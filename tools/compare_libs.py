#!/usr/bin/env python3
"""Decode fixed seeded batches with a given libldpc_b200.so and save the
outputs, or compare two saved runs bit for bit (A/B of a change that must not
alter results).

    python tools/compare_libs.py run  --lib path/to/lib.so --out a.npz
    python tools/compare_libs.py diff a.npz b.npz
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ldpc_workloads as W  # noqa: E402

# (config, frames, iterations, early termination, variant)
CASES = [("C4", 1024, 50, False, 0), ("C3-R1/4", 1000, 50, False, 0), ("C3-R1/2", 1000, 50, False, 0),
         ("C2", 2000, 50, True, 0), ("C1", 2000, 30, False, 0), ("C5", 32, 50, False, 7),
         ("C5", 8, 50, False, 5), ("C4", 2, 50, False, 7), ("C3-R3/4", 1000, 50, False, 0),
         ("T1-R3/4", 2000, 30, False, 0), ("T1-R1/2", 500, 30, False, 0)]


def run(lib_path, out):
    import paper_2201_04265_b200._lib as LL
    LL.LIB_PATH = os.path.abspath(lib_path)
    import torch
    import paper_2201_04265_b200 as L
    res = {}
    for i, (cfg, F, T, et, var) in enumerate(CASES):
        wl = W.ALL[cfg]
        code = L.ldpc_code_bind_device(L.ldpc_make_G(L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)))
        k, n = code.info.k, code.info.n
        info = torch.empty((F, L.words(k)), dtype=torch.int32, device="cuda")
        cw = torch.empty((F, L.words(n)), dtype=torch.int32, device="cuda")
        llr = torch.empty((F, n), dtype=torch.float32, device="cuda")
        L.ldpc_gen_info(wl.frame_seeds[0], 0, F, k, info)
        L.ldpc_encode(code, info, cw, F)
        L.ldpc_channel(code, wl.frame_seeds[0], 0, F, cw, wl.sigma(), llr)
        o = L.decode(code, llr, max_iter=T, early_term=et, posterior=True, variant=var)
        torch.cuda.synchronize()
        res[f"{i}_post"] = o.posterior.cpu().numpy()
        res[f"{i}_bits"] = o.bits.cpu().numpy()
        res[f"{i}_iters"] = o.iters.cpu().numpy()
        res[f"{i}_syn"] = o.syndrome_ok.cpu().numpy()
        print(cfg, F, T, et, var, "variant", L.ldpc_decode_variant(code, F, T, et, var), flush=True)
    np.savez(out, **res)


def diff(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for key in sorted(A.files):
        same = A[key].tobytes() == B[key].tobytes()
        i = int(key.split("_")[0])
        if not same:
            bad += 1
            extra = ""
            if key.endswith("post"):
                d = np.abs(A[key].astype(np.float64) - B[key])
                extra = f" max|d|={d.max():.3g} differing={np.count_nonzero(d)}"
            print("DIFF", CASES[i], key, extra)
    print("identical" if not bad else f"{bad} arrays differ")
    return bad


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--lib", required=True)
    r.add_argument("--out", required=True)
    d = sub.add_parser("diff")
    d.add_argument("a")
    d.add_argument("b")
    a = ap.parse_args()
    if a.cmd == "run":
        run(a.lib, a.out)
    else:
        sys.exit(1 if diff(a.a, a.b) else 0)
