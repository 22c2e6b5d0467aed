#!/usr/bin/env python3
"""Host (multi-threaded) vs device make_G wall time, and a bit-exact check of
the two results, for the configs' largest codes."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    import torch
    import paper_2201_04265_b200 as L
    out = []
    for n in [int(x) for x in (sys.argv[1:] or ["16200", "64800"])]:
        t0 = time.perf_counter()
        host = L.ldpc_make_G(L.ldpc_make_H(n, 3, 6, 1))
        th = time.perf_counter() - t0
        L.ldpc_make_G_device(L.ldpc_make_H(96, 3, 6, 1))       # warm the context / module
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev = L.ldpc_make_G_device(L.ldpc_make_H(n, 3, 6, 1))
        td = time.perf_counter() - t0
        same = (np.array_equal(L.ldpc_code_copy_perm(dev), L.ldpc_code_copy_perm(host))
                and np.array_equal(L.ldpc_code_copy_P(dev), L.ldpc_code_copy_P(host)))
        out.append({"n": n, "k": dev.info.k, "host_s": th, "host_threads": os.cpu_count(), "device_s": td,
                    "speedup": th / td, "bit_exact": bool(same)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
