#!/usr/bin/env python3
"""Benchmark of the hot path: batched LDPC encode + Sum-Product decode + error
count (+ NCCL all-reduce of the counters when N > 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4] [--frames F]

One step = one pass of every §8(a) row over the step's synthetic frames:
ldpc_encode (e1) -> ldpc_decode (a1-a8) -> ldpc_count_errors (a9) ->
all_reduce(int64[6]) (a9, N > 1).  Default workload: BASELINE.json configs[3]
(C4: n = 16200 (3,6), 200,000 frames, 50 fixed iterations, Eb/N0 1.5 dB, with
the bit-packed encode of all frames) -- the largest config whose LLRs fit one
GPU, resident in HBM.  The step's frames are split across ranks by Eq. 9
(strong scaling, the default: the config's frame count is fixed as
N grows); `--scaling weak` gives every rank a batch of its own.  Frame indices
are global, so results do not depend on N.  `--config C5` runs the 10^6
frames of configs[4] in 16,384-frame chunks per rank (their LLRs, 259 GB, do
not fit), each chunk encode -> channel -> decode -> count.  `--config C2`
sweeps its five Eb/N0 points.

Rank 0 prints one JSON line.  `--impl reference` times the CPU oracle on the
host cores (the reference arm for this paper-only tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ldpc_workloads as W  # noqa: E402

# SFU roofline: 4 MUFU ops per edge-update (2 phi per
# edge per iteration, ex2 + lg2 each), 16 MUFU/clk/SM, 148 SMs.
MUFU_PER_CLK_PER_SM = 16
MUFU_PER_EDGE_UPDATE = 4
E2E_PINNED_BYTES = 16e9          # pinned host memory for the e2e arm, over all ranks
KERNEL_NAMES = {1: "spa_decode_kernel (generic, on-chip)", 2: "spa_decode_kernel (generic, global state)",
                3: "band_kernel (check-major E)", 4: "band_kernel (variable-major E)",
                5: "band_cluster_kernel (L2 gathers)", 6: "band_kernel (variable-major E, 16-bit offsets)",
                7: "xband_kernel (exchange cluster, bulk DSMEM segments; C5 batches: two-frame 16-CTA clusters "
                   "plus gband2_kernel groups on the SMs the clusters leave idle)",
                8: "edge_kernel (lane per edge, small batches)",
                9: "gband2_kernel (16-CTA groups, segments through L2 staging)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4", choices=sorted(W.ALL))
    ap.add_argument("--frames", type=int, default=0,
                    help="override the step's frames (strong: total over ranks; weak: per rank)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the step's frames are split across ranks by Eq. 9 (default); "
                         "weak: every rank decodes a batch of its own")
    ap.add_argument("--chunk", type=int, default=16384,
                    help="frames per launch when a rank's LLRs exceed the 40 GB HBM budget (C5)")
    ap.add_argument("--e2e-frames", type=int, default=0, help="cap on e2e frames per step (0 = the batch)")
    ap.add_argument("--e2e-chunk", type=int, default=8192, help="frames per H2D/compute/D2H pipeline chunk (e2e)")
    ap.add_argument("--early-term", type=int, choices=[0, 1], default=None,
                    help="override the config's early termination (measurement variant)")
    ap.add_argument("--ebn0", type=float, default=None, help="override the config's Eb/N0 in dB (measurement variant)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end arm (profiling runs)")
    ap.add_argument("--no-sweep-one-launch", action="store_true",
                    help="skip the sweep's one-launch measurement (configs with several Eb/N0 points)")
    ap.add_argument("--sweep-order", choices=["asc", "desc"], default="asc",
                    help="one-launch sweep: points by ascending Eb/N0 (longest-running frames first, default) or descending (A/B)")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--eager", action="store_true", help="launch the step's kernels eagerly instead of replaying a CUDA graph")
    ap.add_argument("--mode", choices=["batch", "stream", "simulate"], default="batch",
                    help="stream = frames decoded one per ldpc_decode call, serially (the paper's stream mode); "
                         "simulate = BER-simulation pipeline, fused (ldpc_decode_simulate) vs unfused")
    return ap.parse_args()


def run_stream(args):
    """Stream mode (batch 1): one frame per ldpc_decode call, issued
    serially on one stream; the serial calls are captured once in a CUDA graph
    and replayed, so the number is per-frame device latency, not launch cost."""
    import torch

    import paper_2201_04265_b200 as L
    torch.cuda.set_device(0)
    wl = workload(args)
    code = L.ldpc_code_bind_device(L.ldpc_make_G(L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)))
    k, n = code.info.k, code.info.n
    G = 64
    info = torch.empty((G, L.words(k)), dtype=torch.int32, device="cuda")
    cw = torch.empty((G, L.words(n)), dtype=torch.int32, device="cuda")
    llr = torch.empty((G, n), dtype=torch.float32, device="cuda")
    L.ldpc_gen_info(wl.frame_seeds[0], 0, G, k, info)
    L.ldpc_encode(code, info, cw, G)
    L.ldpc_channel(code, wl.frame_seeds[0], 0, G, cw, wl.sigma(), llr)
    bits = torch.empty((G, L.words(n)), dtype=torch.int32, device="cuda")
    syn = torch.empty(G, dtype=torch.uint8, device="cuda")
    it = torch.empty(G, dtype=torch.int32, device="cuda")
    wsb = max(L.ldpc_decode_workspace_bytes(code, 1, wl.max_iter, wl.early_term), 256)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()

    def serial():
        for f in range(G):
            L.ldpc_decode(code, llr[f:f + 1], 1, bits[f:f + 1], syn[f:f + 1], it[f:f + 1], None, ws,
                          wl.max_iter, wl.early_term, stream=s)

    with torch.cuda.stream(s):
        serial()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        serial()
    with torch.cuda.stream(s):              # graph replays on the current stream
        it.zero_()                          # ordered before the replays on the same stream
        for _ in range(args.warmup):
            g.replay()
    torch.cuda.synchronize()
    assert int(it.min()) >= 1, "graph replay did not decode"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(args.steps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (args.steps * G)
    iters = float(it.double().mean())
    print(json.dumps({"mode": "stream", "metric": "stream-mode decode latency per frame", "value": ms * 1e3,
                      "unit": "us", "frames_per_s": 1e3 / ms, "info_gbit_s": k / (ms * 1e-3) / 1e9,
                      "edge_updates_per_s": wl.edges * iters / (ms * 1e-3), "mean_iterations": iters,
                      "config": workload_config(wl, 1, 1), "frames_timed": args.steps * G,
                      "note": "one CTA decodes the frame; serial calls replayed from a CUDA graph"}), flush=True)
    return 0


def run_simulate(args):
    """BER-simulation pipeline on fresh frames every step:
    gen_info -> encode -> [channel -> decode -> count] (unfused, 4 n bytes of
    LLRs per frame through HBM) vs gen_info -> encode -> ldpc_decode_simulate
    (fused: channel draw in the decode prologue, counters in its epilogue).
    Both arms decode the same frames; their counters must agree."""
    import torch

    import paper_2201_04265_b200 as L
    torch.cuda.set_device(0)
    wl = workload(args)
    F = args.frames or min(wl.frames, 32768)
    code = L.ldpc_code_bind_device(L.ldpc_make_G(L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)))
    k, n = code.info.k, code.info.n
    info = torch.empty((F, L.words(k)), dtype=torch.int32, device="cuda")
    cw = torch.empty((F, L.words(n)), dtype=torch.int32, device="cuda")
    llr = torch.empty((F, n), dtype=torch.float32, device="cuda")
    bits = torch.empty((F, L.words(n)), dtype=torch.int32, device="cuda")
    syn = torch.empty(F, dtype=torch.uint8, device="cuda")
    its = torch.empty(F, dtype=torch.int32, device="cuda")
    ctr_u = torch.zeros(6, dtype=torch.int64, device="cuda")
    ctr_f = torch.zeros(6, dtype=torch.int64, device="cuda")
    tmp = torch.zeros(6, dtype=torch.int64, device="cuda")
    wsb = max(L.ldpc_decode_workspace_bytes(code, F, wl.max_iter, wl.early_term, 6 if wl.n == 16200 else 0), 256)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    seed, sigma = wl.frame_seeds[0], wl.sigma()
    band = 6 if wl.n == 16200 else 0      # both arms on the band kernel (the fused path's decoder)

    def unfused(frame0):
        L.ldpc_gen_info(seed, frame0, F, k, info)
        L.ldpc_encode(code, info, cw, F)
        L.ldpc_channel(code, seed, frame0, F, cw, sigma, llr)
        L.ldpc_decode(code, llr, F, bits, syn, its, None, ws, wl.max_iter, wl.early_term, band)
        tmp.zero_()
        L.ldpc_count_errors(code, info, bits, cw, syn, its, F, tmp)
        ctr_u.add_(tmp)

    def fused(frame0):
        L.ldpc_gen_info(seed, frame0, F, k, info)
        L.ldpc_encode(code, info, cw, F)
        L.ldpc_decode_simulate(code, seed, frame0, F, sigma, info, cw, bits, syn, its, ctr_f, ws,
                               wl.max_iter, wl.early_term, band)

    res = {}
    for name, fn in (("unfused", unfused), ("fused", fused)):
        for w in range(args.warmup):
            fn(10**9 + w * F)
        torch.cuda.synchronize()
        (ctr_u if name == "unfused" else ctr_f).zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            e0.record()
            for st in range(args.steps):
                fn(st * F)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        res[name] = {"ms_per_step": ms, "info_gbit_s": F * k / (ms * 1e-3) / 1e9, "clocks": clk.summary()}
    cu, cf = ctr_u.tolist(), ctr_f.tolist()
    assert cu == cf, (cu, cf)
    print(json.dumps({"mode": "simulate", "metric": "BER-simulation throughput (info Gbit/s)",
                      "value": res["fused"]["info_gbit_s"], "unit": "Gbit/s",
                      "unfused_value": res["unfused"]["info_gbit_s"], "fused": res["fused"], "unfused": res["unfused"],
                      "llr_bytes_saved_per_step": 2 * F * n * 4, "counters": cf,
                      "ber_info": cf[0] / max(cf[5] * k, 1), "fer": cf[2] / max(cf[5], 1),
                      "config": workload_config(wl, F, 1), "steps": args.steps, "warmup": args.warmup,
                      "note": "each step: gen_info + encode + (channel + decode + count | fused simulate) on new frames; "
                              "counters of the two arms identical"}), flush=True)
    return 0


def workload(args):
    """BASELINE.json workload named by --config, with the --early-term /
    --ebn0 overrides (measurement variants; the config's own values by default)."""
    import dataclasses
    wl = W.ALL[args.config]
    if args.early_term is not None:
        wl = dataclasses.replace(wl, early_term=bool(args.early_term))
    if args.ebn0 is not None:
        wl = dataclasses.replace(wl, ebn0_db=(float(args.ebn0),))
    return wl


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- reference arm
def cpu_oracle_run(wl, frames_per_thread: int, threads: int):
    """Time the oracle (as it stands) decoding a bounded sample of the workload
    on `threads` host threads.  Returns (seconds, frames, k)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    code = O.make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)
    code.make_G() if wl.n <= 20000 else None
    k = code.k if code.k is not None else wl.n - code.m + (wl.wc - 1)
    F = frames_per_thread * threads
    if code.k is not None:
        info = O.gen_info(wl.frame_seeds[0], 0, F, code.k)
        c = O.encode(code, info)
    else:
        c = np.zeros((F, wl.n), np.uint8)
    R = O.channel(wl.frame_seeds[0], 0, c, wl.sigma())
    chunks = np.array_split(np.arange(F), threads)

    def run(idx):
        if len(idx):
            O.spa_decode(code, R[idx], wl.max_iter, wl.early_term)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, chunks))
    return time.perf_counter() - t0, F, k


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args)
    threads = max(1, min(os.cpu_count() or 1, 128))
    per_thread = 1
    # warm-up / timed steps, each a bounded sample (one frame per host thread)
    for _ in range(args.warmup):
        cpu_oracle_run(wl, per_thread, threads)
    times = []
    for _ in range(args.steps):
        dt, F, k = cpu_oracle_run(wl, per_thread, threads)
        times.append(dt)
    T = sum(times)
    value = args.steps * F * k / T / 1e9
    sample = f"{F} frames of {wl.name} per step ({per_thread} per host thread), {wl.max_iter} iterations"
    line = {
        "impl": "reference", "metric": "decoded info Gbit/s", "value": value, "unit": "Gbit/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "long double (x87 f80)",
        "data": "synthetic (seeded Philox frames, BASELINE.json recipe)",
        # our arm's workload; each timed step decodes the bounded sample named in cpu_baseline.sample
        "config": dict(workload_config(wl, F, args.gpus, scaling=args.scaling, total=F),
                       reference_sample=sample),
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def dram_traffic(wl, frames):
    """DRAM bytes (read + write) per decode launch from the committed ncu
    --set full capture (profiles/traffic.json), when it was taken on this
    workload and batch size; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(wl.name)
        if e and int(e["frames"]) == int(frames):
            return float(e["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def issue_profile(wl):
    """Warp instructions executed per edge-update of the decode kernel, from
    the committed ncu capture of this workload (profiles/issue.json); None if
    there is none."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            return json.load(f).get(wl.name)
    except Exception:
        return None


def roofline(wl, variant, achieved, sms, clock_mhz, frames):
    """The decode kernel's roofline.  SFU model: 4 MUFU per
    edge-update (2 phi per edge and iteration, ex2 + lg2 each) at 16 MUFU/clk/SM.
    Issue model: thread-instructions per edge-update (ncu) x edge-updates/s
    against 148 SMs x 4 schedulers x 32 lanes per clock.  The SFU model is the
    primary bound unless exact shortcuts (saturation / deep tiers) make the
    kernel beat it (fraction > 1): then the price no longer binds and the
    issue model is primary."""
    peak = sms * MUFU_PER_CLK_PER_SM * clock_mhz * 1e6 / MUFU_PER_EDGE_UPDATE / 1e9
    sfu = {"bound": "alu", "kernel": f"ldpc_decode variant {variant}: {KERNEL_NAMES.get(variant, '?')}",
           "achieved": achieved, "peak": peak, "unit": "Gedge-updates/s", "frac": achieved / peak,
           "traffic": dram_traffic(wl, frames),
           "peak_basis": f"SFU: {sms} SMs x 16 MUFU/clk x {clock_mhz:.0f} MHz / 4 MUFU per edge-update (DESIGN.md)"}
    prof = issue_profile(wl)
    if not prof:
        return sfu
    ipe = float(prof["thread_instructions_per_edge_update"])
    issue_peak = sms * 4 * 32 * clock_mhz * 1e6 / 1e12                     # T thread-instr/s
    issue = {"bound": "issue", "achieved": achieved * 1e9 * ipe / 1e12, "peak": issue_peak,
             "unit": "Tthread-instr/s", "frac": achieved * 1e9 * ipe / 1e12 / issue_peak,
             "thread_instructions_per_edge_update": ipe, "budget_at_100pct": 32.0,
             "source": prof.get("source", "profiles/issue.json")}
    if sfu["frac"] > 1.0:
        out = dict(issue, kernel=sfu["kernel"], traffic=sfu["traffic"],
                   peak_basis=f"issue: {sms} SMs x 4 schedulers x 32 lanes x {clock_mhz:.0f} MHz; "
                              "thread-instructions per edge-update from ncu (the SFU price is beaten by exact "
                              "shortcuts, so it no longer binds)")
        out["sfu_model"] = {k: sfu[k] for k in ("achieved", "peak", "unit", "frac")}
        return out
    sfu["issue_model"] = {k: issue[k] for k in ("achieved", "peak", "unit", "frac",
                                                "thread_instructions_per_edge_update", "source")}
    return sfu


def workload_config(wl, frames, gpus, l2_policy=None, launch=None, scaling="strong", total=None, point=0,
                    chunk=None):
    total = total if total is not None else wl.frames
    par = (f"dp{gpus}: {total} frames per step split across ranks by Eq. 9 (strong scaling)" if scaling == "strong"
           else f"dp{gpus}: every rank decodes its own {frames}-frame batch (weak scaling)")
    return {"workload": f"{wl.name}: Gallager ({wl.wc},{wl.wr}) n={wl.n}, {wl.frames} frames in BASELINE.json, "
                        f"{wl.max_iter} {'max (early term.)' if wl.early_term else 'fixed'} SPA iterations, "
                        f"BPSK/AWGN Eb/N0={wl.ebn0_db[point]} dB, fp32 LLRs",
            "n": wl.n, "wc": wl.wc, "wr": wl.wr, "frames_per_step": total if scaling == "strong" else frames * gpus,
            "frames_per_gpu_per_step": frames, "iterations": wl.max_iter,
            "early_term": wl.early_term, "ebn0_db": wl.ebn0_db[point], "sigma": wl.sigma(point),
            "code_seed": W.CODE_SEED, "frame_seed": wl.frame_seeds[point], "parallelism": par,
            "l2_policy": l2_policy or "inputs larger than L2 (LLR batch >> 126 MB), no flush needed",
            **({"chunk_frames": chunk} if chunk else {}),
            **({"launch": launch} if launch else {})}


# --------------------------------------------------------------------------- our arm
def rank_share(total: int, rank: int, world: int, scaling: str):
    """(frame0, count) of this rank.  Strong scaling: the Eq. 9 block of the
    step's `total` frames (dist.shard); weak: a batch of `total`
    frames of its own at global indices rank*total.  Frame f depends only on
    (seed, f), so the frames -- and the summed counters -- do not depend on N."""
    from paper_2201_04265_b200 import dist as LD
    if scaling == "strong":
        return LD.shard(total, rank, world)
    return LD.weak_shard(total, rank)


def chunk_spans(frame0: int, count: int, chunk: int):
    """Contiguous launches [(f0, m)] covering [frame0, frame0 + count)."""
    return [(frame0 + a, min(chunk, count - a)) for a in range(0, count, max(chunk, 1))]


def reduce_step(counters=None, times=None):
    """The only collectives: all_reduce(SUM) of the int64[6] counters (inside
    every timed step) and all_reduce(MAX) of the ranks' device times (after
    the timed region); no-ops on one process."""
    from paper_2201_04265_b200 import dist as LD
    if counters is not None:
        LD.all_reduce_counters(counters)
    if times is not None:
        LD.max_over_ranks(times)
    return counters, times


class RankWork:
    """One rank's share of a step on the device.

    resident (the share's LLRs fit the HBM budget, e.g. C4): info bits,
      codewords and LLRs are generated once (untimed); a step is encode (e1)
      -> decode (a1-a8) -> count (a9) over the whole share.
    chunked (C5: 10^6 frames x 259 KB of LLRs): the share's info bits are
      resident; a step runs, per chunk of `chunk` frames, encode -> channel
      (BPSK/AWGN LLRs of the chunk, Eq. 4; kept inside the timed region, ~0.2%
      of a chunk) -> decode -> count, all on one stream."""

    def __init__(self, L, code, wl, point, frame0, count, chunk, dev, variant, budget_bytes=40e9):
        import torch
        self.L, self.code, self.wl, self.variant = L, code, wl, variant
        info = code.info
        self.n, self.k = info.n, info.k
        kw, nw = L.words(self.k), L.words(self.n)
        self.frame0, self.count = frame0, count
        self.resident = count * self.n * 4 <= budget_bytes
        self.spans = [(frame0, count)] if self.resident else chunk_spans(frame0, count, chunk)
        Fb = max(count if self.resident else min(chunk, count), 1)
        self.Fb = Fb
        self.seed, self.sigma = wl.frame_seeds[point], wl.sigma(point)
        self.d_info = torch.empty((max(count, 1), kw), dtype=torch.int32, device=dev)
        self.d_cw = torch.empty((Fb, nw), dtype=torch.int32, device=dev)
        self.d_llr = torch.empty((Fb, self.n), dtype=torch.float32, device=dev)
        self.d_bits = torch.empty((Fb, nw), dtype=torch.int32, device=dev)
        self.d_syn = torch.empty(Fb, dtype=torch.uint8, device=dev)
        self.d_it = torch.empty(Fb, dtype=torch.int32, device=dev)
        self.d_ctr = torch.zeros(6, dtype=torch.int64, device=dev)
        wsb = L.ldpc_decode_workspace_bytes(code, Fb, wl.max_iter, wl.early_term, variant)
        self.d_ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None
        self.ev = [(torch.cuda.Event(enable_timing=True, external=True),
                    torch.cuda.Event(enable_timing=True, external=True)) for _ in self.spans]

        if count:
            L.ldpc_gen_info(self.seed, frame0, count, self.k, self.d_info)
            if self.resident:
                L.ldpc_encode(code, self.d_info, self.d_cw, count)
                L.ldpc_channel(code, self.seed, frame0, count, self.d_cw, self.sigma, self.d_llr)

    def device_work(self, s):
        import torch
        L, code, wl = self.L, self.code, self.wl
        # a memset node, not a kernel: small steps (C1: ~25 us) feel every node
        memset_async(self.d_ctr, s)
        for (f0, m), (e0, e1) in zip(self.spans, self.ev):
            if m == 0:
                continue
            a = f0 - self.frame0
            info = self.d_info[a:a + m]
            L.ldpc_encode(code, info, self.d_cw, m, stream=s)
            if not self.resident:
                L.ldpc_channel(code, self.seed, f0, m, self.d_cw, self.sigma, self.d_llr, stream=s)
            e0.record(s)
            L.ldpc_decode(code, self.d_llr, m, self.d_bits, self.d_syn, self.d_it, None, self.d_ws, wl.max_iter,
                          wl.early_term, self.variant, stream=s)
            e1.record(s)
            L.ldpc_count_errors(code, info, self.d_bits, self.d_cw, self.d_syn, self.d_it, m, self.d_ctr, stream=s)

    def decode_ms(self):
        return sum(e0.elapsed_time(e1) for (f0, m), (e0, e1) in zip(self.spans, self.ev) if m)

    def encode_ms(self, reps=3):
        """The step's encode launches timed on their own (CUDA events around
        each chunk's ldpc_encode, after the timed region, mean of `reps`):
        events inside the timed graph would add nodes to small steps."""
        import torch
        s = torch.cuda.current_stream()
        total = 0.0
        for _ in range(reps):
            for f0, m in self.spans:
                if m == 0:
                    continue
                a = f0 - self.frame0
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                self.L.ldpc_encode(self.code, self.d_info[a:a + m], self.d_cw, m, stream=s)
                e1.record(s)
                e1.synchronize()
                total += e0.elapsed_time(e1)
        return total / reps


def memset_async(t, stream):
    """cudaMemsetAsync of a tensor on `stream` (a memset node under capture)."""
    from cuda.bindings import runtime as rt
    err, = rt.cudaMemsetAsync(t.data_ptr(), 0, t.numel() * t.element_size(), stream.cuda_stream)
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(f"cudaMemsetAsync failed: {err}")


def graph_kernel_launches(graph):
    """Kernel nodes of a captured step that are this library's (torch's own
    fill kernels excluded): counted from the CUDA graph itself, by name
    (driver API: cuGraphGetNodes / cuGraphKernelNodeGetParams / cuFuncGetName)."""
    try:
        from cuda.bindings import driver as drv
        g = graph.raw_cuda_graph()
        g = drv.CUgraph(init_value=int(g)) if not isinstance(g, drv.CUgraph) else g
        err, nodes, num = drv.cuGraphGetNodes(g, 0)
        err, nodes, num = drv.cuGraphGetNodes(g, num)
        ours = 0
        for nd in nodes:
            err, ty = drv.cuGraphNodeGetType(nd)
            if ty != drv.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
                continue
            err, prm = drv.cuGraphKernelNodeGetParams(nd)
            err, name = drv.cuFuncGetName(prm.func)
            name = name.decode() if isinstance(name, bytes) else str(name)
            if "ldpc" in name:
                ours += 1
        return ours
    except Exception as e:     # pragma: no cover
        print(f"bench: could not count the graph's kernel nodes: {e!r}", file=sys.stderr)
        return None


def measure_point(args, L, code, wl, point, dev, rank, world, launched, sms, props):
    """Time one Eb/N0 point of the workload: W warm-up steps, K timed steps
    (barrier + synchronize on both sides, CUDA events on the launching stream,
    max over ranks).  Returns the rank-0 result dict."""
    import torch
    import torch.distributed as dist

    total = args.frames or wl.frames
    frame0, count = rank_share(total, rank, world, args.scaling)
    work = RankWork(L, code, wl, point, frame0, count, args.chunk, dev, args.variant)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    # The step's kernels are captured once in a CUDA graph and replayed, so host
    # launch overhead stays out of the device timeline (it dominates small
    # batches such as C1); the decode events are external event nodes.
    work.device_work(stream)                  # plans resolved, attributes set before capture
    torch.cuda.synchronize()
    graph, launches = None, None
    if not args.eager:
        graph = torch.cuda.CUDAGraph(keep_graph=True)
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                work.device_work(cap)
        torch.cuda.synchronize()
        launches = graph_kernel_launches(graph)
        graph.instantiate()

    def step():
        if graph is not None:
            graph.replay()
        else:
            work.device_work(stream)
        if launched:
            reduce_step(work.d_ctr)             # a9: the step's counters summed over ranks (NCCL)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # Batches smaller than twice the L2 are evicted before every step by
    # writing a buffer four times the L2 size, outside the step's events;
    # larger inputs stream through L2 on their own.
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20)
    in_bytes = count * work.n * 4
    flush = torch.empty(l2, dtype=torch.int32, device=dev) if in_bytes < 2 * l2 else None
    l2_policy = (f"LLR batch {in_bytes / 2**20:.1f} MiB < 2 x L2: L2 flushed before every timed step "
                 f"({4 * l2 / 2**20:.0f} MiB write, untimed)" if flush is not None else None)
    ctr_total = torch.zeros(6, dtype=torch.int64, device=dev)
    if launched:
        dist.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dec_ms = []
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.add_(1)                   # evict the previous step's inputs from L2 (untimed)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
            ends[i].synchronize()
            dec_ms.append(work.decode_ms())     # decode kernel time of this step
            ctr_total.add_(work.d_ctr)
        torch.cuda.synchronize()
    if launched:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    enc_ms = [work.encode_ms()] * args.steps  # encode kernels (parity + assemble), untimed re-run
    t = torch.tensor([sum(step_ms), sum(dec_ms), sum(enc_ms)], dtype=torch.float64, device=dev)
    reduce_step(None, t)                        # max over ranks (counters were summed every step)
    total_ms, dec_total_ms, enc_total_ms = float(t[0]), float(t[1]), float(t[2])
    ctr = (ctr_total.cpu().numpy() // max(args.steps, 1)).tolist()   # per step, all ranks
    k = work.k
    variant = L.ldpc_decode_variant(code, work.Fb, wl.max_iter, wl.early_term, args.variant)
    clock_mhz = measured_peaks().get("sm_max_mhz", 1965.0)
    # decode kernel throughput of the slowest rank, per GPU (its own edge-updates)
    eu_rank = count * wl.edges * (ctr[4] / max(ctr[5], 1))
    achieved = eu_rank / (dec_total_ms / args.steps / 1e3) / 1e9 if dec_total_ms > 0 else 0.0
    res = {
        "work": work, "graph": graph, "launches_per_step": launches, "count": count, "frame0": frame0,
        "total_ms": total_ms, "dec_ms": dec_total_ms, "counters": ctr, "k": k, "variant": variant,
        "value": ctr[5] * k * args.steps / (total_ms / 1e3) / 1e9,
        "edge_updates_per_s": ctr[4] * wl.edges * args.steps / (total_ms / 1e3),
        "roofline": roofline(wl, variant, achieved, sms, clock_mhz, work.Fb), "clocks": clk.summary(),
        "l2_policy": l2_policy, "total": total,
        "encode": encode_roofline(work, count, enc_total_ms / args.steps, sms, clock_mhz),
    }
    return res


def encode_roofline(work, count, enc_ms, sms, clock_mhz):
    """Encode (e1, Eq. 3): the parity bits are M.P over GF(2).
    Long messages in large batches run it on the tensor cores
    (encode_mma.cu: 0/1 bytes, exact int32 dot products, parity = LSB):
    2 k (n - k) int8 ops per frame against the int8 dense peak, taken as the
    measured bf16 peak (MEASURED_PEAKS.json) x the nominal int8/bf16 ratio 2.
    Otherwise the INT-pipe kernel: one LOP3 (acc ^= m & p) per 32 bit-MACs,
    (n - k) ceil(k/32) LOP3 per frame against the LOP3 rate measured by
    tools/microbench_lop.cu (profiles/peaks_extra.json).  The time is the
    whole ldpc_encode call (parity product + assemble into H order)."""
    if enc_ms <= 0 or count == 0:
        return None
    kw = (work.k + 31) // 32
    chunk = min((m for _, m in work.spans if m > 0), default=0)
    npp = (work.n - work.k + 127) // 128 * 128
    tiles = (chunk + 255) // 256 * ((npp + 255) // 256)      # encode_mma.cu's rule: tiles >= SMs
    if kw >= 16 and tiles >= sms and os.environ.get("LDPC_ENC_MMA", "") != "0":
        pk = measured_peaks()
        bf16 = float(pk.get("bf16_tflops", 0.0) or 0.0)
        basis = (f"2 x measured bf16 {bf16:.1f} TFLOP/s (MEASURED_PEAKS.json, burst; nominal int8/bf16 ratio 2)"
                 if bf16 > 0 else "nominal 4500 TOPS int8 dense (B200_PROFILING.md fallback)")
        peak = 2.0 * bf16 if bf16 > 0 else 4500.0
        ops = float(count) * 2.0 * work.k * (work.n - work.k)
        ach = ops / (enc_ms / 1e3) / 1e12
        return {"bound": "tensor", "kernel": "encode_mma_kernel (tcgen05.mma kind::i8, TMEM accumulators) + "
                                               "encode_assemble_warp_kernel (ldpc_encode)",
                "achieved": ach, "peak": peak, "unit": "T int8-op/s", "frac": ach / peak, "ms_per_step": enc_ms,
                "algorithmic_ops_per_frame": 2 * work.k * (work.n - work.k), "peak_basis": basis}
    ops = float(count) * (work.n - work.k) * kw
    per_clk, basis = 64.0, "assumed 64 LOP3/clk/SM (ALU pipe, 16 lanes/clk/SMSP)"
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_extra.json")) as f:
            px = json.load(f)
        per_clk = float(px["lop3_per_clk_per_sm"])
        basis = f"measured {per_clk:.1f} LOP3/clk/SM (tools/microbench_lop.cu, profiles/peaks_extra.json)"
    except Exception:
        pass
    peak = sms * per_clk * clock_mhz * 1e6 / 1e12
    ach = ops / (enc_ms / 1e3) / 1e12
    return {"bound": "alu", "kernel": "encode_parity_kernel + encode_assemble_kernel (ldpc_encode)",
            "achieved": ach, "peak": peak, "unit": "T LOP3/s", "frac": ach / peak, "ms_per_step": enc_ms,
            "algorithmic_ops_per_frame": (work.n - work.k) * kw,
            "peak_basis": f"{sms} SMs x {basis} x {clock_mhz:.0f} MHz"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "stream":
        return run_stream(args)
    if args.mode == "simulate":
        return run_simulate(args)

    import torch
    import torch.distributed as dist

    import paper_2201_04265_b200 as L
    from paper_2201_04265_b200 import dist as LD

    rank, world, local = LD.world()
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ     # under torchrun
    torch.cuda.set_device(local if launched else 0)
    if launched:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())
    wl = workload(args)
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count

    # ---- setup (untimed): code and device image
    t_setup = time.perf_counter()
    code = L.ldpc_make_H(wl.n, wl.wc, wl.wr, W.CODE_SEED)
    L.ldpc_make_G_device(code, dev)           # bit-identical to ldpc_make_G, ~15x faster (profiles/r01_make_G.jsonl)
    L.ldpc_code_bind_device(code, dev)
    setup_s = time.perf_counter() - t_setup

    points = list(range(len(wl.ebn0_db))) if args.ebn0 is None else [0]
    results = [measure_point(args, L, code, wl, p, dev, rank, world, launched, sms, props) for p in points]
    main_res = results[0]
    total_ms = sum(r["total_ms"] for r in results)
    k = main_res["k"]

    # ---- end to end through the public API with host buffers (rank-local)
    one_launch = None
    if len(results) > 1 and not args.no_sweep_one_launch:
        one_launch = measure_sweep_one_launch(args, L, code, wl, points, results, dev, rank, world, launched, sms,
                                              props)
    e2e = None if args.no_e2e else e2e_measure(L, code, wl, args, dev, main_res["frame0"], main_res["count"], k,
                                               world, expect=main_res["counters"])

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = max(1, min(os.cpu_count() or 1, 128))
        per_thread = max(1, int(os.environ.get("LDPC_CPU_FRAMES_PER_THREAD", "4")))
        dt, F, kk = cpu_oracle_run(wl, per_thread, threads)
        cpu = {"value": F * kk / dt / 1e9, "unit": "Gbit/s", "cores": threads, "kind": "oracle",
               "sample": f"{F} frames of {wl.name} ({wl.max_iter} iterations), {per_thread} per host thread, "
                         f"{dt:.1f} s wall ({dt * threads:.0f} core-s)"}

    if rank == 0:
        ctr = main_res["counters"]
        frames_all = sum(r["counters"][5] for r in results)
        launch = "eager" if main_res["graph"] is None else \
            ("cuda_graph (encode, decode, count)" if main_res["work"].resident
             else f"cuda_graph ({len(main_res['work'].spans)} chunks x (encode, channel, decode, count))")
        line = {
            "metric": "decoded info Gbit/s", "value": frames_all * k * args.steps / (total_ms / 1e3) / 1e9,
            "unit": "Gbit/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox info bits, BPSK/AWGN LLRs; BASELINE.json recipe)",
            "config": workload_config(wl, main_res["count"], world, main_res["l2_policy"], launch, args.scaling,
                                      main_res["total"], points[0],
                                      None if main_res["work"].resident else args.chunk),
            "edge_updates_per_s": sum(r["edge_updates_per_s"] * r["total_ms"] for r in results) / total_ms,
            "decode_ms_per_step": main_res["dec_ms"] / args.steps,
            "mean_iterations": ctr[4] / max(ctr[5], 1), "k": k,
            "counters": {"info_bit_errors": int(ctr[0]), "cw_bit_errors": int(ctr[1]),
                         "frame_errors": int(ctr[2]), "undetected": int(ctr[3]), "frames": int(ctr[5])},
            "roofline": main_res["roofline"],
            "encode_roofline": main_res["encode"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": main_res["clocks"],
            "gpu_launches": (sum(r["launches_per_step"] or 0 for r in results) * args.steps)
            if main_res["launches_per_step"] is not None else None,
            "setup_s": setup_s,
        }
        if len(results) > 1:
            line["points"] = [point_summary(wl, p, r, args.steps) for p, r in zip(points, results)]
            line["sweep_fit"] = sweep_fit(wl, results, args.steps)
            if one_launch is not None:
                line["sweep_one_launch"] = one_launch
            line["config"]["ebn0_db"] = list(wl.ebn0_db)
            line["config"]["frame_seed"] = list(wl.frame_seeds)
            line["config"]["workload"] += f" (sweep {', '.join(str(x) for x in wl.ebn0_db)} dB)"
        print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()
    return 0


def measure_sweep_one_launch(args, L, code, wl, points, results, dev, rank, world, launched, sms, props):
    """The whole Eb/N0 sweep as ONE step: the points' frames (each rank's Eq. 9
    share of every point) form one batch, ordered by ascending Eb/N0 so the
    frames that run longest start first and the batch ends on the ones that
    converge in a few iterations; one ldpc_encode, one ldpc_decode (early
    termination) and one ldpc_count_errors per point slice (per-point BER/FER).
    Frames are independent, so every frame decodes as it does in
    its own point's launch; the per-point counters are compared with those of
    the per-point steps.  Same timing rules as measure_point."""
    import torch
    import torch.distributed as dist

    total = args.frames or wl.frames
    if getattr(args, "sweep_order", "asc") == "desc":   # A/B: shortest-running frames first
        points, results = list(points)[::-1], list(results)[::-1]
    shares = [rank_share(total, rank, world, args.scaling) for _ in points]
    offs = [0]
    for _, c in shares:
        offs.append(offs[-1] + c)
    F = offs[-1]
    k, n = code.info.k, code.info.n
    kw, nw = L.words(k), L.words(n)
    Fa = max(F, 1)
    d_info = torch.empty((Fa, kw), dtype=torch.int32, device=dev)
    d_cw = torch.empty((Fa, nw), dtype=torch.int32, device=dev)
    d_llr = torch.empty((Fa, n), dtype=torch.float32, device=dev)
    d_bits = torch.empty((Fa, nw), dtype=torch.int32, device=dev)
    d_syn = torch.empty(Fa, dtype=torch.uint8, device=dev)
    d_it = torch.empty(Fa, dtype=torch.int32, device=dev)
    d_ctr = torch.zeros((len(points), 6), dtype=torch.int64, device=dev)
    wsb = L.ldpc_decode_workspace_bytes(code, Fa, wl.max_iter, wl.early_term, args.variant)
    d_ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None
    for i, p in enumerate(points):
        f0, c = shares[i]
        if c:
            a = offs[i]
            L.ldpc_gen_info(wl.frame_seeds[p], f0, c, k, d_info[a:a + c])
            L.ldpc_encode(code, d_info[a:a + c], d_cw[a:a + c], c)
            L.ldpc_channel(code, wl.frame_seeds[p], f0, c, d_cw[a:a + c], wl.sigma(p), d_llr[a:a + c])
    ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))

    def device_work(s):
        memset_async(d_ctr, s)
        if F == 0:
            return
        L.ldpc_encode(code, d_info, d_cw, F, stream=s)
        ev[0].record(s)
        L.ldpc_decode(code, d_llr, F, d_bits, d_syn, d_it, None, d_ws, wl.max_iter, wl.early_term, args.variant,
                      stream=s)
        ev[1].record(s)
        for i in range(len(points)):
            a, c = offs[i], shares[i][1]
            if c:
                L.ldpc_count_errors(code, d_info[a:a + c], d_bits[a:a + c], d_cw[a:a + c], d_syn[a:a + c],
                                    d_it[a:a + c], c, d_ctr[i], stream=s)

    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    device_work(stream)
    torch.cuda.synchronize()
    graph, launches = None, None
    if not args.eager:
        graph = torch.cuda.CUDAGraph(keep_graph=True)
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                device_work(cap)
        torch.cuda.synchronize()
        launches = graph_kernel_launches(graph)
        graph.instantiate()

    def step():
        if graph is not None:
            graph.replay()
        else:
            device_work(stream)
        if launched:
            reduce_step(d_ctr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20)
    in_bytes = F * n * 4
    flush = torch.empty(l2, dtype=torch.int32, device=dev) if in_bytes < 2 * l2 else None
    if launched:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, dec_ms = [], []
    ctr = None
    for _ in range(args.steps):
        if flush is not None:
            flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        dec_ms.append(ev[0].elapsed_time(ev[1]) if F else 0.0)
        ctr = d_ctr.cpu().numpy().tolist()
    if launched:
        dist.barrier()
    t = torch.tensor([sum(step_ms), sum(dec_ms)], dtype=torch.float64, device=dev)
    reduce_step(None, t)
    total_ms, dec_total_ms = float(t[0]), float(t[1])
    frames_all = sum(c[5] for c in ctr)
    it_all = sum(c[4] for c in ctr)
    clock_mhz = measured_peaks().get("sm_max_mhz", 1965.0)
    peak = sms * MUFU_PER_CLK_PER_SM * clock_mhz * 1e6 / MUFU_PER_EDGE_UPDATE / 1e9
    it_rank = it_all / max(world, 1)           # the slowest rank's own edge-updates (equal shares up to Eq. 9's remainder)
    ach = it_rank * wl.edges / (dec_total_ms / args.steps / 1e3) / 1e9 if dec_total_ms > 0 else 0.0
    per_point = sum(r["total_ms"] for r in results) / args.steps
    return {
        "value": frames_all * k * args.steps / (total_ms / 1e3) / 1e9, "unit": "Gbit/s",
        "ms_per_step": total_ms / args.steps, "decode_ms_per_step": dec_total_ms / args.steps,
        "frames_per_step": frames_all, "mean_iterations": it_all / max(frames_all, 1),
        "edge_updates_per_s": it_all * wl.edges * args.steps / (total_ms / 1e3),
        "roofline_frac_on_executed_iterations": ach / peak,
        "counters_match_points": [list(map(int, c)) for c in ctr] == [list(map(int, r["counters"])) for r in results],
        "vs_points_one_by_one": per_point / (total_ms / args.steps),
        "gpu_launches_per_step": launches,
        "l2_policy": ("L2 flushed before every timed step" if flush is not None else "inputs larger than 2 x L2"),
        "order_ebn0_db": [wl.ebn0_db[p] for p in points],
        "note": f"the {len(points)} points' frames decoded as one batch in one ldpc_decode call, in `order_ebn0_db` "
                "(ascending Eb/N0 = longest-running frames first); count per point slice; `value`/`points` above time the "
                "points one launch each",
    }


def sweep_fit(wl, results, steps):
    """Early-termination sweep (C2): a least-squares fit of decode time per
    step against mean iterations over the points, t = a + b x iterations.
    b is the cost of one iteration of every frame (its SFU-model fraction is
    the decoder's per-iteration efficiency); a / b is the per-frame fixed cost
    in iterations (ingest, output, the check phase that detects convergence
    one phase late, the tail of the persistent grid) -- it is what pulls the
    fraction down at high Eb/N0, where frames stop after 5-7 iterations."""
    xs = [r["counters"][4] / max(r["counters"][5], 1) for r in results]
    ys = [r["dec_ms"] / steps for r in results]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    if sxx <= 0:
        return None
    b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    a = my - b * mx
    frames = results[0]["counters"][5]
    peak = results[0]["roofline"].get("sfu_model", results[0]["roofline"])["peak"]
    per_iter = frames * wl.edges / (b / 1e3) / 1e9 if b > 0 else None
    return {"decode_ms_per_iteration_of_all_frames": b, "decode_ms_fixed_per_step": a,
            "fixed_cost_in_iterations_per_frame": a / b if b > 0 else None,
            "per_iteration_gedge_updates_per_s": per_iter,
            "per_iteration_sfu_frac": per_iter / peak if per_iter else None,
            "note": "decode time = fixed + per-iteration x mean iterations, fitted over the sweep; at high Eb/N0 "
                    "the fixed cost weighs on 5-7 iterations, so the fraction on executed iterations falls below "
                    "the per-iteration efficiency.  Measured at 3.0 dB (DESIGN.md section 12): 10k frames 0.388, "
                    "40k 0.440, 160k 0.457 -- about 0.05 ms of the 10k-frame step is the tail of the few frames "
                    "that run all 50 iterations, the rest ~1.2 iterations per frame (ingest, output, the check "
                    "phase that detects convergence)"}


def point_summary(wl, p, r, steps):
    c = r["counters"]
    k = r["k"]
    return {"ebn0_db": wl.ebn0_db[p], "sigma": wl.sigma(p), "frame_seed": wl.frame_seeds[p],
            "info_gbit_s": r["value"], "ms_per_step": r["total_ms"] / steps,
            "decode_ms_per_step": r["dec_ms"] / steps, "mean_iterations": c[4] / max(c[5], 1),
            "ber_info": c[0] / max(c[5] * k, 1), "fer": c[2] / max(c[5], 1),
            "undetected": c[3], "frames": c[5],
            "roofline_frac_on_executed_iterations": r["roofline"]["frac"],
            "roofline_bound": r["roofline"]["bound"]}


def e2e_measure(L, code, wl, args, dev, frame0, count, k, world, expect=None):
    """Same metric through the public API with pinned host buffers: H2D of the
    step's info bits and LLRs, encode, decode, count, D2H of the decoded bits
    and the counters, all inside the timed region.  Pinned host memory is
    capped at E2E_PINNED_BYTES over all ranks (the frames beyond it are not
    part of the e2e sample; C4 fits whole at every N)."""
    import torch
    n = code.info.n
    kw, nw = L.words(k), L.words(n)
    per_frame = n * 4 + kw * 4 + nw * 4
    cap = int(E2E_PINNED_BYTES / max(world, 1) / per_frame)
    F = min(count, cap)
    if args.e2e_frames:
        F = min(F, args.e2e_frames)
    if F <= 0:
        return {"value": None, "unit": "Gbit/s", "error": "no frames on this rank"}
    Fc = min(F, args.e2e_chunk)              # pipeline chunk
    # chunk sizes ramp up from Fc/8 by x2.5: the pipeline's fill (the first
    # chunk's H2D, which nothing overlaps) shrinks 8x, and each next chunk's
    # H2D still lands before the compute of the one before it ends (H2D of a
    # frame is faster than its decode)
    # (multiples of the SM count, so each chunk's decode ends in full waves)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    if F > Fc and Fc >= 8 * sms:
        Fc = Fc // sms * sms
    sizes, a = [], 0
    c = max(1, Fc // 8 // sms * sms if Fc >= 8 * sms else Fc // 8) if F > Fc else F
    while a < F:
        m = min(c, F - a)
        sizes.append((a, m))
        a += m
        c = min(Fc, int(c * 2.5) // sms * sms if c >= sms else int(c * 2.5))
    nchunks = len(sizes)
    try:
        h_info = torch.empty((F, kw), dtype=torch.int32, pin_memory=True)
        h_llr = torch.empty((F, n), dtype=torch.float32, pin_memory=True)
        h_bits = torch.empty((F, nw), dtype=torch.int32, pin_memory=True)
        h_ctr = torch.empty(6, dtype=torch.int64, pin_memory=True)
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "Gbit/s", "error": f"pinned alloc failed: {e}"}
    bufs = [dict(info=torch.empty((Fc, kw), dtype=torch.int32, device=dev),
                 cw=torch.empty((Fc, nw), dtype=torch.int32, device=dev),
                 llr=torch.empty((Fc, n), dtype=torch.float32, device=dev),
                 bits=torch.empty((Fc, nw), dtype=torch.int32, device=dev),
                 syn=torch.empty(Fc, dtype=torch.uint8, device=dev),
                 it=torch.empty(Fc, dtype=torch.int32, device=dev)) for _ in range(2)]
    # the rank's frames, generated once on the device and parked in host memory (untimed)
    seed = wl.frame_seeds[0]
    for c in range(nchunks):
        a, m = sizes[c]
        b = bufs[0]
        L.ldpc_gen_info(seed, frame0 + a, m, k, b["info"])
        L.ldpc_encode(code, b["info"], b["cw"], m)
        L.ldpc_channel(code, seed, frame0 + a, m, b["cw"], wl.sigma(), b["llr"])
        h_info[a:a + m].copy_(b["info"][:m])
        h_llr[a:a + m].copy_(b["llr"][:m])
    d_ctr = torch.zeros(6, dtype=torch.int64, device=dev)
    wsb = max(L.ldpc_decode_workspace_bytes(code, m, wl.max_iter, wl.early_term, args.variant)
              for m in sorted({m for _, m in sizes}))
    # one workspace and one compute stream per buffer: consecutive chunks
    # compute on different streams, so a chunk's decode starts on the SMs the
    # previous chunk's last frames leave idle instead of after them
    d_ws = [torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev) if wsb else None for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s_cmp = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def step():
        """Three-stage pipeline over chunks: H2D (s_in) -> encode, decode,
        count (s_cmp[c % 2]) -> D2H of the decoded bits (s_out), double-buffered."""
        s_cmp[0].wait_stream(s_out)                 # the previous step's counters have been read
        with torch.cuda.stream(s_cmp[0]):
            d_ctr.zero_()
        s_cmp[1].wait_stream(s_cmp[0])
        for c in range(nchunks):
            (a, m), i = sizes[c], c % 2
            b, sc = bufs[i], s_cmp[i]
            if c >= 2:
                s_in.wait_event(ev_cmp[i])          # buffer i's inputs consumed
            with torch.cuda.stream(s_in):
                b["info"][:m].copy_(h_info[a:a + m], non_blocking=True)
                b["llr"][:m].copy_(h_llr[a:a + m], non_blocking=True)
                ev_in[i].record(s_in)
            sc.wait_event(ev_in[i])
            if c >= 2:
                sc.wait_event(ev_out[i])            # buffer i's bits drained
            L.ldpc_encode(code, b["info"], b["cw"], m, stream=sc)
            L.ldpc_decode(code, b["llr"], m, b["bits"], b["syn"], b["it"], None, d_ws[i], wl.max_iter,
                          wl.early_term, args.variant, stream=sc)
            L.ldpc_count_errors(code, b["info"], b["bits"], b["cw"], b["syn"], b["it"], m, d_ctr, stream=sc)
            ev_cmp[i].record(sc)
            s_out.wait_event(ev_cmp[i])
            with torch.cuda.stream(s_out):
                h_bits[a:a + m].copy_(b["bits"][:m], non_blocking=True)
                ev_out[i].record(s_out)
        with torch.cuda.stream(s_out):
            h_ctr.copy_(d_ctr, non_blocking=True)

    for sc in s_cmp:
        sc.wait_stream(torch.cuda.current_stream())
    step()
    torch.cuda.synchronize()
    steps = max(1, args.steps)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(s_in)
    for _ in range(steps):
        s_in.wait_stream(s_out)                     # steps do not overlap each other
        step()
    s_in.wait_stream(s_out)
    end.record(s_in)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    frames_all = torch.tensor([F], dtype=torch.int64, device=dev)
    from paper_2201_04265_b200 import dist as LD
    LD.max_over_ranks(t)
    LD.all_reduce_counters(frames_all)
    ms = float(t[0])
    bi = F * kw * 4 + F * n * 4
    bo = F * nw * 4 + 6 * 8
    # the pipelined path's six counters (last step, all ranks) against the
    # device-timed step's, when the e2e sample is the whole shard
    c = h_ctr.to(dev)
    LD.all_reduce_counters(c)
    match = (c.cpu().tolist() == [int(x) for x in expect]) if (expect is not None and F == count) else None
    return {"value": int(frames_all[0]) * steps * k / (ms / 1e3) / 1e9, "unit": "Gbit/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "frames_per_gpu_per_step": F, "counters_match_device": match,
            "note": f"pinned host buffers; H2D / encode+decode+count / D2H pipelined over {nchunks} chunks (ramping "
                    f"{sizes[0][1]} -> {Fc} frames) on four streams (two compute streams alternating by chunk); "
                    f"max over ranks" +
                    ("" if F == count else f"; sample of {F} of the rank's {count} frames (pinned-memory cap "
                                           f"{E2E_PINNED_BYTES / 1e9:.0f} GB over all ranks)")}


if __name__ == "__main__":
    sys.exit(main())
