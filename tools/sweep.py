#!/usr/bin/env python
"""Knob sweeps on one GPU, printed as markdown tables.

  * C5: TS in {8, 16, 32} x BS in {32, 64, 128, 256}: runtime (median of 5 renders, CUDA
    events on the context stream, device outputs) and the device memory the context holds
    (Table 6 style).  Also max |bounds - bounds(16, 64)| (TS/BS are
    performance knobs only, reading O1).
  * C3: parts = 1 vs 8 on yaw: runtime and mean bound width (MPG): the
    partition trades time for tightness.

usage (GPU box): python tools/sweep.py [--reps 5] > gpurun_out/sweep.md
"""
import argparse
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_00308_b200 import Context  # noqa: E402
from workloads import make_config  # noqa: E402


def timed(ctx, ts, bs, reps):
    lo, hi, st = ctx.as_render_bounds(ts, bs)
    s = torch.cuda.current_stream()
    ms = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        lo, hi, st = ctx.as_render_bounds(ts, bs)
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms), lo, hi, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    print(f"GPU: {torch.cuda.get_device_name(0)}\n")
    ctx = Context(0)
    w = make_config("C5")
    ctx.load_workload(w)
    _, blo, bhi, _ = timed(ctx, 16, 64, 1)
    print("## C5 tile (TS) x batch (BS) sweep\n")
    print("| TS | BS (requested) | ms / render | abstract px/s | context device MB | items | "
          "max abs diff vs (16, 64) |")
    print("|---|---|---|---|---|---|---|")
    for ts in (8, 16, 32):
        for bs in (32, 64, 128, 256):
            ctx.close()
            ctx = Context(0)  # fresh context: device_bytes = what this (TS, BS) needs
            ctx.load_workload(w)
            ms, lo, hi, st = timed(ctx, ts, bs, args.reps)
            d = max(float((lo - blo).abs().max()), float((hi - bhi).abs().max()))
            px = w.camera["W"] * w.camera["H"] * w.n_sub / (ms * 1e-3)
            print(f"| {ts} | {bs} | {ms:.3f} | {px:.4g} | {st['device_bytes'] / 2**20:.1f} | "
                  f"{st['n_items']} | {d:.2e} |")
    print("\n## C3 partition (parts on yaw)\n")
    print("| parts | sub-boxes | ms / render | abstract px/s | MPG (mean hi-lo per channel) |")
    print("|---|---|---|---|---|")
    for parts in (1, 8):
        w3 = make_config("C3")
        pb = dict(w3.pose_box)
        pb["parts"] = [1, 1, 1, 1, 1, parts]
        w3.pose_box = pb
        ctx.load_workload(w3)
        ms, lo, hi, st = timed(ctx, 16, 16, args.reps)
        mpg = float((hi - lo).double().mean())
        px = w3.camera["W"] * w3.camera["H"] * w3.n_sub / (ms * 1e-3)
        print(f"| {parts} | {w3.n_sub} | {ms:.3f} | {px:.4g} | {mpg:.4f} |")
    ctx.close()


if __name__ == "__main__":
    main()
