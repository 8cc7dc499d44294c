#!/usr/bin/env python
"""globaltimer timeline of the MBGMV group kernel (GPU, diagnostics).

Runs the bench workload's layer sequence from a CUDA graph with SLORA_TRACE=1;
the q/k/v and o launches of layer SLORA_TRACE_LAYER (default 16) record events
for CTAs 0-15 (mbgmv.cu GTRACE).  Prints each CTA's events in microseconds
relative to the earliest q/k/v event.

    SLORA_TRACE=1 python tools/trace_group.py [--workload c2] [--layers 32]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {0: "start", 1: "desc", 2: "ids", 3: "emit0", 4: "prod_end", 8: "pdl", 9: "dbar", 10: "slot0",
         16: "shrink0", 63: "end"}


def name(e):
    if e in NAMES:
        return NAMES[e]
    if 17 <= e < 63:
        i, k = divmod(e - 17, 3)
        return ["shrink+1", "v", "expand"][k] + f"[{i}]"
    return str(e)


def main():
    os.environ.setdefault("SLORA_TRACE", "1")
    import torch
    import bench
    from synth import workload as wl

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--layers", type=int, default=32)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.workload]
    s = torch.cuda.current_stream()
    W = bench.Workload(cfg, a.layers, 1, 0, 0, s)
    W.capture(s)
    for _ in range(5):
        W.step(s)
    torch.cuda.synchronize()
    raw = W.pool.debug_trace().reshape(-1).astype(np.int64)
    tr = np.stack([raw[0:4096].reshape(16, 256), raw[8192:8192 + 4096].reshape(16, 256)])
    allc = np.stack([raw[4096:4096 + 2048].reshape(512, 4), raw[8192 + 4096:8192 + 4096 + 2048].reshape(512, 4)])
    for a in allc:  # column 2 holds item counts, not timestamps
        a[:, 2] = np.where(a[:, 0] > 0, a[:, 2], 0)
    t0 = allc[0][:, 0][allc[0][:, 0] > 0].min()
    for call, arr in (("qkv", tr[0]), ("o", tr[1])):
        print(f"== {call} launch of layer {os.environ.get('SLORA_TRACE_LAYER', '16')} (us after qkv start)")
        for cta in range(16):
            ev = [(e, (arr[cta, e] - t0) / 1e3) for e in range(64) if arr[cta, e] > 0]
            print(f"cta{cta:2d} " + " ".join(f"{name(e)}={t:.2f}" for e, t in sorted(ev, key=lambda z: z[1])))
        a = allc[0 if call == "qkv" else 1]
        live = a[:, 0] > 0
        rel = (a[live].astype(np.float64) - t0) / 1e3
        if rel.size:
            q = lambda col: np.percentile(rel[:, col], [0, 10, 50, 90, 100]).round(2).tolist()
            nit = a[live][:, 2]
            print(f"all {int(live.sum())} CTAs: start {q(0)} pdl {q(1)} end {q(3)} "
                  f"items/CTA min {nit.min()} median {int(np.median(nit))} max {nit.max()}")
            late = np.argsort(-rel[:, 3])[:12]
            idx = np.nonzero(live)[0]
            print("latest CTAs (id, start, end, items): " +
                  " ".join(f"({idx[i]},{rel[i,0]:.1f},{rel[i,3]:.1f},{nit[i]})" for i in late))
        for cta in range(2):
            print(f"cta{cta} slot k: issued (weights) / consumer waits from / consumer got it (us)")
            for k in range(64):
                w, g, i = arr[cta, 128 + k], arr[cta, 64 + k], arr[cta, 192 + k]
                if g <= 0:
                    continue
                f = lambda v: f"{(v - t0) / 1e3:7.2f}" if v > 0 else "      -"
                print(f"  k={k:2d} issued {f(i)} wait {f(w)} got {f(g)}  stall {(g - w) / 1e3:5.2f}")


if __name__ == "__main__":
    main()
