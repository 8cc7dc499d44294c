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
    t0 = tr[0][tr[0] > 0].min()
    for call, arr in (("qkv", tr[0]), ("o", tr[1])):
        print(f"== {call} launch of layer {os.environ.get('SLORA_TRACE_LAYER', '16')} (us after qkv start)")
        for cta in range(16):
            ev = [(e, (arr[cta, e] - t0) / 1e3) for e in range(64) if arr[cta, e] > 0]
            print(f"cta{cta:2d} " + " ".join(f"{name(e)}={t:.2f}" for e, t in sorted(ev, key=lambda z: z[1])))
        a = allc[0 if call == "qkv" else 1]
        live = a[:, 0] > 0
        rel = (a[live] - t0) / 1e3
        if rel.size:
            q = lambda col: np.percentile(rel[:, col], [0, 10, 50, 90, 100]).round(2).tolist()
            print(f"all {int(live.sum())} CTAs: start {q(0)} pdl {q(1)} slot0 {q(2)} end {q(3)}")
            late = np.argsort(-rel[:, 3])[:12]
            idx = np.nonzero(live)[0]
            print("latest CTAs (id, start, slot0, end): " +
                  " ".join(f"({idx[i]},{rel[i,0]:.1f},{rel[i,2]:.1f},{rel[i,3]:.1f})" for i in late))
        for cta in range(4):
            iss = [(arr[cta, 160 + k] - t0) / 1e3 for k in range(96) if arr[cta, 160 + k] > 0]
            rdy = [(arr[cta, 64 + k] - t0) / 1e3 for k in range(96) if arr[cta, 64 + k] > 0]
            print(f"cta{cta} slots issued: " + " ".join(f"{t:.2f}" for t in iss))
            print(f"cta{cta} slots ready : " + " ".join(f"{t:.2f}" for t in rdy))


if __name__ == "__main__":
    main()
