#!/usr/bin/env python
"""Fused vs split MBGMV (GPU, diagnostics): 32-layer CUDA graphs of
  fused:  q/k/v apply, o apply                      (2 launches per layer)
  split:  q/k/v shrink -> expand, o shrink -> expand (4 launches per layer,
          v through a workspace; the expand prefetches B before its PDL wait)
on the C2 decode batch; prints us per layer and the relative max difference.

    python tools/split_micro.py [--workload c2] [--layers 32] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from synth import workload as wl

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.workload]
    s = torch.cuda.current_stream()
    W = bench.Workload(cfg, a.layers, 1, 0, 0, s)
    b = W.dbatch
    H = W.H
    b.prepare(W.batch.token_adapter, stream=s)
    vq = torch.empty(b.v_elems("qkv"), dtype=torch.float32, device="cuda")
    vo = torch.empty(b.v_elems("o"), dtype=torch.float32, device="cuda")
    y0 = W.y.clone()

    def fused():
        for l in range(a.layers):
            ys = [W.y[l, p] for p in range(4)]
            b.apply(l, "qkv", W.x[l], H, ys, [H] * 4, stream=torch.cuda.current_stream())
            b.apply(l, "o", W.x[l], H, ys, [H] * 4, stream=torch.cuda.current_stream())

    def split():
        st = torch.cuda.current_stream()
        for l in range(a.layers):
            ys = [W.y[l, p] for p in range(4)]
            b.shrink(l, "qkv", W.x[l], H, vq, stream=st)
            b.expand(l, "qkv", vq, 1, ys, [H] * 4, stream=st)
            b.shrink(l, "o", W.x[l], H, vo, stream=st)
            b.expand(l, "o", vo, 1, ys, [H] * 4, stream=st)

    out = {"workload": cfg.name}
    res = {}
    for name, fn in (("fused", fused), ("split", split)):
        W.y.copy_(y0)
        fn()
        torch.cuda.synchronize()
        res[name] = W.y.clone()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=cs):
            fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.reps):
            g.replay()
        t1.record()
        torch.cuda.synchronize()
        out[name + "_us_per_layer"] = round(t0.elapsed_time(t1) * 1e3 / a.reps / a.layers, 2)
    d = (res["fused"].float() - res["split"].float()).abs().max().item()
    out["max_abs_diff_fused_vs_split"] = d
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
