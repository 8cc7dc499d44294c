#!/usr/bin/env python
"""Per-call timing breakdown of the fused LoRA launches (GPU, diagnostics).

Captures CUDA graphs of L layers of {q/k/v apply, o apply} (as bench.py),
{q/k/v only} and {o only}, replays each and prints the mean time per launch.
Knobs are the library's env variables (SLORA_DBG, SLORA_NS, ...), read once
per process, so run one process per setting.

    python tools/layer_micro.py [--workload c2] [--layers 32] [--reps 20]
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
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.workload]
    s = torch.cuda.current_stream()
    W = bench.Workload(cfg, a.layers, 1, 0, 0, s)
    b = W.dbatch
    H = W.H
    b.prepare(W.batch.token_adapter, stream=s)
    torch.cuda.synchronize()

    def seq(which):
        for l in range(a.layers):
            ys = [W.y[l, p] for p in range(4)]
            for m in which:
                b.apply(l, m, W.x[l], H, ys, [H] * 4, stream=torch.cuda.current_stream())

    out = {"tag": a.tag, "workload": cfg.name, "env": {k: v for k, v in os.environ.items() if k.startswith("SLORA")}}
    for name, which in (("layer", ("qkv", "o")), ("qkv", ("qkv",)), ("o", ("o",))):
        for _ in range(2):
            seq(which)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=cs):
            seq(which)
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
        us = t0.elapsed_time(t1) * 1e3 / a.reps / (a.layers * len(which))
        byts = {"layer": (W.bytes_qkv + W.bytes_o) / 2, "qkv": W.bytes_qkv, "o": W.bytes_o}[name]
        out[name] = {"us_per_launch": round(us, 2), "GBps": round(byts / us / 1e3, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
