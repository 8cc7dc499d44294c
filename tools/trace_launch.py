#!/usr/bin/env python
"""Timeline of one fused launch from the kernel's globaltimer trace
(SLORA_TRACE=1; the first 16 CTAs record events, see TRACE() in kernels.cu).

Per traced CTA: entry, exit, and per consumer piece (start, data ready, done)
in microseconds from the earliest entry, with the piece code (kind, tokens,
rows or rank) the resolver recorded.

    SLORA_TRACE=1 python tools/trace_launch.py [--workload c2] [--call qkv|o]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    os.environ.setdefault("SLORA_TRACE", "1")
    import torch
    import bench
    from synth import workload as wl

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--call", default="qkv")
    ap.add_argument("--layers", type=int, default=4)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.workload]
    s = torch.cuda.current_stream()
    W = bench.Workload(cfg, a.layers, 1, 0, 0, s)
    b = W.dbatch
    H = W.H
    b.prepare(W.batch.token_adapter, stream=s)
    for rep in range(3):
        for l in range(a.layers):
            ys = [W.y[l, p] for p in range(4)]
            b.apply(l, a.call, W.x[l], H, ys, [H] * 4, stream=s)
            b.apply(l, a.call, W.x[l], H, ys, [H] * 4, stream=s)
    torch.cuda.synchronize()
    tr = W.pool.debug_trace().reshape(16, 1024).astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    us = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")  # noqa: E731
    ends = []
    for c in range(16):
        row = tr[c]
        if row[0] == 0:
            continue
        ends.append(us(row[2]))
        print(f"CTA {c:2d}: entry {us(row[0]):6.2f}  exit {us(row[2]):6.2f}")
        for i in range(48):
            st, rd, dn = row[64 + i], row[256 + i], row[112 + i]
            if st == 0:
                break
            code = int(row[208 + i])
            kind = "S" if code // 1000000 == 0 else "E"
            nt = (code // 100000) % 10
            rr = code % 100000
            print(f"    {kind} nt={nt} {'rows' if kind == 'S' else 'r'}={rr:3d}  start {us(st):6.2f}"
                  f"  ready {us(rd):6.2f}  slots {us(row[304 + i]):6.2f}  math {us(row[352 + i]):6.2f}"
                  f"  sync {us(row[400 + i]):6.2f}  done {us(dn):6.2f}  ({us(dn) - us(st):5.2f})")
    for c in range(2):
        row = tr[c]
        iss = [(sq, us(row[768 + sq]), us(row[512 + sq])) for sq in range(240) if row[768 + sq] > 0]
        print(f"CTA {c} slots (seq: issue -> full, latency):")
        print("   " + "  ".join(f"{sq}:{a:.2f}->{b:.2f}({b - a:.2f})" for sq, a, b in iss[:60]))
    print(f"max exit {np.nanmax(ends):.2f} us, min exit {np.nanmin(ends):.2f} us")


if __name__ == "__main__":
    main()
