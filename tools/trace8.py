#!/usr/bin/env python
"""Per-warp task timeline of the warp-task MBGMV kernel (mbgmv8.cu) from its
globaltimer trace (SLORA_TRACE=1): CTAs 0-15, warps 0-11, up to 20 tasks each.

    SLORA_TRACE=1 python tools/trace8.py [--workload c2] [--call qkv|o] [--ctas 4]
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
    ap.add_argument("--ctas", type=int, default=4)
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
    torch.cuda.synchronize()
    tr = W.pool.debug_trace().reshape(16, 1024).astype(np.int64)
    starts = [tr[c, w * 64] for c in range(16) for w in range(16) if tr[c, w * 64] > 0]
    t0 = min(starts)
    us = lambda v: (v - t0) / 1e3  # noqa: E731
    ends = []
    for c in range(16):
        for w in range(16):
            row = tr[c, w * 64: w * 64 + 64]
            if row[0] == 0:
                continue
            segs = []
            for k in range(10):
                st, wt, cp, fi, fe, code = row[1 + 6 * k: 7 + 6 * k]
                if st == 0 or fi == 0 or fi < st:
                    break
                kind = "S" if code // 1000000 == 0 else "E"
                f = lambda v: f"{us(v):.1f}" if v > 0 else "-"  # noqa: E731
                segs.append(f"{kind}{(code // 100000) % 10}r{code % 100000}[{f(st)} w{f(wt)} c{f(cp)} f{f(fi)} n{f(fe)}]")
                ends.append(us(fi))
            if c < a.ctas:
                print(f"c{c:02d}w{w:02d} | " + " ".join(segs))
    print(f"last task end {max(ends):.2f} us")


if __name__ == "__main__":
    main()
