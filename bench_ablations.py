"""NEXT-2 kernel-level ablations of the paper's design, timed on
the C2 decode batch (BASELINE configs[2], 32 layers, fp16) beside the paged,
unpadded fused kernel that bench.py reports:

* no-unify-mem -- every adapter in its own contiguous memory (pages claimed
  in ascending order with no KV pages between them), the same fused kernel.
  The paper's variant keeps a separate contiguous buffer per adapter; at the
  kernel level the only difference is page placement, which our kernels are
  invariant to (G3), so this quantifies what Unified Paging costs the kernel.
* S-LoRA-bmm -- "copy to contiguous memory, pad to the max rank, cuBLAS
  bmm": per (layer, projection) the batch's adapter rows are gathered out of
  the pool pages (slora_gather_pages), laid out zero-padded to r_max
  ([U, r_max, h] and [U, r_max, d]), expanded per token and multiplied with
  torch.bmm (cuBLAS) -- the padded, per-token-copy path the paper's MBGMV
  replaces.  Its bytes are counted the same way as ours (unique adapters'
  weights, x, y), so its GB/s is comparable.
Called by bench.py (the "ablations" key of the JSON line); also runnable alone.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _time(fn, stream, steps):
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        fn()
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps


def run(stream=None, layers=32, steps=5):
    import torch
    import bench
    from synth import workload as wl
    stream = stream or torch.cuda.current_stream()
    cfg = wl.CONFIGS["c2"]
    out = {"workload": cfg.name, "layers": layers}
    # ---- no-unify-mem: contiguous per-adapter placement, same fused kernel (graph replay as bench.py)
    W = bench.Workload(cfg, layers, 1, 0, torch.cuda.current_device(), stream, order="ascending", kv_tokens=0)
    W.capture(stream)
    ms_c, _ = bench.timed_steps(W, stream, steps * 2, 1)
    bytes_step = (W.bytes_qkv + W.bytes_o) * layers
    out["no_unify_mem"] = {"ms_per_step": round(ms_c, 4), "GBps": round(bytes_step / ms_c / 1e6, 1),
                           "value": round(W.Tad * layers / (ms_c / 1e3), 1),
                           "placement": "ascending page ids, no KV pages: each adapter's rows contiguous"}
    # ---- S-LoRA-bmm on the same pool: gather -> pad -> per-token bmm
    b = W.batch
    ids = b.unique
    ranks = [b.ranks[a] for a in ids]
    U, rmax, H = len(ids), max(ranks), W.H
    tok_ad = np.array([ids.index(a) if a >= 0 else -1 for a in b.token_adapter])
    sel = torch.from_numpy(np.nonzero(tok_ad >= 0)[0]).cuda()
    tok_idx = torch.from_numpy(tok_ad[tok_ad >= 0]).cuda()
    pages = {a: W.pool.adapter_pages(a) for a in ids}
    # page list per (layer, proj, tensor): adapter-major, r rows each (claim order layer, proj, A/B, row)
    plist, dst_rows = {}, {}
    for l in range(layers):
        for p in range(4):
            for t in range(2):
                lst, rows = [], []
                for ui, a in enumerate(ids):
                    r = b.ranks[a]
                    base = ((l * 4 + p) * 2 + t) * r
                    lst.extend(pages[a][base:base + r].tolist())
                    rows.extend(ui * rmax + j for j in range(r))
                plist[(l, p, t)] = np.array(lst, np.int32)
                dst_rows[(l, p, t)] = torch.tensor(rows, device="cuda")
    nr = sum(ranks)
    cat = torch.empty((nr, H), dtype=W.td, device="cuda")
    padA = torch.zeros((U * rmax, H), dtype=W.td, device="cuda")
    padB = torch.zeros((U * rmax, H), dtype=W.td, device="cuda")

    def bmm_step():
        for l in range(layers):
            x = W.x[l][sel]  # [Tad, H]
            for p in range(4):
                for t, pad in ((0, padA), (1, padB)):
                    W.pool.gather_pages(plist[(l, p, t)], cat, stream=stream)  # copy out of the pool pages
                    pad.index_copy_(0, dst_rows[(l, p, t)], cat)               # pad to r_max
                A_tok = padA.view(U, rmax, H)[tok_idx]                          # [Tad, rmax, H] per-token copy
                B_tok = padB.view(U, rmax, H)[tok_idx]
                v = torch.bmm(x.unsqueeze(1), A_tok.transpose(1, 2))           # [Tad, 1, rmax] (cuBLAS)
                d = torch.bmm(v, B_tok).squeeze(1)                              # [Tad, H]
                y = W.y[l, p]
                y.index_add_(0, sel, d)

    ms_b = _time(bmm_step, stream, steps)
    out["s_lora_bmm"] = {"ms_per_step": round(ms_b, 4), "GBps_on_our_alg_bytes": round(bytes_step / ms_b / 1e6, 1),
                         "value": round(W.Tad * layers / (ms_b / 1e3), 1), "r_max": rmax,
                         "padded_weight_bytes_per_step": int(2 * 4 * layers * U * rmax * H * W.es),
                         "note": "gather (slora_gather_pages) + zero-pad to r_max + per-token torch.bmm (cuBLAS), "
                                 "eager"}
    W.close()
    return out


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    print(json.dumps(run()))
