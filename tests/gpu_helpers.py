"""Helpers for the GPU parity tests: set up a pool + adapters from synth/,
run the CUDA path through the C-ABI binding, and compute the oracle on the
same stored values."""
from __future__ import annotations

import numpy as np

import oracle
from synth import workload as wl

TOL = {"f32": 1e-5, "f16": 2e-2, "bf16": 2e-2}   # BASELINE.json north_star


def torch_dtype(dtype):
    import torch
    return {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dtype]


def to_device(arr, dtype):
    """Stored numpy array -> cuda tensor of the same bits."""
    import torch
    if dtype == "bf16":
        t = torch.from_numpy(arr.view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.cuda()


def from_device(t, dtype):
    """cuda tensor -> float64 numpy (exact)."""
    return t.double().cpu().numpy()


def normalized_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30)) if ref.size else 0.0


class Case:
    """One pool with the batch's adapters loaded, placed by (order, seed),
    optionally interleaved with KV pages (KV and adapters interleaved)."""

    def __init__(self, cfg, batch, num_layers=1, order="ascending", seed=0, kv_interleave=0,
                 extra_capacity=0, weight_fn=None, scale=None, stream=None):
        import torch
        from paper_2311_03285_b200 import Pool
        self.cfg, self.batch, self.L = cfg, batch, num_layers
        h = cfg.hidden
        need = sum(num_layers * 4 * 2 * r for r in batch.ranks.values())
        cap = need + 2 * kv_interleave * num_layers * (len(batch.ranks) + 1) + extra_capacity + 16
        self.pool = Pool(h, num_layers, cap, dtype=cfg.dtype, device=0, order=order, seed=seed,
                         max_adapters=max(64, len(batch.ranks) + 8))
        self.stream = stream or torch.cuda.current_stream()
        self.weights = {}   # adapter -> [ (A, B) per layer*4+proj ] stored dtype
        self.scale = scale or {}
        rid = 10_000
        for a in batch.unique:
            if kv_interleave:
                self.pool.kv_alloc(rid, kv_interleave)
                rid += 1
            r = batch.ranks[a]
            if weight_fn is None:
                wts = [wl.adapter_weights(cfg, a, l, p, r) for l in range(num_layers) for p in range(4)]
            else:
                wts = [weight_fn(a, l, p, r) for l in range(num_layers) for p in range(4)]
            host = np.concatenate([np.concatenate([A.ravel(), B.ravel()]) for A, B in wts])
            self.pool.adapter_load(a, r, host, scale=self.scale.get(a, 1.0), stream=self.stream)
            self.weights[a] = wts
        if kv_interleave:
            self.pool.kv_alloc(rid, kv_interleave)

    def oracle_proj(self, x, y_in, layer, proj):
        dt = self.cfg.dtype
        ids = self.batch.unique
        slot = np.array([ids.index(a) if a >= 0 else -1 for a in self.batch.token_adapter], np.int64)
        As = [oracle.to_f64(self.weights[a][layer * 4 + proj][0], dt) for a in ids]
        Bs = [oracle.to_f64(self.weights[a][layer * 4 + proj][1], dt) for a in ids]
        sc = np.array([self.scale.get(a, 1.0) for a in ids], np.float64) if ids else None
        return oracle.lora_apply(oracle.to_f64(x, dt), oracle.to_f64(y_in, dt), As, Bs, slot, sc,
                                 nthreads=8)


def run_apply(case: Case, layer=0, projs="qkvo", x=None, ys=None, seed_offset=0):
    """Run the fused apply; returns (x, ys_in, ys_out_f64)."""
    from paper_2311_03285_b200 import Batch
    cfg, T, h = case.cfg, case.batch.T, case.cfg.hidden
    if x is None:
        x = wl.activations(cfg, T, h, tag=100 + layer, seed_offset=seed_offset)
    if ys is None:
        ys = [wl.activations(cfg, T, h, tag=200 + 4 * layer + p, seed_offset=seed_offset) for p in range(4)]
    xd = to_device(x, cfg.dtype)
    yd = [to_device(y, cfg.dtype) for y in ys]
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter, stream=case.stream)
    b.apply(layer, projs, xd, h, yd, [h] * 4, stream=case.stream)
    case.pool.sync(case.stream)
    out = [from_device(t, cfg.dtype) for t in yd]
    b.close()
    return x, ys, out
