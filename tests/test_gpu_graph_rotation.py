"""Iteration-level batching: a CUDA graph captured for one decode
batch replays every later batch.  The MBGMV launches read their descriptors
through a per-(batch, call shape) header at a fixed device address that
slora_batch_prepare rewrites, so after prepare(B) a replay of the graph
captured on batch A computes batch B.  Checked against the oracle for several
re-sampled batches (different adapters, token counts, adapter-less tokens),
and bit-identical to eager launches of the same batch.  Mark: gpu.
"""
import numpy as np
import pytest

import oracle
from synth import workload as wl
from gpu_helpers import TOL, from_device, normalized_err, to_device

pytestmark = pytest.mark.gpu


def test_graph_replays_rotating_batches():
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    cfg = wl.CONFIGS["c2"]
    L, h, Tmax = 2, cfg.hidden, 64
    base = wl.make_batch(cfg)
    ads = list(base.unique)
    ranks = dict(base.ranks)
    need = sum(L * 8 * r for r in ranks.values())
    pool = Pool(h, L, need + 64, dtype=cfg.dtype, device=0, order="shuffle", seed=11, max_adapters=128)
    s = torch.cuda.Stream()
    weights = {}
    for a in ads:
        wts = [wl.adapter_weights(cfg, a, l, p, ranks[a]) for l in range(L) for p in range(4)]
        pool.adapter_load(a, ranks[a], np.concatenate([np.concatenate([A.ravel(), B.ravel()]) for A, B in wts]),
                          stream=s)
        weights[a] = wts
    td = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[cfg.dtype]
    X = torch.zeros((L, Tmax, h), dtype=td, device="cuda")
    Y = torch.zeros((L, 4, Tmax, h), dtype=td, device="cuda")
    b = Batch(pool)
    b.set_options(mbgmv_only=True)  # every batch on the MBGMV path: graph-stable launch set

    def layers():
        for l in range(L):
            b.apply(l, "qkv", X[l], h, [Y[l, p] for p in range(4)], [h] * 4, stream=torch.cuda.current_stream())
            b.apply(l, "o", X[l], h, [Y[l, p] for p in range(4)], [h] * 4, stream=torch.cuda.current_stream())

    rng = np.random.default_rng(7)
    pop = np.array([1.0 / (i + 1) for i in range(len(ads))])
    pop /= pop.sum()

    def draw(T):
        tok = rng.choice(ads, size=T, p=pop).astype(np.int64)
        tok[rng.random(T) < 0.1] = -1
        return tok

    with torch.cuda.stream(s):
        b.prepare(base.token_adapter, stream=s)
        layers()  # eager once: builds every call shape before capture
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            layers()
    for it, T in enumerate([64, 40, 64, 17]):
        tok = draw(T)
        xs = [wl.activations(cfg, T, h, tag=500 + 10 * it + l) for l in range(L)]
        ys = [[wl.activations(cfg, T, h, tag=600 + 40 * it + 4 * l + p) for p in range(4)] for l in range(L)]
        with torch.cuda.stream(s):
            b.prepare(tok, stream=s)
            assert b.info()["mbgmm_segments"] == 0
            for l in range(L):
                X[l, :T].copy_(to_device(xs[l], cfg.dtype))
                for p in range(4):
                    Y[l, p, :T].copy_(to_device(ys[l][p], cfg.dtype))
            g.replay()
            s.synchronize()
            got = Y.clone()
            # eager launches of the same batch: bit-identical
            for l in range(L):
                X[l, :T].copy_(to_device(xs[l], cfg.dtype))
                for p in range(4):
                    Y[l, p, :T].copy_(to_device(ys[l][p], cfg.dtype))
            layers()
            s.synchronize()
        assert torch.equal(got[:, :, :T], Y[:, :, :T]), f"batch {it}: graph replay != eager"
        uniq = sorted(set(int(a) for a in tok if a >= 0))
        slot = np.array([uniq.index(a) if a >= 0 else -1 for a in tok], np.int64)
        for l in range(L):
            for p in range(4):
                ref = oracle.lora_apply(oracle.to_f64(xs[l], cfg.dtype), oracle.to_f64(ys[l][p], cfg.dtype),
                                        [oracle.to_f64(weights[a][l * 4 + p][0], cfg.dtype) for a in uniq],
                                        [oracle.to_f64(weights[a][l * 4 + p][1], cfg.dtype) for a in uniq], slot,
                                        nthreads=8)
                err = normalized_err(from_device(got[l, p, :T], cfg.dtype), ref)
                assert err <= TOL[cfg.dtype], (it, l, p, err)
    b.close()
    pool.close()


def test_apply_many_equals_per_call_applies():
    """slora_lora_apply_many enqueues the same launches as one slora_lora_apply per call:
    bit-identical outputs; a bad call stops the list at its index."""
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    from paper_2311_03285_b200.slora import SloraError
    cfg = wl.CONFIGS["c1"]
    L, h = 3, cfg.hidden
    batch = wl.make_batch(cfg)
    need = sum(L * 8 * r for r in batch.ranks.values())
    pool = Pool(h, L, need + 16, dtype=cfg.dtype, device=0, max_adapters=128)
    s = torch.cuda.current_stream()
    for a in batch.unique:
        pool.adapter_load(a, batch.ranks[a], wl.adapter_host_buffer(cfg, a, L), stream=s)
    b = Batch(pool)
    b.prepare(batch.token_adapter, stream=s)
    T = batch.T
    td = torch.float16
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn((L, T, h), generator=g, device="cuda").to(td)
    Y0 = torch.randn((L, 4, T, h), generator=g, device="cuda").to(td)
    Y1 = Y0.clone()
    for l in range(L):
        b.apply(l, "qkv", X[l], h, [Y0[l, p] for p in range(4)], [h] * 4, stream=s)
        b.apply(l, "o", X[l], h, [Y0[l, p] for p in range(4)], [h] * 4, stream=s)
    calls = []
    for l in range(L):
        calls.append((l, "qkv", X[l], h, [Y1[l, p] for p in range(4)], [h] * 4))
        calls.append((l, "o", X[l], h, [Y1[l, p] for p in range(4)], [h] * 4))
    b.apply_many(Batch.make_calls(calls), stream=s)
    torch.cuda.synchronize()
    assert torch.equal(Y0, Y1)
    bad = Batch.make_calls(calls[:2] + [(L + 5, "q", X[0], h, [Y1[0, p] for p in range(4)], [h] * 4)])
    with pytest.raises(SloraError) as e:
        b.apply_many(bad, stream=s)
    assert e.value.name == "INVALID_ARG"
    b.close()
    pool.close()
