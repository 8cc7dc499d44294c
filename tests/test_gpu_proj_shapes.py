"""NEXT-4: LoRA on projections that are not hidden -> hidden (P:321-327 uses the
MLP as its worked example): the Llama-7B MLP (gate/up 4096 ->
11008, down 11008 -> 4096: stored rows spanning 3 pages, the last partly used)
and GQA-shaped k/v (4096 -> 1024: a B row is a quarter of a page), on the
fused MBGMV path.  Parity with the fp64 oracle (2e-2 normalized, fp16) and, in
the exact-integer regime, bit-exact.  Calls group projections that share x
(q,k,v | o | gate,up | down); a call mixing input widths is a SHAPE error.
Mark: gpu.
"""
import numpy as np
import pytest

import oracle
from synth import workload as wl
from gpu_helpers import TOL, from_device, normalized_err, to_device

pytestmark = pytest.mark.gpu

MLP7B = [(4096, 4096)] * 4 + [(4096, 11008), (4096, 11008), (11008, 4096)]
GQA = [(4096, 4096), (4096, 1024), (4096, 1024), (4096, 4096)]
CALLS_MLP = [(0, 1, 2), (3,), (4, 5), (6,)]
CALLS_GQA = [(0, 1, 2), (3,)]


def run_case(dims, calls, L=1, exact=False, seed=3, decode=48):
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    from paper_2311_03285_b200.slora import SloraError
    cfg = wl.Config("shapes", 9, 4096, 300, (64, 32, 16, 8), "f16", 1.0, decode, num_layers=L,
                    proj_dims=tuple(dims))
    batch = wl.make_batch(cfg)
    batch.token_adapter[::7] = -1  # some base-only tokens (reading R7)
    h = cfg.hidden
    need = sum(L * r * sum(-(-i // h) + -(-o // h) for i, o in dims) for r in batch.ranks.values())
    pool = Pool(h, L, need + 64, dtype="f16", device=0, order="shuffle", seed=seed, max_adapters=128,
                proj_dims=dims)
    s = torch.cuda.current_stream()
    W = {}
    ids = sorted(set(int(a) for a in batch.token_adapter if a >= 0))
    for a in ids:
        r = batch.ranks[a]
        wts = []
        for l in range(L):
            for p, (hi, do) in enumerate(dims):
                if exact:
                    rng = np.random.default_rng([a, l, p, 5])
                    A = wl.round_to(wl.integer_weights((hi, r), rng, -1, 1, max_nnz_per_col=4), "f16")
                    B = wl.round_to(wl.integer_weights((r, do), rng, -1, 1), "f16")
                else:
                    A, B = wl.adapter_weights(cfg, a, l, p, r)
                wts.append((A, B))
        pool.adapter_load(a, r, np.concatenate([np.concatenate([A.ravel(), B.ravel()]) for A, B in wts]), stream=s)
        W[a] = wts
    b = Batch(pool)
    b.prepare(batch.token_adapter, stream=s)
    T = batch.T
    slot = np.array([ids.index(a) if a >= 0 else -1 for a in batch.token_adapter], np.int64)
    rng = np.random.default_rng(17)
    for l in range(L):
        for call in calls:
            hin = dims[call[0]][0]
            if exact:
                x = wl.round_to(rng.integers(-1, 2, size=(T, hin)).astype(np.float32), "f16")
                ys = {p: np.zeros((T, dims[p][1]), np.float16) for p in call}
            else:
                x = wl.activations(cfg, T, hin, tag=900 + 10 * l + call[0])
                ys = {p: wl.activations(cfg, T, dims[p][1], tag=1000 + 10 * l + p) for p in call}
            xd = to_device(x, "f16")
            yd = [None] * len(dims)
            for p in call:
                yd[p] = to_device(ys[p], "f16")
            b.apply(l, list(call), xd, hin, yd, [dims[p][1] for p in range(len(dims))], stream=s)
            pool.sync(s)
            for p in call:
                ref = oracle.lora_apply(oracle.to_f64(x, "f16"), oracle.to_f64(ys[p], "f16"),
                                        [oracle.to_f64(W[a][l * len(dims) + p][0], "f16") for a in ids],
                                        [oracle.to_f64(W[a][l * len(dims) + p][1], "f16") for a in ids], slot,
                                        nthreads=8)
                got = from_device(yd[p], "f16")
                if exact:
                    assert np.array_equal(got, ref), (l, p, np.abs(got - ref).max())
                else:
                    assert normalized_err(got, ref) <= TOL["f16"], (l, p, normalized_err(got, ref))
                none = batch.token_adapter < 0
                assert np.array_equal(got[none], oracle.to_f64(ys[p], "f16")[none])
    if len(dims) > 4:  # a call whose projections read different x widths
        x = torch.zeros((T, 11008), dtype=torch.float16, device="cuda")
        y = [torch.zeros((T, max(d)), dtype=torch.float16, device="cuda") for d in dims]
        with pytest.raises(SloraError) as e:
            b.apply(0, [0, 6], x, 11008, y, [max(d) for d in dims], stream=s)
        assert e.value.name == "SHAPE"
    b.close()
    pool.close()


def test_llama7b_mlp_parity():
    run_case(MLP7B, CALLS_MLP, L=2)


def test_llama7b_mlp_exact_integer_bit_exact():
    run_case(MLP7B, CALLS_MLP, L=1, exact=True, seed=8)


def test_gqa_kv_parity_and_exact():
    run_case(GQA, CALLS_GQA, L=2)
    run_case(GQA, CALLS_GQA, L=1, exact=True, seed=9)
