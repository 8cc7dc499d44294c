"""GPU parity of gathered MBGMM: decode batches whose adapter segments hold
many scattered tokens (reading R9: dispatch by segment token count, not by
phase).  With no consecutive prefill runs, segments of >= 4 tokens and rank
>= 32 (when they hold at least half of the adapted tokens) go to the
tensor-core MBGMM kernels on x rows gathered into a contiguous workspace, y
written back through the token index; the rest of the batch stays on MBGMV.
Exact-integer inputs make the result bit-exact against the fp64 oracle; C4
shapes (h = 8192, bf16: 16-row shrink units over two 4096-column K parts)
are checked within tolerance.
Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, Case, normalized_err, run_apply
from test_gpu_parity import int_weights

pytestmark = pytest.mark.gpu


def _segments(case):
    from paper_2311_03285_b200 import Batch
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter, stream=case.stream)
    n = b.info()["mbgmm_segments"]
    b.close()
    return n


def decode_cfg(dtype, ranks, tokens=96, n_adapters=4, hidden=4096, idx=31):
    return wl.Config(f"gather-{dtype}", idx, hidden, n_adapters, ranks, dtype, 1.0, tokens, num_layers=1)


@pytest.mark.parametrize("dtype,ranks", [("f16", (64, 32, 16, 8)), ("bf16", (32, 32, 16, 8))])
def test_gathered_mbgmm_exact_integer_bit_exact(dtype, ranks):
    cfg = decode_cfg(dtype, ranks)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=9, weight_fn=int_weights(cfg), kv_interleave=2)
    assert _segments(case) >= 1, "segments of >= 4 scattered tokens must go to MBGMM"
    rng = np.random.default_rng(4)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-64, 65, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    x, ys, out = run_apply(case, x=x, ys=ys)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert np.array_equal(out[p], ref), f"proj {p}: max diff {np.abs(out[p] - ref).max()}"


def test_gathered_mbgmm_adapterless_rows_untouched():
    cfg = decode_cfg("f16", (64, 32), tokens=80, idx=32)
    batch = wl.make_batch(cfg)
    ta = batch.token_adapter.copy()
    ta[::5] = -1
    pb = wl.Batch(batch.requests, ta, batch.ranks)
    case = Case(cfg, pb)
    assert _segments(case) >= 1
    x, ys, out = run_apply(case)
    from oracle import to_f64
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert normalized_err(out[p], ref) <= TOL["f16"]
        none = ta == -1
        assert np.array_equal(out[p][none], to_f64(ys[p], "f16")[none])


def test_gathered_mbgmm_c4_shapes_bf16():
    """70B shapes on one GPU: h = 8192 (16-row shrink units over two 4096-column K parts), 10 rank-64
    adapters, 256 decode tokens, bf16."""
    cfg = wl.CONFIGS["c4"]
    cfg1 = wl.Config(cfg.name, cfg.index, cfg.hidden, cfg.n_adapters, cfg.rank_list, cfg.dtype, 1.0, 256,
                     num_layers=1)
    batch = wl.make_batch(cfg1)
    case = Case(cfg1, batch, order="shuffle", seed=2)
    assert _segments(case) >= 2
    x, ys, out = run_apply(case)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        err = normalized_err(out[p], ref)
        assert err <= TOL["bf16"], f"proj {p}: {err}"
