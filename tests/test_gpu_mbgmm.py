"""GPU parity of the tensor-core MBGMM path (long prefill runs, PAPER.md
Sec. 5.3) against the fp64 oracle.

Runs of >= 32 consecutive tokens of one adapter go to mbgmm_shrink/expand;
the rest of the batch to MBGMV in the same call.  Exact-integer inputs make
every fp32 accumulation exact, so the mixed call must equal the oracle
bit-exactly (this also pins the v = hi + lo split of the expand: integer v
has lo = 0).  Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, Case, normalized_err, run_apply
from test_gpu_parity import int_weights

pytestmark = pytest.mark.gpu


def mixed_cfg(dtype, ranks, prefill=(33, 150), n_pre=5, n_dec=20, hidden=4096, idx=21):
    return wl.Config(f"mbgmm-{dtype}", idx, hidden, 40, ranks, dtype, 1.0, n_dec, prefill_requests=n_pre,
                     prefill_range=prefill, num_layers=1)


def _runs(case):
    from paper_2311_03285_b200 import Batch
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter, stream=case.stream)
    n = b.info()["mbgmm_segments"]
    b.close()
    return n


@pytest.mark.parametrize("dtype,ranks", [("f16", (64, 32, 16, 8)), ("bf16", (32, 16, 8, 24))])
def test_mbgmm_exact_integer_bit_exact(dtype, ranks):
    cfg = mixed_cfg(dtype, ranks)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=5, weight_fn=int_weights(cfg), kv_interleave=2)
    assert _runs(case) >= 3, "the batch must route prefill runs to MBGMM"
    rng = np.random.default_rng(2)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-64, 65, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    x, ys, out = run_apply(case, x=x, ys=ys)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert np.array_equal(out[p], ref), f"proj {p}: max diff {np.abs(out[p] - ref).max()}"


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_mbgmm_random_within_tolerance(dtype):
    """Seeded N(0,1) activations, A ~ N(0,1/h), B ~ N(0,1/r); ragged tiles
    (run lengths not multiples of 64) and every rank of the C2 list."""
    cfg = mixed_cfg(dtype, (64, 32, 16, 8), prefill=(40, 200), n_pre=6, n_dec=10, idx=22)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=3, kv_interleave=1)
    assert _runs(case) >= 3
    x, ys, out = run_apply(case)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        err = normalized_err(out[p], ref)
        assert err <= TOL[dtype], f"proj {p}: {err}"


def test_mbgmm_rows_outside_runs_untouched_and_adapterless():
    """A run next to adapter-less tokens: their y rows stay bit-identical."""
    cfg = mixed_cfg("f16", (16, 8), n_pre=3, n_dec=8, idx=23)
    batch = wl.make_batch(cfg)
    ta = batch.token_adapter.copy()
    ta[::7] = -1   # breaks some runs, leaves the others >= 32
    pb = wl.Batch(batch.requests, ta, batch.ranks)
    case = Case(cfg, pb)
    x, ys, out = run_apply(case)
    from oracle import to_f64
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert normalized_err(out[p], ref) <= TOL["f16"]
        none = ta == -1
        assert np.array_equal(out[p][none], to_f64(ys[p], "f16")[none])
