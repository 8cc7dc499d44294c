"""Next-call L2 prefetch hints (slora_lora_prefetch_next) never change results.

The hint makes the ring kernel pull the pages of the following call into L2
while it runs; outputs must be bit-identical to the un-hinted sequence and
within tolerance of the oracle (C2 decode batch, two layers, shuffled pages
interleaved with KV pages; the layer-0 o call prefetches layer 1's q/k/v).
Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, Case, from_device, normalized_err, to_device

pytestmark = pytest.mark.gpu


def _run_layers(case, hints):
    from paper_2311_03285_b200 import Batch
    cfg, T, h = case.cfg, case.batch.T, case.cfg.hidden
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter, stream=case.stream)
    outs, inputs = [], []
    for l in range(case.L):
        x = wl.activations(cfg, T, h, tag=100 + l)
        ys = [wl.activations(cfg, T, h, tag=200 + 4 * l + p) for p in range(4)]
        xd = to_device(x, cfg.dtype)
        yd = [to_device(y, cfg.dtype) for y in ys]
        if hints:
            b.prefetch_next(l, "o")
        b.apply(l, "qkv", xd, h, yd, [h] * 4, stream=case.stream)
        if hints and l + 1 < case.L:
            b.prefetch_next(l + 1, "qkv")
        b.apply(l, "o", xd, h, yd, [h] * 4, stream=case.stream)
        case.pool.sync(case.stream)
        outs.append([from_device(t, cfg.dtype) for t in yd])
        inputs.append((x, ys))
    b.close()
    return inputs, outs


@pytest.mark.parametrize("name", ["c2", "c1"])
def test_prefetch_hints_bit_identical_and_in_tolerance(name):
    cfg = wl.CONFIGS[name]
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, num_layers=2, order="shuffle", seed=3, kv_interleave=4)
    _, plain = _run_layers(case, hints=False)
    inputs, hinted = _run_layers(case, hints=True)
    for l in range(case.L):
        for p in range(4):
            assert np.array_equal(plain[l][p], hinted[l][p]), (l, p)
    x, ys = inputs[1]
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 1, p)
        assert normalized_err(hinted[1][p], ref) <= TOL[cfg.dtype]


def test_prefetch_hint_argument_errors():
    from paper_2311_03285_b200 import Batch, SloraError
    cfg = wl.CONFIGS["c0"]
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, num_layers=1)
    b = Batch(case.pool)
    b.prepare(batch.token_adapter, stream=case.stream)
    with pytest.raises(SloraError):
        b.prefetch_next(1, "qkv")   # layer out of range
    b.prefetch_next(0, 0)           # clears
    b.close()
