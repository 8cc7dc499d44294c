"""GPU: the tensor-parallel path behind the C ABI (slora_tp_init /
slora_tp_lora_qkv / slora_tp_lora_o, include/slora.h a6/a8) with the
library's own NCCL communicator.  One GPU holds a one-rank communicator
(NCCL refuses two ranks on one device), so this checks the library's
sequence shrink -> ncclAllGather -> expand and shrink -> ncclAllReduce ->
expand-into-the-base-slice against the fp64 oracle (bit-exact in the exact
integer regime, within tolerance on the synthetic values), CUDA-graph
capture of it, and the exchange counters (zero sent for N = 1; counts taken
from the NCCL arguments).  The N > 1 exchange math is covered by the
oracle's TP emulation (O8) and the world-size-2 gloo test.  Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, Case, from_device, normalized_err, to_device
from test_gpu_parity import int_weights

pytestmark = pytest.mark.gpu


def _run(case, x, ys, graph=False):
    import torch
    from paper_2311_03285_b200 import Batch
    from paper_2311_03285_b200.tp import LibraryTP
    cfg, h = case.cfg, case.cfg.hidden
    tp = LibraryTP(case.pool)
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter, stream=case.stream)  # after tp_init: sizes the exchange buffers
    xd = to_device(x, cfg.dtype)
    yd = [to_device(y, cfg.dtype) for y in ys]
    if graph:
        y0 = [t.clone() for t in yd]
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=s):
            tp.qkv(b, 0, xd, h, yd[:3], [h] * 3, stream=torch.cuda.current_stream())
            tp.o(b, 0, xd, h, yd[3], h, stream=torch.cuda.current_stream())
        for t, t0 in zip(yd, y0):  # capture ran nothing: restore and replay once
            t.copy_(t0)
        g.replay()
    else:
        tp.qkv(b, 0, xd, h, yd[:3], [h] * 3, stream=case.stream)
        tp.o(b, 0, xd, h, yd[3], h, stream=case.stream)
    case.pool.sync(case.stream)
    torch.cuda.synchronize()
    st = tp.stats()
    b.close()
    return [from_device(t, cfg.dtype) for t in yd], st


@pytest.mark.parametrize("dtype,ranks", [("f16", (64, 32, 16, 8)), ("bf16", (32, 16, 8))])
def test_tp_cabi_one_rank_exact_integer(dtype, ranks):
    cfg = wl.Config(f"tp-int-{dtype}", 41, 4096, 24, ranks, dtype, 1.0, 40, num_layers=1)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=6, weight_fn=int_weights(cfg), kv_interleave=1)
    rng = np.random.default_rng(2)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-64, 65, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    out, st = _run(case, x, ys)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert np.array_equal(out[p], ref), f"proj {p}: max diff {np.abs(out[p] - ref).max()}"
    NR = sum(batch.ranks[a] for a in batch.token_adapter if a >= 0)
    assert st["allgather_calls"] == 1 and st["allreduce_calls"] == 1
    assert st["allreduce_count"] == NR  # the o partial: NR fp32 elements
    assert st["allgather_send_elems"] == 0 and st["allreduce_send_elems"] == 0  # N = 1: nothing crosses a link


def test_tp_cabi_one_rank_graph_capture_c2_tolerance():
    cfg0 = wl.CONFIGS["c2"]
    cfg = wl.Config(cfg0.name, cfg0.index, cfg0.hidden, cfg0.n_adapters, cfg0.rank_list, cfg0.dtype, 1.0, 64,
                    num_layers=1)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=8)
    x = wl.activations(cfg, batch.T, cfg.hidden, tag=100)
    ys = [wl.activations(cfg, batch.T, cfg.hidden, tag=200 + p) for p in range(4)]
    out, st = _run(case, x, ys, graph=True)
    for p in range(4):
        err = normalized_err(out[p], case.oracle_proj(x, ys[p], 0, p))
        assert err <= TOL["f16"], (p, err)
