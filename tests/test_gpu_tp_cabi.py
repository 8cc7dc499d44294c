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


def _run(case, x, ys, graph=False, p2p=False):
    import torch
    from paper_2311_03285_b200 import Batch
    from paper_2311_03285_b200.tp import LibraryTP
    cfg, h = case.cfg, case.cfg.hidden
    tp = LibraryTP(case.pool)
    if p2p:
        tp.enable_p2p()
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


@pytest.mark.parametrize("dtype,ranks", [("f16", (64, 32, 16, 8)), ("bf16", (32, 16, 8))])
def test_tp_device_initiated_one_rank_equals_nccl_path(dtype, ranks):
    """NEXT-3: slora_tp_fused_qkv / _o (shrink -> peer stores of v into every rank's exchange region
    + system-scope counter release -> expand, one kernel per call) with one rank: bit-identical to the
    NCCL path and, in the exact-integer regime, to the oracle; CUDA-graph capturable."""
    cfg = wl.Config(f"tp-p2p-{dtype}", 43, 4096, 24, ranks, dtype, 1.0, 40, num_layers=1)
    batch = wl.make_batch(cfg)
    rng = np.random.default_rng(4)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-64, 65, size=(batch.T, cfg.hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    case = Case(cfg, batch, order="shuffle", seed=6, weight_fn=int_weights(cfg), kv_interleave=1)
    ref_out, _ = _run(case, x, ys)
    case2 = Case(cfg, batch, order="shuffle", seed=6, weight_fn=int_weights(cfg), kv_interleave=1)
    out, st = _run(case2, x, ys, p2p=True)
    for p in range(4):
        assert np.array_equal(out[p], ref_out[p]), f"proj {p}"
        assert np.array_equal(out[p], case.oracle_proj(x, ys[p], 0, p)), f"proj {p} vs oracle"
    assert st["allgather_calls"] == 0 and st["allreduce_calls"] == 0  # no NCCL on the fused path
    case3 = Case(cfg, batch, order="shuffle", seed=6, weight_fn=int_weights(cfg), kv_interleave=1)
    out_g, _ = _run(case3, x, ys, graph=True, p2p=True)
    for p in range(4):
        assert np.array_equal(out_g[p], ref_out[p]), f"graph proj {p}"


def test_tp_device_initiated_on_a_batch_the_single_gpu_path_routes_to_mbgmm():
    """Regression: a decode batch whose rank-64 segments hold most tokens is routed to gathered
    MBGMM by the single-GPU fused call; the device-initiated TP calls are one MBGMV kernel each,
    so every segment must stay on MBGMV there (bit-identical to the NCCL path)."""
    cfg = wl.Config("tp-p2p-gather", 44, 4096, 24, (64, 32, 16, 8), "f16", 1.0, 40, num_layers=1)
    batch = wl.make_batch(cfg)
    x = wl.activations(cfg, batch.T, cfg.hidden, tag=100)
    ys = [wl.activations(cfg, batch.T, cfg.hidden, tag=200 + p) for p in range(4)]
    ref, _ = _run(Case(cfg, batch, order="shuffle", seed=8), x, ys)
    out, _ = _run(Case(cfg, batch, order="shuffle", seed=8), x, ys, p2p=True)
    for p in range(4):
        assert np.array_equal(out[p], ref[p]), f"proj {p}"
