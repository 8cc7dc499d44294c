"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star): normalized max-abs error
max|g - o| / max|o| <= 1e-5 (fp32) and 2e-2 (fp16 / bf16); bookkeeping and
the exact-integer regime bit-exact.  Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, Case, from_device, normalized_err, run_apply, to_device

pytestmark = pytest.mark.gpu


def check_all(case, x, ys, out, projs=range(4), layer=0):
    tol = TOL[case.cfg.dtype]
    for p in projs:
        ref = case.oracle_proj(x, ys[p], layer, p)
        err = normalized_err(out[p], ref)
        assert err <= tol, f"proj {p}: err {err} > {tol}"
        # rows without an adapter are byte-identical (reading R7)
        none = case.batch.token_adapter < 0
        if none.any():
            from oracle import to_f64
            assert np.array_equal(out[p][none], to_f64(ys[p], case.cfg.dtype)[none])


# ------------------------------------------------------------------- C0
def test_c0_tiny_fp32_all_projections():
    cfg = wl.CONFIGS["c0"]
    case = Case(cfg, wl.make_batch(cfg), order="shuffle", seed=3, kv_interleave=2)
    x, ys, out = run_apply(case)
    check_all(case, x, ys, out)


def test_c0_adapterless_requests_and_scale():
    cfg = wl.CONFIGS["c0"]
    batch = wl.make_batch(cfg)
    batch.token_adapter[5] = -1            # request 1 has no adapter
    batch.ranks.pop(1)
    case = Case(cfg, batch, scale={0: 0.5, 2: 2.0, 3: 1.25})
    x, ys, out = run_apply(case)
    check_all(case, x, ys, out)


@pytest.mark.parametrize("projs", ["q", "kv", "o", "qkv"])
def test_c0_projection_masks(projs):
    cfg = wl.CONFIGS["c0"]
    case = Case(cfg, wl.make_batch(cfg))
    x, ys, out = run_apply(case, projs=projs)
    bits = [i for i, c in enumerate("qkvo") if c in projs]
    check_all(case, x, ys, out, projs=bits)
    from oracle import to_f64
    for p in range(4):
        if p not in bits:
            assert np.array_equal(out[p], to_f64(ys[p], cfg.dtype))


# ------------------------------------------------- exact-integer regime (G2)
def int_weights(cfg):
    def fn(a, l, p, r):
        rng = np.random.default_rng([a, l, p, 5])
        A = wl.integer_weights((cfg.hidden, r), rng, -1, 1, max_nnz_per_col=4)
        B = wl.integer_weights((r, cfg.hidden), rng, -1, 1)
        return wl.round_to(A, cfg.dtype), wl.round_to(B, cfg.dtype)
    return fn


@pytest.mark.parametrize("dtype,hidden,ranks", [("f32", 256, (4, 8)), ("f16", 4096, (64, 32, 16, 8)),
                                                ("bf16", 4096, (32, 16, 8))])
def test_exact_integer_regime_bit_exact(dtype, hidden, ranks):
    """Integer inputs with |v| <= 4 and |y| <= 4r + 64: fp32 accumulation is
    exact in any order, so the GPU must equal the oracle BIT-exactly."""
    cfg = wl.Config(f"int-{dtype}", 9, hidden, 40, ranks, dtype, 1.0, 48, num_layers=1)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=11, weight_fn=int_weights(cfg), kv_interleave=1)
    rng = np.random.default_rng(1)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-64, 65, size=(batch.T, hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    x, ys, out = run_apply(case, x=x, ys=ys)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert np.array_equal(out[p], ref), f"proj {p}: max diff {np.abs(out[p] - ref).max()}"


# ------------------------------------------- placement / permutation (G3, G4)
def test_page_placement_invariance_bit_identical():
    cfg = wl.CONFIGS["c2"]
    cfg = wl.Config(cfg.name, cfg.index, cfg.hidden, cfg.n_adapters, cfg.rank_list, cfg.dtype, 1.0, 64,
                    num_layers=2)
    batch = wl.make_batch(cfg)
    outs = []
    for order, seed, kv in [("ascending", 0, 0), ("shuffle", 1, 3), ("shuffle", 2, 1), ("shuffle", 3, 7)]:
        case = Case(cfg, batch, num_layers=2, order=order, seed=seed, kv_interleave=kv)
        x, ys, out = run_apply(case, layer=1)
        outs.append(out)
        case.pool.close()
    for o in outs[1:]:
        for p in range(4):
            assert np.array_equal(o[p], outs[0][p])


def test_batch_permutation_invariance_bit_identical():
    cfg = wl.CONFIGS["c2"]
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch)
    x, ys, out = run_apply(case)
    perm = np.random.default_rng(4).permutation(batch.T)
    pb = wl.Batch(batch.requests, batch.token_adapter[perm], batch.ranks)
    case.batch = pb
    _, _, outp = run_apply(case, x=x[perm], ys=[y[perm] for y in ys])
    for p in range(4):
        assert np.array_equal(outp[p], out[p][perm])


# ----------------------------------------------- library special case (G5)
def test_single_adapter_matches_cublas():
    import torch
    cfg = wl.CONFIGS["c1"]
    batch = wl.Batch([(3, 32)], np.full(32, 3, np.int64), {3: 8})
    case = Case(cfg, batch)
    x, ys, out = run_apply(case, projs="q")
    A, B = case.weights[3][0]
    xt = to_device(x, "f16").float()
    ref = to_device(ys[0], "f16").float() + (xt @ to_device(A, "f16").float()) @ to_device(B, "f16").float()
    err = normalized_err(out[0], ref.double().cpu().numpy())
    assert err <= 2e-2


# ------------------------------------------------------- bookkeeping (G6)
def test_gather_round_trip_bit_exact():
    import torch
    cfg = wl.CONFIGS["c2"]
    batch = wl.Batch([(0, 1), (3, 1)], np.array([0, 3]), {0: 64, 3: 8})
    case = Case(cfg, batch, num_layers=2, order="shuffle", seed=5, kv_interleave=2)
    for a in (0, 3):
        pages = case.pool.adapter_pages(a)
        r = batch.ranks[a]
        dst = torch.empty((len(pages), cfg.hidden), dtype=torch.float16, device="cuda")
        case.pool.gather_pages(pages, dst)
        case.pool.sync()
        got = dst.cpu().numpy()
        i = 0
        for l in range(2):
            for p in range(4):
                A, B = case.weights[a][l * 4 + p]
                assert np.array_equal(got[i:i + r], A.T), (a, l, p, "A")
                i += r
                assert np.array_equal(got[i:i + r], B), (a, l, p, "B")
                i += r
    from paper_2311_03285_b200 import SloraError
    free = sorted(set(range(case.pool.capacity)) - set(np.concatenate(
        [case.pool.adapter_pages(0), case.pool.adapter_pages(3)]).tolist()) - set(
        np.concatenate([case.pool.kv_pages(r, l, k) for r in (10000, 10001, 10002) for l in range(2)
                        for k in range(2)]).tolist()))
    with pytest.raises(SloraError) as e:
        case.pool.gather_pages([free[0]], dst)
    assert e.value.name == "FREE_PAGE_READ"


def test_stale_batch_after_evict_and_empty_batch():
    from paper_2311_03285_b200 import Batch, SloraError
    cfg = wl.CONFIGS["c0"]
    case = Case(cfg, wl.make_batch(cfg))
    b = Batch(case.pool)
    b.prepare(case.batch.token_adapter)
    case.pool.adapter_evict(3)
    x = to_device(wl.activations(cfg, 16, 256, 1), "f32")
    with pytest.raises(SloraError) as e:
        b.apply(0, "q", x, 256, [x, x, x, x], [256] * 4)
    assert e.value.name == "STALE_HANDLE"
    b.prepare(np.full(16, -1))
    y = x.clone()
    b.apply(0, "qkvo", x, 256, [y] * 4, [256] * 4)
    case.pool.sync()
    assert torch_equal(y, x)
    b.prepare(np.zeros(0, np.int64))
    b.apply(0, "q", x, 256, [y] * 4, [256] * 4)


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


# ------------------------------------------------------ full-size configs
@pytest.mark.parametrize("name", ["c1", "c2", "c2-mixed"])
def test_full_size_layer_parity(name):
    cfg = wl.CONFIGS[name]
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, num_layers=2, order="shuffle", seed=1, kv_interleave=4)
    x, ys, out = run_apply(case, layer=1)
    check_all(case, x, ys, out, layer=1)


def test_bf16_70b_shapes_single_gpu():
    cfg = wl.CONFIGS["c4"]
    cfg1 = wl.Config(cfg.name, cfg.index, cfg.hidden, cfg.n_adapters, cfg.rank_list, cfg.dtype, 1.0, 256,
                     num_layers=1)
    batch = wl.make_batch(cfg1)
    case = Case(cfg1, batch)
    x, ys, out = run_apply(case)
    check_all(case, x, ys, out)


# ------------------------------------------------ degenerate / ragged ranks
@pytest.mark.parametrize("dtype,hidden", [("f32", 512), ("f16", 4096), ("bf16", 5120)])
def test_odd_ranks_bit_exact(dtype, hidden):
    """Ranks that are not multiples of the 8-row shrink piece or the 4-row expand unroll (1, 3, 5,
    7, 9, 33, 63): the ragged tails of both phases, bit-exact in the integer regime."""
    ranks = (1, 3, 5, 7, 9, 33, 63)
    cfg = wl.Config(f"odd-{dtype}", 12, hidden, 14, ranks, dtype, None, 40, num_layers=1)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=21, weight_fn=int_weights(cfg), kv_interleave=1)
    rng = np.random.default_rng(3)
    x = wl.round_to(rng.integers(-1, 2, size=(batch.T, hidden)).astype(np.float32), dtype)
    ys = [wl.round_to(rng.integers(-32, 33, size=(batch.T, hidden)).astype(np.float32), dtype)
          for _ in range(4)]
    x, ys, out = run_apply(case, x=x, ys=ys)
    for p in range(4):
        ref = case.oracle_proj(x, ys[p], 0, p)
        assert np.array_equal(out[p], ref), f"proj {p}: max diff {np.abs(out[p] - ref).max()}"


def test_single_token_single_adapter_and_all_tokens_one_adapter():
    """Degenerate batches: one token; and every token on one rank-64 adapter (one segment of 64
    scattered decode tokens: the gathered-MBGMM route)."""
    from oracle import to_f64
    cfg = wl.Config("one", 13, 4096, 1, (64,), "f16", None, 1, num_layers=1)
    batch = wl.make_batch(cfg)
    case = Case(cfg, batch, order="shuffle", seed=2)
    x, ys, out = run_apply(case)
    check_all(case, x, ys, out)
    cfg = wl.Config("all-one", 14, 4096, 1, (64,), "f16", None, 64, num_layers=1)
    batch = wl.make_batch(cfg)
    assert len(batch.ranks) == 1
    case = Case(cfg, batch, order="shuffle", seed=2)
    x, ys, out = run_apply(case)
    check_all(case, x, ys, out)
