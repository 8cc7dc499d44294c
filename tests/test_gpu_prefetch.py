"""NEXT-1: asynchronous adapter loads on the pool's loader thread
and copy stream (slora_adapter_prefetch), checked end to end on the GPU.

* prefetched adapters (pageable numpy and page-locked torch buffers) used by a
  batch prepared at once (prepare fences the loads on its stream): parity with
  the oracle, and the stored pages equal the host rows bit-exactly;
* page-reuse fence: a kernel still queued behind a long sleep reads an
  adapter's pages while that adapter is evicted and another one is prefetched
  into the same pages -- the queued kernel must still see the old weights;
* evicting an adapter whose load is still in flight.
Mark: gpu.
"""
import numpy as np
import pytest

from synth import workload as wl
from gpu_helpers import TOL, from_device, normalized_err, to_device
import oracle

pytestmark = pytest.mark.gpu


def host_buffer(cfg, a, r, L, pinned=False):
    import torch
    wts = [wl.adapter_weights(cfg, a, l, p, r) for l in range(L) for p in range(4)]
    host = np.concatenate([np.concatenate([A.ravel(), B.ravel()]) for A, B in wts])
    if pinned:
        t = torch.from_numpy(host.view(np.int16) if cfg.dtype == "bf16" else host)
        host = t.pin_memory()
    return wts, host


def gather(pool, pages, like, s):
    """Stored rows of `pages` (whole pages) as an array shaped like `like`."""
    import torch
    dst = torch.empty(like.nbytes, dtype=torch.uint8, device="cuda")
    pool.gather_pages(pages, dst, stream=s)
    pool.sync(s)
    return dst.cpu().numpy().view(like.dtype).reshape(like.shape)


def oracle_proj(cfg, batch, weights, x, y, layer, proj):
    dt = cfg.dtype
    ids = batch.unique
    slot = np.array([ids.index(a) if a >= 0 else -1 for a in batch.token_adapter], np.int64)
    return oracle.lora_apply(oracle.to_f64(x, dt), oracle.to_f64(y, dt),
                             [oracle.to_f64(weights[a][layer * 4 + proj][0], dt) for a in ids],
                             [oracle.to_f64(weights[a][layer * 4 + proj][1], dt) for a in ids], slot, nthreads=8)


@pytest.mark.parametrize("pinned", [False, True])
def test_prefetch_then_prepare_parity(pinned):
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    cfg = wl.CONFIGS["c2"]
    L = 2
    batch = wl.make_batch(cfg)
    h = cfg.hidden
    need = sum(L * 8 * r for r in batch.ranks.values())
    pool = Pool(h, L, need + 64, dtype=cfg.dtype, device=0, order="shuffle", seed=5, max_adapters=128)
    s = torch.cuda.current_stream()
    weights = {}
    for a in batch.unique:
        wts, host = host_buffer(cfg, a, batch.ranks[a], L, pinned)
        pool.adapter_prefetch(a, batch.ranks[a], host)
        weights[a] = wts
    T = batch.T
    b = Batch(pool)
    b.prepare(batch.token_adapter, stream=s)  # fences the loads still in flight
    for layer in range(L):
        x = wl.activations(cfg, T, h, tag=300 + layer)
        ys = [wl.activations(cfg, T, h, tag=400 + 4 * layer + p) for p in range(4)]
        xd = to_device(x, cfg.dtype)
        yd = [to_device(y, cfg.dtype) for y in ys]
        b.apply(layer, "qkvo", xd, h, yd, [h] * 4, stream=s)
        pool.sync(s)
        for p in range(4):
            ref = oracle_proj(cfg, batch, weights, x, ys[p], layer, p)
            err = normalized_err(from_device(yd[p], cfg.dtype), ref)
            assert err <= TOL[cfg.dtype], (layer, p, err)
    for a in batch.unique:
        pool.adapter_wait(a)
        assert not pool.adapter_loading(a)
    st = pool.loader_stats()
    assert st["loads"] == len(batch.unique) and st["queued"] == 0
    assert st["direct_loads"] == (len(batch.unique) if pinned else 0)
    # stored rows == host rows (bit-exact): B rows of adapter 0, layer 1, proj o are whole pages
    a = batch.unique[0]
    r = batch.ranks[a]
    pages = pool.adapter_pages(a)
    per_tensor = r
    off = ((1 * 4 + 3) * 2 + 1) * per_tensor  # layer 1, proj o, tensor B (claim order)
    B = weights[a][1 * 4 + 3][1]
    assert np.array_equal(gather(pool, pages[off:off + r], B, s), B)
    b.close()
    pool.close()


def test_page_reuse_is_fenced_against_queued_kernels():
    """The queued apply reads adapter A's pages after a long sleep; A is evicted and B is
    prefetched into the freed pages (LIFO reuse) before the sleep ends.  The copy stream
    waits for the release, so the apply still sees A."""
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    cfg = wl.CONFIGS["c1"]
    h, L = cfg.hidden, 1
    r = 8
    pool = Pool(h, L, L * 8 * r * 2 + 8, dtype=cfg.dtype, device=0, max_adapters=8)
    s = torch.cuda.current_stream()
    wa, ha = host_buffer(cfg, 0, r, L)
    wb, hb = host_buffer(cfg, 1, r, L)
    pool.adapter_load(0, r, ha, stream=s)
    pages_a = pool.adapter_pages(0)
    T = 16
    tok = np.zeros(T, np.int64)
    x = wl.activations(cfg, T, h, tag=7)
    ys = [wl.activations(cfg, T, h, tag=8 + p) for p in range(4)]
    xd = to_device(x, cfg.dtype)
    yd = [to_device(y, cfg.dtype) for y in ys]
    b = Batch(pool)
    b.prepare(tok, stream=s)
    torch.cuda._sleep(200_000_000)  # ~100 ms of GPU time ahead of the apply
    b.apply(0, "qkvo", xd, h, yd, [h] * 4, stream=s)
    pool.adapter_evict(0, stream=s)
    pool.adapter_prefetch(1, r, hb)
    assert sorted(pool.adapter_pages(1)) == sorted(pages_a)  # the same pages, reused
    pool.sync(s)
    pool.adapter_wait(1)

    class One:
        unique = [0]
        token_adapter = tok
    for p in range(4):
        ref = oracle_proj(cfg, One, {0: wa}, x, ys[p], 0, p)
        assert normalized_err(from_device(yd[p], cfg.dtype), ref) <= TOL[cfg.dtype]
    b.close()
    pool.close()


def test_evict_while_loading_and_reload():
    import torch
    from paper_2311_03285_b200 import Pool
    cfg = wl.CONFIGS["c1"]
    h, L, r = cfg.hidden, 4, 16
    pool = Pool(h, L, L * 8 * r * 3 + 8, dtype=cfg.dtype, device=0, max_adapters=8)
    s = torch.cuda.current_stream()
    w, host = host_buffer(cfg, 3, r, L)
    for _ in range(3):
        pool.adapter_prefetch(3, r, host)
        pool.adapter_evict(3, stream=s)  # fences the load in flight, then releases
    pool.adapter_prefetch(3, r, host)
    pool.adapter_wait(3)
    pages = pool.adapter_pages(3)
    off = ((2 * 4 + 1) * 2 + 1) * r  # layer 2, proj k, tensor B
    B = w[2 * 4 + 1][1]
    assert np.array_equal(gather(pool, pages[off:off + r], B, s), B)
    assert pool.frag_report()["free_pages"] == pool.capacity - L * 8 * r
    pool.close()
