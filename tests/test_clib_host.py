"""CPU tests of the C-ABI library (no GPU, no compute calls): symbols, and the
C++ Unified Paging bookkeeping against the reference model in oracle/
(page ids bit-exact)."""
import re
import os

import numpy as np
import pytest

from oracle import pool_model as pm
from paper_2311_03285_b200 import slora as sl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "slora.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(slora_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = sl.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    assert L.slora_status_string(3) == b"SLORA_ERR_OUT_OF_PAGES"
    assert set(sl.SIGNATURES) <= set(names)


def mk(cap, hidden=8, L=2, tp=1, rank=0, order="ascending", seed=0, max_ad=64, dims=None):
    c = sl.Pool(hidden, L, cap, dtype="f16", device=-1, tp_size=tp, tp_rank=rank, order=order, seed=seed,
                max_adapters=max_ad, proj_dims=dims)
    m = pm.PoolModel(cap, hidden, L, tp_size=tp, tp_rank=rank, order=order, seed=seed, max_adapters=max_ad,
                     proj_dims=dims)
    return c, m


# NEXT-4 shapes at hidden 16: q, GQA k/v (16 -> 8), o, MLP gate/up (16 -> 40: 3 pages per B row),
# down (40 -> 16: 3 pages per stored A row)
MLP_DIMS = [(16, 16), (16, 8), (16, 8), (16, 16), (16, 40), (16, 40), (40, 16)]


def same_outcome(fc, fm):
    """Run the op on both; they must agree on success/error code and result."""
    rc = rm = None
    try:
        rc = fc()
    except sl.SloraError as e:
        rc = ("err", e.code)
    try:
        rm = fm()
    except pm.PoolError as e:
        rm = ("err", e.code)
    if isinstance(rc, np.ndarray):
        rc = rc.tolist()
    assert rc == rm, (rc, rm)
    return rc


def compare_state(c, m):
    rep = c.frag_report()
    mr = m.fragmentation_report()
    for k in ("used", "free", "largest_free_run", "kv_pages", "adapter_pages"):
        key = {"used": "used_pages", "free": "free_pages"}.get(k, k)
        assert rep[key] == mr[k], (k, rep, mr)
    for aid, ad in m.adapters.items():
        assert c.adapter_pages(aid).tolist() == ad.pages
    for rid, hd in m.kv.items():
        for l in range(m.L):
            for kind in range(2):
                assert c.kv_pages(rid, l, kind).tolist() == hd.pages[(l, kind)]


@pytest.mark.parametrize("order,tp,rank,dims", [("ascending", 1, 0, None), ("shuffle", 1, 0, None),
                                                ("shuffle", 4, 3, None), ("shuffle", 1, 0, MLP_DIMS)])
def test_pool_matches_model_random_ops(order, tp, rank, dims):
    c, m = mk(2500, hidden=16, L=2, tp=tp, rank=rank, order=order, seed=99, dims=dims)
    rng = np.random.default_rng(7)
    nid = 0
    for step in range(10_000):
        op = int(rng.integers(0, 8))
        if op == 0:
            n = int(rng.integers(0, 30))
            same_outcome(lambda: c.kv_alloc(nid, n), lambda: m.kv_alloc(nid, n))
            nid += 1
        elif op == 1:
            rid = int(rng.integers(0, max(nid, 1)))
            n = int(rng.integers(0, 4))
            same_outcome(lambda: c.kv_append(rid, n), lambda: m.kv_append(rid, n))
        elif op == 2:
            rid = int(rng.integers(0, max(nid, 1)))
            same_outcome(lambda: c.kv_free(rid), lambda: m.kv_free(rid))
        elif op == 3:
            r = int(rng.choice([4, 8, 16, 6]))
            aid = int(rng.integers(0, 40))
            same_outcome(lambda: c.adapter_load(aid, r), lambda: m.adapter_load(aid, r))
        elif op == 4:
            aid = int(rng.integers(0, 40))
            same_outcome(lambda: c.adapter_evict(aid), lambda: m.adapter_evict(aid))
        elif op == 5:
            aid = int(rng.integers(0, 40))
            same_outcome(lambda: c.pin(aid), lambda: m.pin(aid))
        elif op == 6:
            aid = int(rng.integers(0, 40))
            same_outcome(lambda: c.unpin(aid), lambda: m.unpin(aid))
        else:
            pages = rng.integers(0, 2500, size=3)
            try:
                m.check_gather(pages.tolist())
                want = sl.STATUS[15]  # valid pages: bookkeeping pool refuses the device copy
            except pm.PoolError as e:
                want = sl.STATUS[e.code]
            with pytest.raises(sl.SloraError) as ei:
                c.gather_pages(pages, 0)
            assert ei.value.name == want
        if step % 500 == 0:
            compare_state(c, m)
    compare_state(c, m)


def test_device_calls_refused_on_bookkeeping_pool():
    c, _ = mk(100)
    c.adapter_load(1, 4)
    b = sl.Batch(c)
    b.prepare(np.array([1, -1, 1, 1], np.int64))
    info = b.info()
    assert info["segments"] == 1 and info["adapted_tokens"] == 3 and info["sum_rank_tokens"] == 12
    with pytest.raises(sl.SloraError) as e:
        b.apply(0, "qkv", 0, 8, [0, 0, 0, 0], [8] * 4)
    assert e.value.name == "NO_DEVICE"
    with pytest.raises(sl.SloraError) as e:
        b.prepare(np.array([1, 5], np.int64))
    assert e.value.name == "NONRESIDENT_ADAPTER"
    assert b.v_elems("qkv", 1) == 36
    with pytest.raises(sl.SloraError) as e:
        c.adapter_load(2, 4, np.zeros(4, np.float16))
    assert e.value.name == "NO_DEVICE"


def test_batch_grouping_counts():
    c, _ = mk(100_000, hidden=64, L=1, max_ad=64)
    ranks = {a: [8, 16, 32, 64][a % 4] for a in range(20)}
    for a, r in ranks.items():
        c.adapter_load(a, r)
    rng = np.random.default_rng(1)
    tok = rng.integers(-1, 20, size=300)
    b = sl.Batch(c)
    b.prepare(tok)
    info = b.info()
    used = [int(a) for a in tok if a >= 0]
    assert info["T"] == 300
    assert info["adapted_tokens"] == len(used)
    assert info["segments"] == len(set(used))
    assert info["sum_rank_tokens"] == sum(ranks[a] for a in used)
    assert info["weight_bytes_per_proj"] == sum(ranks[a] * 2 * 64 * 2 for a in set(used))


def test_adapter_load_validates_host_buffer():
    """The binding checks the host buffer before the library reads from it
    (ADVICE r01): wrong element type or wrong size raise ValueError."""
    import paper_2311_03285_b200.slora as sl2
    p = sl2.Pool.__new__(sl2.Pool)  # a device pool's attributes without creating one
    p.dtype, p.num_layers, p.hidden, p.device, p.h = "f16", 1, 64, 0, None
    p.proj_dims = [(64, 64)] * 4
    good = np.zeros(1 * 4 * 2 * 64 * 4, np.float16)
    with pytest.raises(ValueError):
        p.adapter_load(1, 4, good.astype(np.float32))  # wider dtype
    with pytest.raises(ValueError):
        p.adapter_load(1, 4, good[:-1])                 # undersized


def test_tp_entry_points_refuse_without_device_or_communicator():
    """slora_tp_* on a bookkeeping pool: NO_DEVICE for init; the TP compute
    calls need a communicator first (INVALID_ARG), before any CUDA work."""
    c, _ = mk(1000, hidden=64, L=1, max_ad=8)
    with pytest.raises(sl.SloraError) as e:
        c.tp_init(bytes(128), 0, 1)
    assert e.value.name == "NO_DEVICE"
    c.adapter_load(1, 4)
    b = sl.Batch(c)
    b.prepare(np.array([1, 1], np.int64))
    with pytest.raises(sl.SloraError) as e:
        b.tp_qkv(0, 0, 64, [0, 0, 0], [64] * 3)
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(sl.SloraError) as e:
        b.tp_o(0, 0, 64, 0, 64)
    assert e.value.name == "INVALID_ARG"
    assert c.tp_stats()["allgather_calls"] == 0


def test_pool_destroy_detaches_live_batches():
    """Destroying a pool while a batch is alive leaves the batch a
    stale handle instead of a dangling pointer: prepare -> STALE_HANDLE, and
    destroying it afterwards is safe."""
    c, _ = mk(1000, hidden=64, L=1, max_ad=8)
    c.adapter_load(1, 4)
    b = sl.Batch(c)
    b.prepare(np.array([1, -1], np.int64))
    c.close()
    with pytest.raises(sl.SloraError) as e:
        b.prepare(np.array([1], np.int64))
    assert e.value.name == "STALE_HANDLE"
    b.close()


def test_prefetch_on_bookkeeping_pool():
    """slora_adapter_prefetch claims pages exactly like slora_adapter_load (same errors, same
    pop order); with no device there is nothing in flight: wait / query return at once."""
    a, b = mk(64)[0], mk(64)[0]
    a.adapter_load(1, 2)
    b.adapter_prefetch(1, 2, None)
    assert np.array_equal(a.adapter_pages(1), b.adapter_pages(1))
    b.adapter_wait(1)
    assert not b.adapter_loading(1)
    with pytest.raises(sl.SloraError) as e:
        b.adapter_prefetch(1, 2, None)
    assert e.value.name == "ALREADY_RESIDENT"
    with pytest.raises(sl.SloraError) as e:
        b.adapter_prefetch(2, 64, None)
    assert e.value.name == "OUT_OF_PAGES"
    with pytest.raises(sl.SloraError) as e:
        b.adapter_wait(9)
    assert e.value.name == "NOT_RESIDENT"
    assert b.loader_stats()["loads"] == 0


def test_projection_shapes_page_accounting():
    """NEXT-4 (reading R2): a stored row of n elements takes ceil(n / H) pages.  Square
    projections reduce to P:262 (a rank-R tensor takes R pages: 8R per layer for q,k,v,o);
    the C++ pool claims exactly the model's pages, in claim order layer, proj, tensor, row, chunk;
    TP with non-square projections and rows of more than 8 pages are refused."""
    H, L, r = 16, 3, 4
    c, m = mk(4096, hidden=H, L=L, dims=MLP_DIMS)
    want = L * r * sum(-(-i // H) + -(-o // H) for i, o in MLP_DIMS)
    assert m.adapter_page_count(r) == want == L * r * (2 + 2 + 2 + 2 + 4 + 4 + 4)
    c.adapter_load(5, r)
    m.adapter_load(5, r)
    assert c.adapter_pages(5).tolist() == m.adapters[5].pages
    assert len(m.adapters[5].pages) == want
    sq, msq = mk(4096, hidden=H, L=L)
    assert msq.adapter_page_count(r) == L * 8 * r
    with pytest.raises(sl.SloraError) as e:
        mk(64, hidden=H, L=1, tp=2, dims=MLP_DIMS)
    assert e.value.name == "SHAPE"
    with pytest.raises(sl.SloraError) as e:
        mk(64, hidden=H, L=1, dims=[(16, 16 * 9)])
    assert e.value.name == "SHAPE"
