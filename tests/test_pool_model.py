"""Pins for the Unified Paging reference model (oracle/pool_model.py) against
what the paper fixes and the invariants of paging.
P:L = /root/reference/PAPER.md line L (documentation only)."""
import json
import os

import numpy as np
import pytest

from oracle import pool_model as pm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_page_counts_from_paper():
    g = GOLD["kv_pages"]
    p = pm.PoolModel(100, hidden=8, num_layers=g["layers"])
    pages = p.kv_alloc(1, g["seq_len"])
    # K and V are two (S, H) tensors (reading R11): S pages each
    assert len(pages) == 2 * g["pages_per_tensor"]
    for kind in range(2):
        assert len(p.kv[1].pages[(0, kind)]) == g["seq_len"]
    g = GOLD["lora_pages_adapter"]
    p = pm.PoolModel(1000, hidden=8, num_layers=g["layers"])
    p.adapter_load(5, g["rank"])
    assert p.used_pages == g["pages"]
    g = GOLD["lora_pages_single_tensor"]
    p = pm.PoolModel(10_000, hidden=64, num_layers=1)
    p.adapter_load(0, g["rank"])
    ad = p.adapters[0]
    per_tensor = [o for o in (p.owner[q] for q in ad.pages) if o[3] == 0 and o[4] == 0]
    assert len(per_tensor) == g["pages"]


@pytest.mark.parametrize("N", [2, 4, 8])
def test_tp_pages_per_tensor(N):
    """Under TP each LoRA tensor shard still takes r pages of H/N (R3)."""
    p = pm.PoolModel(100_000, hidden=64, num_layers=2, tp_size=N, tp_rank=N - 1)
    assert p.page_elems == 64 // N
    p.adapter_load(0, 16)
    assert p.used_pages == 2 * 4 * 2 * 16
    with pytest.raises(pm.PoolError) as e:
        p.adapter_load(1, 6 if N != 2 else 3)
    assert e.value.code == pm.ERR_INDIVISIBLE


def test_allocation_order():
    p = pm.PoolModel(10, hidden=4, num_layers=1)
    assert p.kv_alloc(1, 2) == [0, 1, 2, 3]
    p.kv_alloc(2, 1)
    assert p.kv_free(1) == 4
    # LIFO: released pages come back in reverse release order
    assert p.kv_alloc(3, 1) == [3, 2]
    s = pm.initial_free_stack(50, "shuffle", 1234)
    assert sorted(s) == list(range(50)) and s != list(range(49, -1, -1))


def test_errors_leave_state_unchanged():
    p = pm.PoolModel(20, hidden=4, num_layers=1)
    p.kv_alloc(1, 3)
    snap = (list(p.free), list(p.owner))
    for fn, code in [(lambda: p.kv_alloc(2, 8), pm.ERR_OUT_OF_PAGES),   # needs 16, 14 free
                     (lambda: p.kv_alloc(1, 1), pm.ERR_INVALID_ARG),
                     (lambda: p.kv_append(9, 1), pm.ERR_STALE_HANDLE),
                     (lambda: p.adapter_evict(3), pm.ERR_NOT_RESIDENT),
                     (lambda: p.pin(3), pm.ERR_NOT_RESIDENT),
                     (lambda: p.adapter_load(0, 2), pm.ERR_OUT_OF_PAGES),  # needs 16
                     (lambda: p.check_gather([19]), pm.ERR_FREE_PAGE_READ)]:
        with pytest.raises(pm.PoolError) as e:
            fn()
        assert e.value.code == code
        assert (list(p.free), list(p.owner)) == snap
    assert p.kv_free(1) == 6
    with pytest.raises(pm.PoolError) as e:
        p.kv_free(1)
    assert e.value.code == pm.ERR_STALE_HANDLE
    p.adapter_load(7, 1)
    with pytest.raises(pm.PoolError) as e:
        p.adapter_load(7, 1)
    assert e.value.code == pm.ERR_ALREADY_RESIDENT
    p.pin(7)
    with pytest.raises(pm.PoolError) as e:
        p.adapter_evict(7)
    assert e.value.code == pm.ERR_PINNED
    p.unpin(7)
    with pytest.raises(pm.PoolError) as e:
        p.unpin(7)
    assert e.value.code == pm.ERR_NOT_PINNED
    assert p.adapter_evict(7) == 8


def test_random_ops_conservation_and_zero_external_fragmentation():
    """10^4 random ops: conservation, no double ownership, and an
    allocation of k pages succeeds iff free >= k regardless of layout."""
    rng = np.random.default_rng(0)
    p = pm.PoolModel(3000, hidden=8, num_layers=2, order="shuffle", seed=42)
    live_kv, live_ad = [], []
    nid = 0
    for _ in range(10_000):
        op = rng.integers(0, 6)
        try:
            if op == 0:
                n = int(rng.integers(0, 40))
                ok = 2 * 2 * n <= p.free_pages
                try:
                    p.kv_alloc(nid, n); live_kv.append(nid); assert ok
                except pm.PoolError as e:
                    assert not ok and e.code == pm.ERR_OUT_OF_PAGES
                nid += 1
            elif op == 1 and live_kv:
                rid = live_kv[int(rng.integers(len(live_kv)))]
                n = int(rng.integers(1, 5))
                ok = 2 * 2 * n <= p.free_pages
                try:
                    p.kv_append(rid, n); assert ok
                except pm.PoolError as e:
                    assert not ok and e.code == pm.ERR_OUT_OF_PAGES
            elif op == 2 and live_kv:
                rid = live_kv.pop(int(rng.integers(len(live_kv))))
                p.kv_free(rid)
            elif op == 3:
                r = int(rng.choice([4, 8, 16]))
                need = p.adapter_page_count(r)
                ok = need <= p.free_pages
                try:
                    p.adapter_load(nid, r); live_ad.append(nid); assert ok
                except pm.PoolError as e:
                    assert not ok and e.code == pm.ERR_OUT_OF_PAGES
                nid += 1
            elif op == 4 and live_ad:
                aid = live_ad[int(rng.integers(len(live_ad)))]
                if p.adapters[aid].pinned:
                    p.unpin(aid)
                else:
                    p.pin(aid)
            elif op == 5 and live_ad:
                aid = live_ad[int(rng.integers(len(live_ad)))]
                if p.adapters[aid].pinned:
                    with pytest.raises(pm.PoolError):
                        p.adapter_evict(aid)
                else:
                    p.adapter_evict(aid); live_ad.remove(aid)
        finally:
            p.audit()


def test_checkerboard_contrast():
    """Checkerboard free pattern: largest free run is 1, yet any k <= free
    page allocation succeeds in the paged pool; a contiguous best-fit
    allocator on the same sequence fails."""
    cap = 64
    p = pm.PoolModel(cap, hidden=4, num_layers=1)
    bf = pm.ContiguousBestFit(cap)
    # 32 requests of S=1 (2 pages each: K and V) fill the pool
    for i in range(32):
        p.kv_alloc(i, 1)
        assert bf.alloc(i, 2)
    for i in range(0, 32, 2):
        p.kv_free(i)
        bf.free(i)
    rep = p.fragmentation_report()
    assert rep["free"] == 32 and rep["largest_free_run"] == 2
    # a request needing 32 pages: paged pool succeeds, contiguous fails
    assert not bf.alloc("big", 32)
    p.kv_alloc(100, 16)
    assert p.free_pages == 0
    p.audit()
