"""Reference model of the Unified Paging pool (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import anything under oracle/.  This module shares no code with the C++ pool
in paper_2311_03285_b200/csrc/; the tests drive both with the same operation
sequence and compare page ids bit-exactly.

What the paper fixes (P:L = /root/reference/PAPER.md line L):
  * one statically allocated buffer, "each page corresponding to a vector of
    H";
  * "a KV cache tensor with a sequence length of S uses up S pages, while a
    LoRA weight tensor of rank R takes up R pages";
  * KV caches and adapter weights "stored interleaved and non-contiguously"
    (Fig. unified_memory_pool).
What the paper leaves open, with the readings used here:
  * R10 allocation order: a LIFO free stack.  Initially the stack pops page
    0, 1, 2, ... ('ascending'), or a splitmix64-seeded Fisher-Yates shuffle of
    that stack ('shuffle').  Released pages are pushed in release order.
  * R11 K and V are separate (S, H) tensors: 2*S pages per layer per request.
  * R3  under N-way tensor parallelism the per-GPU page is H/N elements; every
    LoRA tensor still takes r pages per GPU (q/k/v A shard: r/N rank columns
    of length H, i.e. N pages each; all other shards: r rows of H/N).
  * Adapter slots: the lowest free slot index is assigned on load.
  * R2 (NEXT-4, P:321-327 uses the MLP as its worked example): projections
    need not be square.  A stored row of n elements (A row j = column j of the
    h_in x r matrix A; B row j of r x d_out) spans ceil(n/H) pages, the last
    one partly used; for n = H this is P:262's one page per rank row.  Pools
    with non-square projections are single-GPU (tp_size 1).
Error names follow SPEC S:114-163 (see include/slora.h).
"""
from __future__ import annotations

from dataclasses import dataclass, field

MASK64 = (1 << 64) - 1

# status codes (same numbering as include/slora.h; the numbers are the
# interface, written out here independently)
OK = 0
ERR_INVALID_ARG = 1
ERR_SHAPE = 2
ERR_OUT_OF_PAGES = 3
ERR_ALREADY_RESIDENT = 4
ERR_NOT_RESIDENT = 5
ERR_PINNED = 6
ERR_NOT_PINNED = 7
ERR_STALE_HANDLE = 8
ERR_FREE_PAGE_READ = 9
ERR_NONRESIDENT_ADAPTER = 10
ERR_SEGMENT_OVERLAP = 11
ERR_TOKEN_COUNT_NOT_ONE = 12
ERR_INDIVISIBLE = 13


class PoolError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


def splitmix64(state: int):
    """splitmix64 step; returns (new_state, output)."""
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def initial_free_stack(capacity: int, order: str, seed: int) -> list[int]:
    """Free stack, top = last element.  'ascending' pops 0, 1, 2, ...
    'shuffle': for i = cap-1 .. 1: j = splitmix64() % (i+1); swap(s[i], s[j])."""
    stack = list(range(capacity - 1, -1, -1))
    if order == "shuffle":
        st = seed & MASK64
        for i in range(capacity - 1, 0, -1):
            st, z = splitmix64(st)
            j = z % (i + 1)
            stack[i], stack[j] = stack[j], stack[i]
    elif order != "ascending":
        raise ValueError(order)
    return stack


@dataclass
class Adapter:
    adapter_id: int
    rank: int
    slot: int
    pages: list  # pop order: layer, proj, tensor(A=0,B=1), row, chunk
    pinned: bool = False


@dataclass
class KvHandle:
    request_id: int
    seq_len: int
    pages: dict = field(default_factory=dict)  # (layer, kind) -> [page per position]


class PoolModel:
    NUM_PROJ = 4  # q, k, v, o (LoRA on the attention projections)

    def __init__(self, capacity_pages: int, hidden: int, num_layers: int,
                 tp_size: int = 1, tp_rank: int = 0, order: str = "ascending",
                 seed: int = 0, max_adapters: int = 1024, proj_dims=None):
        if capacity_pages < 1 or hidden < 1 or num_layers < 1 or tp_size < 1:
            raise PoolError(ERR_INVALID_ARG, "sizes must be >= 1")
        # (h_in, d_out) per LoRA'd projection; default q, k, v, o square
        self.dims = [(hidden, hidden)] * 4 if proj_dims is None else [tuple(d) for d in proj_dims]
        self.NUM_PROJ = len(self.dims)
        if tp_size > 1 and self.dims != [(hidden, hidden)] * 4:
            raise PoolError(ERR_SHAPE, "tensor parallelism needs the four square projections")
        if not (0 <= tp_rank < tp_size):
            raise PoolError(ERR_INVALID_ARG, "tp_rank")
        if hidden % tp_size:
            raise PoolError(ERR_INDIVISIBLE, "hidden % tp_size")
        self.capacity = capacity_pages
        self.hidden = hidden
        self.page_elems = hidden // tp_size  # R3
        self.L = num_layers
        self.N = tp_size
        self.k = tp_rank
        self.free = initial_free_stack(capacity_pages, order, seed)
        self.owner: list = [None] * capacity_pages
        self.adapters: dict[int, Adapter] = {}
        self.slots: list = [None] * max_adapters
        self.kv: dict[int, KvHandle] = {}

    # ---------------------------------------------------------------- helpers
    @property
    def free_pages(self) -> int:
        return len(self.free)

    @property
    def used_pages(self) -> int:
        return self.capacity - len(self.free)

    def _pop(self, n: int) -> list[int]:
        out = []
        for _ in range(n):
            out.append(self.free.pop())
        return out

    def tensor_shape(self, proj: int, tensor: int, rank: int):
        """(rows, chunks per row) of one LoRA tensor shard on this GPU (R3).
        A is stored transposed: one row per rank column (R1)."""
        N = self.N
        if N > 1:
            if proj < 3 and tensor == 0:  # q/k/v A: column partition along r
                return rank // N, N
            return rank, 1
        n = self.dims[proj][0 if tensor == 0 else 1]  # stored row length (R2)
        return rank, -(-n // self.page_elems)

    def adapter_page_count(self, rank: int) -> int:
        n = 0
        for _l in range(self.L):
            for p in range(self.NUM_PROJ):
                for t in range(2):
                    rows, chunks = self.tensor_shape(p, t, rank)
                    n += rows * chunks
        return n

    # -------------------------------------------------------------------- KV
    def kv_alloc(self, request_id: int, n_tokens: int) -> list[int]:
        if n_tokens < 0 or request_id in self.kv:
            raise PoolError(ERR_INVALID_ARG, "kv_alloc")
        need = 2 * n_tokens * self.L  # R11: K and V, S pages each, per layer
        if need > self.free_pages:
            raise PoolError(ERR_OUT_OF_PAGES, f"needed={need} free={self.free_pages}")
        hd = KvHandle(request_id, 0)
        for l in range(self.L):
            for kind in range(2):
                hd.pages[(l, kind)] = []
        self.kv[request_id] = hd
        return self._kv_grow(hd, n_tokens)

    def _kv_grow(self, hd: KvHandle, n: int) -> list[int]:
        got = []
        for l in range(self.L):
            for kind in range(2):
                for pos in range(hd.seq_len, hd.seq_len + n):
                    p = self.free.pop()
                    self.owner[p] = ("kv", hd.request_id, l, kind, pos)
                    hd.pages[(l, kind)].append(p)
                    got.append(p)
        hd.seq_len += n
        return got

    def kv_append(self, request_id: int, n_tokens: int) -> list[int]:
        hd = self.kv.get(request_id)
        if hd is None:
            raise PoolError(ERR_STALE_HANDLE, "kv_append")
        if n_tokens < 0:
            raise PoolError(ERR_INVALID_ARG, "n_tokens")
        need = 2 * n_tokens * self.L
        if need > self.free_pages:
            raise PoolError(ERR_OUT_OF_PAGES, f"needed={need} free={self.free_pages}")
        return self._kv_grow(hd, n_tokens)

    def kv_free(self, request_id: int) -> int:
        hd = self.kv.pop(request_id, None)
        if hd is None:
            raise PoolError(ERR_STALE_HANDLE, "kv_free")
        n = 0
        for l in range(self.L):
            for kind in range(2):
                for p in hd.pages[(l, kind)]:
                    self.owner[p] = None
                    self.free.append(p)
                    n += 1
        return n

    # -------------------------------------------------------------- adapters
    def adapter_load(self, adapter_id: int, rank: int) -> int:
        if rank < 1:
            raise PoolError(ERR_INVALID_ARG, "rank")
        if rank % self.N:
            raise PoolError(ERR_INDIVISIBLE, "rank % tp_size")
        if adapter_id in self.adapters:
            raise PoolError(ERR_ALREADY_RESIDENT, str(adapter_id))
        try:
            slot = self.slots.index(None)
        except ValueError:
            raise PoolError(ERR_OUT_OF_PAGES, "no free adapter slot") from None
        need = self.adapter_page_count(rank)
        if need > self.free_pages:
            raise PoolError(ERR_OUT_OF_PAGES, f"needed={need} free={self.free_pages}")
        pages = []
        for l in range(self.L):
            for p in range(self.NUM_PROJ):
                for t in range(2):
                    rows, chunks = self.tensor_shape(p, t, rank)
                    for row in range(rows):
                        for c in range(chunks):
                            pg = self.free.pop()
                            self.owner[pg] = ("adapter", adapter_id, l, p, t, row, c)
                            pages.append(pg)
        ad = Adapter(adapter_id, rank, slot, pages)
        self.adapters[adapter_id] = ad
        self.slots[slot] = adapter_id
        return slot

    def adapter_evict(self, adapter_id: int) -> int:
        ad = self.adapters.get(adapter_id)
        if ad is None:
            raise PoolError(ERR_NOT_RESIDENT, str(adapter_id))
        if ad.pinned:
            raise PoolError(ERR_PINNED, str(adapter_id))
        for pg in ad.pages:
            self.owner[pg] = None
            self.free.append(pg)
        del self.adapters[adapter_id]
        self.slots[ad.slot] = None
        return len(ad.pages)

    def pin(self, adapter_id: int) -> None:
        ad = self.adapters.get(adapter_id)
        if ad is None:
            raise PoolError(ERR_NOT_RESIDENT, str(adapter_id))
        ad.pinned = True

    def unpin(self, adapter_id: int) -> None:
        ad = self.adapters.get(adapter_id)
        if ad is None:
            raise PoolError(ERR_NOT_RESIDENT, str(adapter_id))
        if not ad.pinned:
            raise PoolError(ERR_NOT_PINNED, str(adapter_id))
        ad.pinned = False

    # ---------------------------------------------------------------- checks
    def check_gather(self, pages) -> None:
        for p in pages:
            if not (0 <= p < self.capacity):
                raise PoolError(ERR_INVALID_ARG, f"page {p}")
            if self.owner[p] is None:
                raise PoolError(ERR_FREE_PAGE_READ, f"page {p}")

    def fragmentation_report(self) -> dict:
        run = best = 0
        for p in range(self.capacity):
            if self.owner[p] is None:
                run += 1
                best = max(best, run)
            else:
                run = 0
        kv = sum(1 for o in self.owner if o is not None and o[0] == "kv")
        ad = sum(1 for o in self.owner if o is not None and o[0] == "adapter")
        return {"used": self.used_pages, "free": self.free_pages,
                "largest_free_run": best, "kv_pages": kv, "adapter_pages": ad}

    def audit(self) -> None:
        """Invariants S:166-169: conservation, no double ownership, owner
        table consistent with handles, pinned adapters resident."""
        assert self.used_pages + self.free_pages == self.capacity
        assert len(set(self.free)) == len(self.free)
        seen = set()
        for hd in self.kv.values():
            for lst in hd.pages.values():
                assert len(lst) == hd.seq_len
                for p in lst:
                    assert p not in seen
                    seen.add(p)
        for ad in self.adapters.values():
            for p in ad.pages:
                assert p not in seen
                seen.add(p)
        assert len(seen) == self.used_pages
        assert seen.isdisjoint(self.free)
        for p in range(self.capacity):
            assert (self.owner[p] is None) == (p not in seen)


class ContiguousBestFit:
    """Contrast harness: a contiguous best-fit allocator.
    Used only to show external fragmentation that paging does not have."""

    def __init__(self, capacity: int):
        self.capacity = capacity
        self.used = [False] * capacity
        self.allocs: dict = {}

    def alloc(self, key, n: int) -> bool:
        best = None
        p = 0
        while p < self.capacity:
            if self.used[p]:
                p += 1
                continue
            q = p
            while q < self.capacity and not self.used[q]:
                q += 1
            if q - p >= n and (best is None or q - p < best[1] - best[0]):
                best = (p, q)
            p = q
        if best is None:
            return False
        for i in range(best[0], best[0] + n):
            self.used[i] = True
        self.allocs[key] = (best[0], n)
        return True

    def free(self, key) -> None:
        s, n = self.allocs.pop(key)
        for i in range(s, s + n):
            self.used[i] = False
