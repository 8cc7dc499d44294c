"""Thin ctypes binding of libslora (include/slora.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no fallback -- if libslora.so is missing, import
fails loudly (build it with ``python -c "import __graft_entry__ as g; g.build()"``).
Device pointers are plain ints; torch tensors are accepted where noted and
only their data_ptr() is passed (PyTorch is used for device memory, streams
and process groups only).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLORA_LIB") or os.path.join(_HERE, "libslora.so")  # SLORA_LIB: alternate build (experiments)

DTYPES = {"f32": 0, "f16": 1, "bf16": 2}
ESIZE = {"f32": 4, "f16": 2, "bf16": 2}
PROJ_BITS = {"q": 1, "k": 2, "v": 4, "o": 8}  # + projection indices 0..7 (ints) for proj_dims pools

STATUS = {
    0: "OK", 1: "INVALID_ARG", 2: "SHAPE", 3: "OUT_OF_PAGES", 4: "ALREADY_RESIDENT",
    5: "NOT_RESIDENT", 6: "PINNED", 7: "NOT_PINNED", 8: "STALE_HANDLE", 9: "FREE_PAGE_READ",
    10: "NONRESIDENT_ADAPTER", 11: "SEGMENT_OVERLAP", 12: "TOKEN_COUNT_NOT_ONE", 13: "INDIVISIBLE",
    14: "CUDA", 15: "NO_DEVICE", 16: "NCCL",
}
TP_ID_BYTES = 128
TP_P2P_HANDLE_BYTES = 64


class SloraError(RuntimeError):
    def __init__(self, code: int, detail: str):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"SLORA_ERR_{self.name}: {detail}")


class PoolConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("dtype", ctypes.c_int), ("hidden", ctypes.c_int64),
                ("num_layers", ctypes.c_int32), ("tp_size", ctypes.c_int32), ("tp_rank", ctypes.c_int32),
                ("capacity_pages", ctypes.c_int64), ("device_buffer", ctypes.c_void_p),
                ("device_buffer_bytes", ctypes.c_int64), ("max_adapters", ctypes.c_int32),
                ("alloc_order", ctypes.c_int), ("seed", ctypes.c_uint64), ("num_proj", ctypes.c_int32),
                ("proj_in", ctypes.c_int64 * 8), ("proj_out", ctypes.c_int64 * 8)]


class FragReport(ctypes.Structure):
    _fields_ = [("capacity_pages", ctypes.c_int64), ("used_pages", ctypes.c_int64),
                ("free_pages", ctypes.c_int64), ("largest_free_run", ctypes.c_int64),
                ("kv_pages", ctypes.c_int64), ("adapter_pages", ctypes.c_int64),
                ("page_elems", ctypes.c_int64), ("resident_adapters", ctypes.c_int32)]


class BatchInfo(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("adapted_tokens", ctypes.c_int32), ("segments", ctypes.c_int32),
                ("sum_rank_tokens", ctypes.c_int64), ("weight_bytes_per_proj", ctypes.c_int64),
                ("mbgmm_segments", ctypes.c_int32)]


class Call(ctypes.Structure):  # slora_call
    _fields_ = [("layer", ctypes.c_int32), ("proj_mask", ctypes.c_uint32), ("x", ctypes.c_void_p),
                ("ldx", ctypes.c_int64), ("y", ctypes.c_void_p * 8), ("ldy", ctypes.c_int64 * 8)]


class LoaderStats(ctypes.Structure):
    _fields_ = [("loads", ctypes.c_int64), ("direct_loads", ctypes.c_int64), ("bytes", ctypes.c_int64),
                ("busy_s", ctypes.c_double), ("queued", ctypes.c_int64)]


class TPStats(ctypes.Structure):
    _fields_ = [("allgather_calls", ctypes.c_int64), ("allgather_send_elems", ctypes.c_int64),
                ("allgather_recv_elems", ctypes.c_int64), ("allreduce_calls", ctypes.c_int64),
                ("allreduce_count", ctypes.c_int64), ("allreduce_send_elems", ctypes.c_int64)]


_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)

# (name, argtypes); every function returns slora_status (int)
SIGNATURES = {
    "slora_pool_create": [ctypes.POINTER(PoolConfig), ctypes.POINTER(_VP)],
    "slora_pool_destroy": [_VP],
    "slora_fragmentation_report": [_VP, ctypes.POINTER(FragReport)],
    "slora_adapter_load": [_VP, _I64, _I32, _VP, ctypes.c_float, _VP, _PI32],
    "slora_adapter_evict": [_VP, _I64, _VP, _PI64],
    "slora_adapter_pin": [_VP, _I64],
    "slora_adapter_unpin": [_VP, _I64],
    "slora_adapter_pages": [_VP, _I64, _PI32, _I64, _PI64],
    "slora_kv_alloc": [_VP, _I64, _I32, _PI32],
    "slora_kv_append": [_VP, _I64, _I32, _PI32],
    "slora_kv_free": [_VP, _I64, _VP, _PI64],
    "slora_kv_pages": [_VP, _I64, _I32, _I32, _PI32, _I64, _PI64],
    "slora_gather_pages": [_VP, _PI32, _I32, _VP, _VP],
    "slora_batch_create": [_VP, ctypes.POINTER(_VP)],
    "slora_batch_destroy": [_VP],
    "slora_batch_prepare": [_VP, _PI64, _I32, _VP],
    "slora_batch_get_info": [_VP, ctypes.POINTER(BatchInfo)],
    "slora_lora_apply": [_VP, _VP, _I32, _U32, _VP, _I64, ctypes.POINTER(_VP), _PI64, _VP],
    "slora_lora_v_elems": [_VP, _U32, _I32, _PI64],
    "slora_lora_shrink": [_VP, _VP, _I32, _U32, _VP, _I64, _VP, _VP],
    "slora_lora_expand": [_VP, _VP, _I32, _U32, _VP, _I32, ctypes.POINTER(_VP), _PI64, _VP],
    "slora_tp_unique_id": [_VP],
    "slora_tp_init": [_VP, _VP, _I32, _I32],
    "slora_tp_lora_qkv": [_VP, _VP, _I32, _VP, _I64, ctypes.POINTER(_VP), _PI64, _VP],
    "slora_tp_lora_o": [_VP, _VP, _I32, _VP, _I64, _VP, _I64, _VP],
    "slora_tp_get_stats": [_VP, ctypes.POINTER(TPStats)],
    "slora_batch_set_options": [_VP, ctypes.c_uint32],
    "slora_tp_p2p_export": [_VP, _VP],
    "slora_tp_p2p_open": [_VP, _VP],
    "slora_tp_fused_qkv": [_VP, _VP, _I32, _VP, _I64, _VP, _VP, _VP],
    "slora_tp_fused_o": [_VP, _VP, _I32, _VP, _I64, _VP, _I64, _VP],
    "slora_lora_apply_many": [_VP, _VP, _VP, _I32, _VP, ctypes.POINTER(_I32)],
    "slora_adapter_prefetch": [_VP, _I64, _I32, _VP, ctypes.c_float, ctypes.POINTER(_I32)],
    "slora_adapter_wait": [_VP, _I64],
    "slora_adapter_query": [_VP, _I64, ctypes.POINTER(_I32)],
    "slora_loader_get_stats": [_VP, ctypes.POINTER(LoaderStats)],
    "slora_sync": [_VP, _VP],
    "slora_debug_trace": [_VP, _PI64, _I32],
}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA extension is not built "
                              "(run __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.slora_status_string.argtypes = [ctypes.c_int]
        L.slora_status_string.restype = ctypes.c_char_p
        L.slora_last_error.argtypes = []
        L.slora_last_error.restype = ctypes.c_char_p
        L.slora_launch_count.argtypes = []
        L.slora_launch_count.restype = ctypes.c_int64
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise SloraError(rc, lib().slora_last_error().decode())


def launch_count() -> int:
    return int(lib().slora_launch_count())


def _ptr(t) -> int:
    """Device pointer of a torch tensor or a plain int (0 for None)."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return int(t.data_ptr())


def _stream(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


def tp_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0); broadcast the bytes to the other ranks."""
    buf = ctypes.create_string_buffer(TP_ID_BYTES)
    _check(lib().slora_tp_unique_id(buf))
    return buf.raw


def mask_of(projs) -> int:
    if isinstance(projs, int):
        return projs
    m = 0
    for p in projs:
        m |= (1 << p) if isinstance(p, int) else PROJ_BITS[p]
    return m


class Pool:
    """Unified Paging pool.  device=-1: bookkeeping only (CPU)."""

    def __init__(self, hidden: int, num_layers: int, capacity_pages: int, dtype: str = "f16",
                 device: int = 0, buffer=None, tp_size: int = 1, tp_rank: int = 0,
                 max_adapters: int = 1024, order: str = "ascending", seed: int = 0, proj_dims=None):
        """proj_dims: [(in, out)] per LoRA'd projection (NEXT-4); None = q,k,v,o square."""
        self.hidden, self.num_layers, self.dtype = hidden, num_layers, dtype
        self.proj_dims = [(hidden, hidden)] * 4 if proj_dims is None else [tuple(d) for d in proj_dims]
        self.tp_size, self.tp_rank = tp_size, tp_rank
        self.page_elems = hidden // tp_size
        self.capacity = capacity_pages
        self.device = device
        self.buffer = buffer
        nbytes = 0
        if device >= 0 and buffer is None:
            import torch
            nbytes = capacity_pages * self.page_elems * ESIZE[dtype]
            self.buffer = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        if self.buffer is not None:
            nbytes = self.buffer.numel() * self.buffer.element_size()
        pin = (ctypes.c_int64 * 8)(*([d[0] for d in self.proj_dims] + [0] * (8 - len(self.proj_dims))))
        pout = (ctypes.c_int64 * 8)(*([d[1] for d in self.proj_dims] + [0] * (8 - len(self.proj_dims))))
        cfg = PoolConfig(device, DTYPES[dtype], hidden, num_layers, tp_size, tp_rank, capacity_pages,
                         _ptr(self.buffer) or None, nbytes, max_adapters,
                         {"ascending": 0, "shuffle": 1}[order], seed,
                         0 if proj_dims is None else len(self.proj_dims), pin, pout)
        h = _VP()
        self._inflight, self._retired = {}, []
        _check(lib().slora_pool_create(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().slora_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------------- a2
    def _host_ptr(self, host_w, rank: int):
        """(pointer, kept object) of a host adapter buffer: a numpy array, or a CPU torch tensor
        (pinned tensors are read directly by the loader).  Checks dtype and size."""
        if host_w is None:
            return None, None
        want_item = ESIZE[self.dtype]
        need = self.num_layers * sum(i + o for i, o in self.proj_dims) * rank * want_item
        if hasattr(host_w, "data_ptr"):  # torch CPU tensor
            import torch
            ok = {"f32": (torch.float32,), "f16": (torch.float16,),
                  "bf16": (torch.bfloat16, torch.int16, torch.uint16)}[self.dtype]
            if host_w.device.type != "cpu" or not host_w.is_contiguous():
                raise ValueError("host_w must be a contiguous CPU tensor")
            if host_w.dtype not in ok:
                raise ValueError(f"host_w dtype {host_w.dtype} does not match the pool dtype {self.dtype}")
            if host_w.numel() * host_w.element_size() != need:
                raise ValueError(f"host_w holds {host_w.numel() * host_w.element_size()} bytes, "
                                 f"the canonical layout needs {need}")
            return int(host_w.data_ptr()), host_w
        host_w = np.ascontiguousarray(host_w)
        # the library reads exactly this many bytes of the pool's element type from the pointer
        kind_ok = (host_w.dtype == np.float32 if self.dtype == "f32" else
                   host_w.dtype == np.float16 if self.dtype == "f16" else
                   host_w.dtype in (np.uint16, np.int16))
        if self.device < 0:
            pass  # bookkeeping-only pool: the library refuses host weights (NO_DEVICE)
        elif not kind_ok or host_w.itemsize != want_item:
            raise ValueError(f"host_w dtype {host_w.dtype} does not match the pool dtype {self.dtype}")
        elif host_w.nbytes != need:
            raise ValueError(f"host_w holds {host_w.nbytes} bytes, the canonical layout needs {need}")
        return host_w.ctypes.data, host_w

    def adapter_load(self, adapter_id: int, rank: int, host_w=None,
                     scale: float = 1.0, stream=None) -> int:
        slot = ctypes.c_int32(-1)
        ptr, _keep = self._host_ptr(host_w, rank)
        _check(lib().slora_adapter_load(self.h, adapter_id, rank, ptr, scale, _stream(stream),
                                        ctypes.byref(slot)))
        return slot.value

    # ------------------------------------------------------------- NEXT-1
    def adapter_prefetch(self, adapter_id: int, rank: int, host_w, scale: float = 1.0) -> int:
        """Asynchronous load on the pool's loader thread and copy stream; host_w is kept
        alive here until adapter_wait / adapter_loading reports the load complete."""
        slot = ctypes.c_int32(-1)
        ptr, keep = self._host_ptr(host_w, rank)
        _check(lib().slora_adapter_prefetch(self.h, adapter_id, rank, ptr, scale, ctypes.byref(slot)))
        self._inflight[adapter_id] = keep
        return slot.value

    def adapter_wait(self, adapter_id: int) -> None:
        _check(lib().slora_adapter_wait(self.h, adapter_id))
        self._inflight.pop(adapter_id, None)

    def adapter_loading(self, adapter_id: int) -> bool:
        v = ctypes.c_int32(0)
        _check(lib().slora_adapter_query(self.h, adapter_id, ctypes.byref(v)))
        if not v.value:
            self._inflight.pop(adapter_id, None)
        return bool(v.value)

    def loader_stats(self) -> dict:
        st = LoaderStats()
        _check(lib().slora_loader_get_stats(self.h, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in LoaderStats._fields_}

    def adapter_evict(self, adapter_id: int, stream=None) -> int:
        n = ctypes.c_int64(0)
        _check(lib().slora_adapter_evict(self.h, adapter_id, _stream(stream), ctypes.byref(n)))
        keep = self._inflight.pop(adapter_id, None)
        if keep is not None:  # a load still in flight reads host_w until the fenced stream gets there
            self._retired.append((keep, stream))
        return n.value

    def pin(self, adapter_id: int) -> None:
        _check(lib().slora_adapter_pin(self.h, adapter_id))

    def unpin(self, adapter_id: int) -> None:
        _check(lib().slora_adapter_unpin(self.h, adapter_id))

    def adapter_pages(self, adapter_id: int) -> np.ndarray:
        n = ctypes.c_int64(0)
        _check(lib().slora_adapter_pages(self.h, adapter_id, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.int32)
        _check(lib().slora_adapter_pages(self.h, adapter_id, out.ctypes.data_as(_PI32), n.value,
                                         ctypes.byref(n)))
        return out

    # ----------------------------------------------------------------- a3
    def kv_alloc(self, request_id: int, n_tokens: int) -> np.ndarray:
        out = np.zeros(max(1, 2 * n_tokens * self.num_layers), np.int32)
        _check(lib().slora_kv_alloc(self.h, request_id, n_tokens, out.ctypes.data_as(_PI32)))
        return out[:2 * n_tokens * self.num_layers]

    def kv_append(self, request_id: int, n_tokens: int) -> np.ndarray:
        out = np.zeros(max(1, 2 * max(n_tokens, 0) * self.num_layers), np.int32)
        _check(lib().slora_kv_append(self.h, request_id, n_tokens, out.ctypes.data_as(_PI32)))
        return out[:2 * n_tokens * self.num_layers]

    def kv_free(self, request_id: int, stream=None) -> int:
        n = ctypes.c_int64(0)
        _check(lib().slora_kv_free(self.h, request_id, _stream(stream), ctypes.byref(n)))
        return n.value

    def kv_pages(self, request_id: int, layer: int, kind: int) -> np.ndarray:
        n = ctypes.c_int64(0)
        _check(lib().slora_kv_pages(self.h, request_id, layer, kind, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value, np.int32)
        _check(lib().slora_kv_pages(self.h, request_id, layer, kind, out.ctypes.data_as(_PI32), n.value,
                                    ctypes.byref(n)))
        return out

    def gather_pages(self, pages, dst, stream=None) -> None:
        pages = np.ascontiguousarray(pages, np.int32)
        _check(lib().slora_gather_pages(self.h, pages.ctypes.data_as(_PI32), int(pages.size), _ptr(dst),
                                        _stream(stream)))

    def frag_report(self) -> dict:
        r = FragReport()
        _check(lib().slora_fragmentation_report(self.h, ctypes.byref(r)))
        return {f: getattr(r, f) for f, _ in FragReport._fields_}

    def sync(self, stream=None) -> None:
        _check(lib().slora_sync(self.h, _stream(stream)))

    # -------------------------------------------------------------- a6/a8
    def tp_init(self, unique_id: bytes, rank: int, size: int) -> None:
        """Create the library's NCCL communicator (all ranks, same id)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), TP_ID_BYTES)
        _check(lib().slora_tp_init(self.h, buf, rank, size))

    def tp_p2p_export(self) -> bytes:
        """NEXT-3: this rank's exchange region (allocated here) as a CUDA IPC handle."""
        buf = ctypes.create_string_buffer(TP_P2P_HANDLE_BYTES)
        _check(lib().slora_tp_p2p_export(self.h, buf))
        return buf.raw

    def tp_p2p_open(self, handles) -> None:
        """Map every rank's exchange region (handles: the N ranks' export bytes, rank order)."""
        blob = b"".join(bytes(h) for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib().slora_tp_p2p_open(self.h, buf))

    def tp_stats(self) -> dict:
        r = TPStats()
        _check(lib().slora_tp_get_stats(self.h, ctypes.byref(r)))
        return {f: getattr(r, f) for f, _ in TPStats._fields_}

    def debug_trace(self) -> np.ndarray:
        """[16 CTAs, 1024 events] globaltimer ns of the last traced launches."""
        out = np.zeros(16 * 1024, np.int64)
        _check(lib().slora_debug_trace(self.h, out.ctypes.data_as(_PI64), 16 * 1024))
        return out.reshape(16, 1024)


class Batch:
    """Batch descriptor (token -> adapter map, segments, work units)."""

    def __init__(self, pool: Pool):
        self.pool = pool
        h = _VP()
        _check(lib().slora_batch_create(pool.h, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().slora_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, token_adapter, stream=None) -> None:
        ta = np.ascontiguousarray(token_adapter, np.int64)
        _check(lib().slora_batch_prepare(self.h, ta.ctypes.data_as(_PI64), int(ta.size), _stream(stream)))

    def set_options(self, mbgmv_only: bool = False) -> None:
        """mbgmv_only: every segment on the MBGMV path (graph replay across batches)."""
        _check(lib().slora_batch_set_options(self.h, 1 if mbgmv_only else 0))

    def info(self) -> dict:
        r = BatchInfo()
        _check(lib().slora_batch_get_info(self.h, ctypes.byref(r)))
        return {f: getattr(r, f) for f, _ in BatchInfo._fields_}

    def v_elems(self, projs, div: int = 1) -> int:
        n = ctypes.c_int64(0)
        _check(lib().slora_lora_v_elems(self.h, mask_of(projs), div, ctypes.byref(n)))
        return n.value

    @staticmethod
    def _ys(ys, ldys):
        ys, ldys = list(ys) + [None] * (8 - len(ys)), list(ldys) + [0] * (8 - len(ldys))
        yp = (_VP * 8)(*[_ptr(y) or None for y in ys])
        ld = (_I64 * 8)(*ldys)
        return yp, ld

    def apply(self, layer: int, projs, x, ldx: int, ys, ldys, stream=None) -> None:
        """Fused shrink->expand (one GPU): ys/ldys indexed by projection id (q,k,v,o, then proj_dims extras)."""
        yp, ld = self._ys(ys, ldys)
        _check(lib().slora_lora_apply(self.pool.h, self.h, layer, mask_of(projs), _ptr(x), ldx, yp, ld,
                                      _stream(stream)))

    @staticmethod
    def make_calls(calls) -> "ctypes.Array":
        """Pack [(layer, projs, x, ldx, ys, ldys)] into a slora_call array (build once, reuse every step)."""
        arr = (Call * len(calls))()
        for c, (layer, projs, x, ldx, ys, ldys) in zip(arr, calls):
            c.layer, c.proj_mask, c.x, c.ldx = layer, mask_of(projs), _ptr(x) or None, ldx
            ys, ldys = list(ys) + [None] * (8 - len(ys)), list(ldys) + [0] * (8 - len(ldys))
            for i in range(8):
                c.y[i] = _ptr(ys[i]) or None
                c.ldy[i] = ldys[i]
        return arr

    def apply_many(self, calls, stream=None) -> None:
        """slora_lora_apply_many: a packed call array (make_calls) enqueued with one ABI crossing."""
        failed = _I32(-1)
        _check(lib().slora_lora_apply_many(self.pool.h, self.h, ctypes.addressof(calls), len(calls),
                                           _stream(stream), ctypes.byref(failed)))

    def shrink(self, layer: int, projs, x, ldx: int, v, stream=None) -> None:
        _check(lib().slora_lora_shrink(self.pool.h, self.h, layer, mask_of(projs), _ptr(x), ldx, _ptr(v),
                                       _stream(stream)))

    def tp_qkv(self, layer: int, x, ldx: int, ys, ldys, stream=None) -> None:
        """TP q/k/v: shrink -> NCCL all-gather -> expand into the three column shards."""
        yp = (_VP * 3)(*[_ptr(y) or None for y in ys])
        ld = (_I64 * 3)(*ldys)
        _check(lib().slora_tp_lora_qkv(self.pool.h, self.h, layer, _ptr(x), ldx, yp, ld, _stream(stream)))

    def tp_o(self, layer: int, z, ldz: int, base_partial, ld_base: int, stream=None) -> None:
        """TP o: shrink -> NCCL all-reduce -> expand into column slice k of the base partial."""
        _check(lib().slora_tp_lora_o(self.pool.h, self.h, layer, _ptr(z), ldz, _ptr(base_partial), ld_base,
                                     _stream(stream)))

    def tp_fused_qkv(self, layer: int, x, ldx: int, ys, ldys, stream=None) -> None:
        """NEXT-3: TP q/k/v in one kernel, the v exchange by NVLink peer stores (slora_tp_fused_qkv)."""
        yp = (_VP * 3)(*[_ptr(y) or None for y in ys])
        ld = (_I64 * 3)(*ldys)
        _check(lib().slora_tp_fused_qkv(self.pool.h, self.h, layer, _ptr(x), ldx, yp, ld, _stream(stream)))

    def tp_fused_o(self, layer: int, z, ldz: int, base_partial, ld_base: int, stream=None) -> None:
        """NEXT-3: TP o in one kernel, the all-reduce by peer stores summed in rank order (slora_tp_fused_o)."""
        _check(lib().slora_tp_fused_o(self.pool.h, self.h, layer, _ptr(z), ldz, _ptr(base_partial), ld_base,
                                      _stream(stream)))

    def expand(self, layer: int, projs, v, v_blocks: int, ys, ldys, stream=None) -> None:
        yp, ld = self._ys(ys, ldys)
        _check(lib().slora_lora_expand(self.pool.h, self.h, layer, mask_of(projs), _ptr(v), v_blocks, yp,
                                       ld, _stream(stream)))
