"""Seeded synthetic inputs shared by the CUDA path's tests/bench and by the
oracle's tests.  This module holds NONE of the method's arithmetic: it only
draws random numbers and rounds them to the storage dtype.

Workload model (Sec. 7.2; Table model_setting P:369-378;
Table default_trace), readings in DESIGN.md:
  * adapter popularity p_i proportional to i^-alpha over adapters i = 1..n
    ("power-law distribution with an exponent alpha", reading R17);
  * ranks assigned round-robin from the setting's rank list in the paper's
    order, adapter i -> list[i mod len] ("round-robin method");
  * prefill lengths ~ U[8, 512] (Table default_trace [I_l, I_u]);
  * decode tokens: one per request.
Values: x ~ N(0,1), y_in ~ N(0,1), A ~ N(0, 1/h), B ~ N(0, 1/r), each rounded
to the config dtype on the host (fp32 / fp16 / bf16 with round-to-nearest-even).
Seeds: data seed 231103285 + config index; weights of (adapter a, layer l,
projection p) come from their own stream so any subset can be regenerated.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DATA_SEED = 231103285
PROJ = ("q", "k", "v", "o")


@dataclass
class Config:
    name: str
    index: int
    hidden: int
    n_adapters: int
    rank_list: tuple
    dtype: str                       # "f32" | "f16" | "bf16"
    alpha: float | None = 1.0        # None -> uniform popularity
    decode_tokens: int = 64
    prefill_requests: int = 0
    prefill_range: tuple = (8, 512)
    tp: int = 1
    num_layers: int = 32
    fixed_requests: list | None = None  # C0: explicit (adapter, length) list
    notes: str = ""
    proj_dims: tuple | None = None   # NEXT-4: (h_in, d_out) per LoRA'd projection; None = q,k,v,o square


CONFIGS = {
    # BASELINE.json configs[0]: tiny single layer fp32, hidden 256, 4 adapters
    # ranks {4,8}, 16 tokens across 4 requests, page size = hidden
    "c0": Config("c0-tiny-fp32", 0, 256, 4, (4, 8), "f32", None, 0, 0, tp=1, num_layers=1,
                 fixed_requests=[(0, 5), (1, 1), (2, 7), (3, 3)]),
    # configs[1]: Llama-7B q/k/v/o (h=4096), 1000 adapters all rank 8, decode 64, fp16 (S1)
    "c1": Config("c1-7b-r8-decode64-fp16", 1, 4096, 1000, (8,), "f16", 1.0, 64),
    # configs[2]: Llama-7B, 2000 adapters ranks {64,32,16,8} Zipf, fp16 (S2)
    "c2": Config("c2-7b-mixedrank-decode64-fp16", 2, 4096, 2000, (64, 32, 16, 8), "f16", 1.0, 64),
    # C2 with uniform adapter popularity (SURVEY 8(d) variant (ii): ~63 distinct adapters of 64 tokens)
    "c2-uniform": Config("c2-7b-mixedrank-decode64-uniform-fp16", 2, 4096, 2000, (64, 32, 16, 8), "f16", None, 64),
    "c2-mixed": Config("c2-7b-mixedrank-prefill8+decode56-fp16", 2, 4096, 2000, (64, 32, 16, 8), "f16",
                       1.0, 56, prefill_requests=8),
    # configs[3]: Llama-13B (h=5120), ranks {64,32,16}, 4-way TP (n=400, Table default_trace 13B@A100-80G)
    "c3": Config("c3-13b-tp4-decode64-fp16", 3, 5120, 400, (64, 32, 16), "f16", 1.0, 64, tp=4,
                 num_layers=40),
    # configs[4]: Llama-70B (h=8192) 8-way TP, rank 64, decode 256, bf16 (n=10)
    "c4": Config("c4-70b-tp8-r64-decode256-bf16", 4, 8192, 10, (64,), "bf16", 1.0, 256, tp=8,
                 num_layers=80),
    # NEXT-4 (P:321-327 takes the MLP as its example): C2's batch with LoRA on all seven Llama-7B
    # projections, q/k/v/o 4096 -> 4096, gate/up 4096 -> 11008, down 11008 -> 4096 (Table model_setting
    # P:369-378 gives the 7B shapes); index 2: the same batch and attention weights as C2
    "c2-mlp": Config("c2-7b-qkvo+mlp-decode64-fp16", 2, 4096, 2000, (64, 32, 16, 8), "f16", 1.0, 64,
                     proj_dims=((4096, 4096),) * 4 + ((4096, 11008), (4096, 11008), (11008, 4096))),
}


def proj_dims(cfg: Config) -> list:
    """(h_in, d_out) of each LoRA'd projection of the config."""
    return [(cfg.hidden, cfg.hidden)] * 4 if cfg.proj_dims is None else [tuple(d) for d in cfg.proj_dims]


def adapter_rank(cfg: Config, adapter: int) -> int:
    """Round-robin rank assignment: adapter i -> rank_list[i mod len]."""
    return cfg.rank_list[adapter % len(cfg.rank_list)]


def popularity(n: int, alpha: float | None) -> np.ndarray:
    """p_i proportional to i^-alpha, i = 1..n (reading R17); uniform if None."""
    if alpha is None:
        return np.full(n, 1.0 / n)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-float(alpha))
    return w / w.sum()


@dataclass
class Batch:
    requests: list                   # [(adapter or -1, n_tokens)]
    token_adapter: np.ndarray        # int64[T], -1 = no adapter
    ranks: dict = field(default_factory=dict)   # adapter -> rank (adapters in the batch)

    @property
    def T(self) -> int:
        return int(self.token_adapter.size)

    @property
    def unique(self) -> list:
        return sorted(self.ranks)


def make_batch(cfg: Config, seed_offset: int = 0, no_adapter_frac: float = 0.0) -> Batch:
    """Batch composition: prefill requests first (lengths ~ U[prefill_range]),
    then decode requests of one token; each request's adapter drawn from the
    popularity law.  `no_adapter_frac` marks that fraction of requests as
    base-only (slot -1)."""
    rng = np.random.default_rng(DATA_SEED + cfg.index + 1000 * seed_offset)
    if cfg.fixed_requests is not None:
        reqs = list(cfg.fixed_requests)
    else:
        n_req = cfg.prefill_requests + cfg.decode_tokens
        p = popularity(cfg.n_adapters, cfg.alpha)
        ads = rng.choice(cfg.n_adapters, size=n_req, p=p)
        lens = [int(rng.integers(cfg.prefill_range[0], cfg.prefill_range[1] + 1))
                for _ in range(cfg.prefill_requests)] + [1] * cfg.decode_tokens
        reqs = [(int(a), int(n)) for a, n in zip(ads, lens)]
    if no_adapter_frac > 0:
        drop = rng.random(len(reqs)) < no_adapter_frac
        reqs = [(-1 if dr else a, n) for (a, n), dr in zip(reqs, drop)]
    tok = np.concatenate([np.full(n, a, np.int64) for a, n in reqs]) if reqs else np.zeros(0, np.int64)
    ranks = {a: adapter_rank(cfg, a) for a, _ in reqs if a >= 0}
    return Batch(reqs, tok, ranks)


# ------------------------------------------------------------------ values
def round_to(x32: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp32 values to the storage dtype; returns the STORED array:
    float32 / float16 / uint16 bf16 bit patterns (round-to-nearest-even)."""
    x32 = np.asarray(x32, np.float32)
    if dtype == "f32":
        return x32
    if dtype == "f16":
        return x32.astype(np.float16)
    if dtype == "bf16":
        b = x32.view(np.uint32).astype(np.uint64)
        b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
        return b.astype(np.uint16)
    raise ValueError(dtype)


def storage_np_dtype(dtype: str):
    return {"f32": np.float32, "f16": np.float16, "bf16": np.uint16}[dtype]


def elem_bytes(dtype: str) -> int:
    return 4 if dtype == "f32" else 2


def _normal(rng, shape, std):
    return rng.standard_normal(shape, dtype=np.float32) * np.float32(std)


def adapter_weights(cfg: Config, adapter: int, layer: int, proj: int, rank: int | None = None,
                    seed_offset: int = 0):
    """(A: h x r, B: r x d) for one (adapter, layer, projection), stored dtype.
    A ~ N(0, 1/h), B ~ N(0, 1/r); h, d = the projection's dims (proj_dims)."""
    r = adapter_rank(cfg, adapter) if rank is None else rank
    h, d = proj_dims(cfg)[proj]
    rng = np.random.default_rng([DATA_SEED + cfg.index, 7 + seed_offset, adapter, layer, proj])
    A = _normal(rng, (h, r), 1.0 / np.sqrt(h))
    B = _normal(rng, (r, d), 1.0 / np.sqrt(r))
    return round_to(A, cfg.dtype), round_to(B, cfg.dtype)


def adapter_host_buffer(cfg: Config, adapter: int, num_layers: int, rank: int | None = None,
                        seed_offset: int = 0) -> np.ndarray:
    """Dense host buffer in the C-ABI's canonical layout (include/slora.h):
    for layer l, for projection p (q,k,v,o, then any proj_dims extras): A
    (h_p x r row-major) then B (r x d_p row-major), contiguous."""
    parts = []
    for l in range(num_layers):
        for p in range(len(proj_dims(cfg))):
            A, B = adapter_weights(cfg, adapter, l, p, rank, seed_offset)
            parts.append(A.ravel())
            parts.append(B.ravel())
    return np.concatenate(parts)


def activations(cfg: Config, T: int, width: int, tag: int, seed_offset: int = 0) -> np.ndarray:
    """T x width activations ~ N(0,1), stored dtype.  `tag` separates streams
    (e.g. x of layer l vs y_in of projection p)."""
    rng = np.random.default_rng([DATA_SEED + cfg.index, 11 + seed_offset, tag])
    return round_to(rng.standard_normal((T, width), dtype=np.float32), cfg.dtype)


def integer_weights(shape, rng, lo=-1, hi=1, max_nnz_per_col=None):
    """Small-integer values for the exact regime: entries in
    [lo, hi]; optionally at most `max_nnz_per_col` nonzeros per column."""
    M = rng.integers(lo, hi + 1, size=shape).astype(np.float32)
    if max_nnz_per_col is not None:
        rows, cols = shape
        mask = np.zeros(shape, bool)
        for c in range(cols):
            idx = rng.choice(rows, size=min(max_nnz_per_col, rows), replace=False)
            mask[idx, c] = True
        M = np.where(mask, M, 0).astype(np.float32)
    return M
