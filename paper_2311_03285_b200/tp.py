"""S-LoRA tensor parallelism over torch.distributed (Sec. 6.1,
P:316-331; Fig. lora_tp), one process per GPU.

Per attention layer on rank k of N (readings R3/R4/R13 in DESIGN.md):
  q, k, v  ("can be seen as W1"): A1 column shard (r/N rank columns),
           B1 column shard (d/N output columns).
             v_k = x A1_k                 slora_lora_shrink  (fp32, B x r/N)
             v   = all_gather(v_k)        one concatenated collective for
                                          q, k and v (reading R14)
             y_k += v B1_k                slora_lora_expand (v_blocks = N)
  o        ("can be seen as W2"): A2 row shard, B2 column shard.
             u_k = z_k A2_k               slora_lora_shrink  (fp32 partial, B x r)
             u   = all_reduce(u_k)
             P_k[:, k-th h/N slice] += u B2_k   slora_lora_expand into the base
                                          partial sum (add_2 fold): the base
                                          layer's own all-reduce then carries
                                          the LoRA result.
The compute steps are the library's CUDA kernels; this module only orders
them around the two collectives and owns the exchange buffers.  Element
counts exchanged per device equal: 3(N-1)/N * NR for the all-gather
and 2(N-1)/N * NR for the all-reduce (NR = sum over tokens of the rank).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class LibraryOps:
    """The compute steps, bound to a prepared slora Batch (CUDA kernels)."""

    def __init__(self, batch):
        self.batch = batch

    def v_elems(self, projs, div):
        return self.batch.v_elems(projs, div)

    def shrink(self, layer, projs, x, ldx, v, stream):
        self.batch.shrink(layer, projs, x, ldx, v, stream)

    def expand(self, layer, projs, v, v_blocks, ys, ldys, stream):
        self.batch.expand(layer, projs, v, v_blocks, ys, ldys, stream)


class TPLoraLayer:
    """Orchestrates shrink -> collective -> expand on one rank.

    `ops` provides v_elems/shrink/expand (LibraryOps on a GPU; tests inject a
    CPU emulation to exercise the exchange logic with gloo)."""

    def __init__(self, ops, group=None, device=None):
        self.ops = ops
        self.group = group
        self.N = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.device = device
        self._buf = {}
        self.sent_elems = {"allgather": 0, "allreduce": 0}

    def _get(self, key, n):
        t = self._buf.get(key)
        if t is None or t.numel() < n:
            t = torch.empty(max(n, 1), dtype=torch.float32, device=self.device)
            self._buf[key] = t
        return t[:n]

    def buffers_for(self):
        """Pre-size exchange buffers (call after batch prepare)."""
        n_loc = self.ops.v_elems("qkv", self.N)
        self._get("v_loc", n_loc)
        self._get("v_all", n_loc * self.N)
        self._get("u", self.ops.v_elems("o", 1))

    def qkv(self, layer, x, ldx, y_shards, ld_y, stream=None):
        """y_shards: q, k, v column shards (T x H/N each)."""
        n_loc = self.ops.v_elems("qkv", self.N)
        if n_loc == 0:
            return
        v_loc = self._get("v_loc", n_loc)
        self.ops.shrink(layer, "qkv", x, ldx, v_loc, stream)
        if self.N > 1:
            v_all = self._get("v_all", n_loc * self.N)
            dist.all_gather_into_tensor(v_all, v_loc, group=self.group)
            self.sent_elems["allgather"] += (self.N - 1) * n_loc
        else:
            v_all = v_loc
        self.ops.expand(layer, "qkv", v_all, self.N, list(y_shards) + [None], list(ld_y) + [0], stream)

    def o(self, layer, z_shard, ldz, base_partial, ld_base, stream=None):
        """z_shard: this rank's T x H/N slice of the attention output;
        base_partial: this rank's T x H base partial sum (z_k W2_k).  The LoRA
        output lands in its column slice k; the caller's base all-reduce then
        completes both (fold)."""
        n = self.ops.v_elems("o", 1)
        if n == 0:
            return
        u = self._get("u", n)
        self.ops.shrink(layer, "o", z_shard, ldz, u, stream)
        if self.N > 1:
            dist.all_reduce(u, group=self.group)
            self.sent_elems["allreduce"] += 2 * (self.N - 1) * n // self.N
        P = base_partial.shape[1] // self.N
        y_slice = base_partial[:, self.rank * P:(self.rank + 1) * P]
        self.ops.expand(layer, "o", u, 1, [None, None, None, y_slice], [0, 0, 0, ld_base], stream)


class LibraryTP:
    """S-LoRA TP through the C ABI (slora_tp_*): the library's own NCCL
    communicator carries the all-gather and the all-reduce between its shrink
    and expand kernels, on the caller's stream (graph-capturable).
    torch.distributed only bootstraps it: rank 0 draws the NCCL unique id and
    broadcasts the 128 bytes (include/slora.h a6/a8)."""

    def __init__(self, pool, group=None):
        from .slora import tp_unique_id
        self.pool = pool
        self.N, self.rank = pool.tp_size, pool.tp_rank
        uid = tp_unique_id() if self.rank == 0 else None
        if self.N > 1:
            obj = [uid]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = obj[0]
        pool.tp_init(uid, self.rank, self.N)

    def enable_p2p(self, group=None):
        """NEXT-3: map every rank's exchange region (CUDA IPC handles all-gathered over
        torch.distributed); qkv/o then run the fused device-initiated kernels."""
        h = self.pool.tp_p2p_export()
        handles = [h]
        if self.N > 1:
            handles = [None] * self.N
            dist.all_gather_object(handles, h, group=group)
        self.pool.tp_p2p_open(handles)
        self.p2p = True

    p2p = False

    def qkv(self, batch, layer, x, ldx, y_shards, ld_y, stream=None):
        if self.p2p:
            batch.tp_fused_qkv(layer, x, ldx, list(y_shards), list(ld_y), stream)
        else:
            batch.tp_qkv(layer, x, ldx, list(y_shards), list(ld_y), stream)

    def o(self, batch, layer, z_shard, ldz, base_partial, ld_base, stream=None):
        if self.p2p:
            batch.tp_fused_o(layer, z_shard, ldz, base_partial, ld_base, stream)
        else:
            batch.tp_o(layer, z_shard, ldz, base_partial, ld_base, stream)

    def stats(self):
        return self.pool.tp_stats()
