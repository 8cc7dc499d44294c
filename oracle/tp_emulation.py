"""S-LoRA tensor parallelism emulated on N logical devices, fp64
(TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Follows P:316-340 (Sec. 6, Fig. lora_tp), step by step, for one attention
layer with heterogeneous per-token adapters:

  qkv ("can be seen as W1"): W column-partitioned (Megatron);
      "A1 and B1 ... are column-partitioned.  An all-gather operation is used
      to collect the intermediate results".  Reading R4: A1 split
      along r, B1 along d.
        device k:  v_k = x A1_k              (B x r/N per token)
                   v   = all_gather(v_k)     (B x r)
                   y_k = x W1_k + v B1_k     (B x d/N columns of y)
  o ("can be seen as W2"): W2 row-partitioned; "A2 and B2 ... are
      row-partitioned and column-partitioned, respectively.  An all-reduce
      operation is used to sum up the intermediate results.  Finally, the
      result from the LoRA computation is added to that from the base model
      (add_2).  A single all-reduce operation is sufficient".
        device k:  P_k = z_k W2_k            (B x h partial sum)
                   u_k = z_k A2_k            (B x r partial sum)
                   u   = all_reduce(u_k)
                   P_k[:, k-th h/N slice] += u B2_k     (fold, reading R13)
                   out = all_reduce(P_k)
Collectives are emulated as ring algorithms over in-process arrays, and every
element a device sends is counted, so the P:337 volumes can be checked
against the traffic the emulation actually generated:
  base 2(N-1)Bh/N, LoRA 3(N-1)Br/N + 2(N-1)Br/N = 5(N-1)Br/N (uniform r);
  with heterogeneous ranks B*r becomes sum_i r_a(i).
"""
from __future__ import annotations

import numpy as np


class IndivisibleDimension(ValueError):
    pass


class Ring:
    """N logical devices; counts elements SENT by each device."""

    def __init__(self, N: int):
        self.N = N
        self.sent = [0] * N

    def all_gather(self, shards):
        """Ring all-gather of N equal shards (1-D).  Step s: device k sends the
        chunk it received at step s-1 (its own at s=0) to device k+1."""
        N = self.N
        n = shards[0].size
        bufs = [[None] * N for _ in range(N)]
        for k in range(N):
            bufs[k][k] = shards[k].copy()
        for s in range(N - 1):
            msgs = []
            for k in range(N):
                c = (k - s) % N
                msgs.append(((k + 1) % N, c, bufs[k][c]))
                self.sent[k] += n
            for dst, c, data in msgs:
                bufs[dst][c] = data.copy()
        return [np.concatenate(bufs[k]) for k in range(N)]

    def all_reduce(self, vecs):
        """Ring all-reduce (reduce-scatter then all-gather) of equal-length
        1-D vectors whose length is divisible by N."""
        N = self.N
        n = vecs[0].size
        if n % N:
            raise IndivisibleDimension(f"all_reduce length {n} % {N}")
        m = n // N
        chunks = [[v[c * m:(c + 1) * m].copy() for c in range(N)] for v in vecs]
        for s in range(N - 1):  # reduce-scatter
            msgs = []
            for k in range(N):
                c = (k - s) % N
                msgs.append(((k + 1) % N, c, chunks[k][c].copy()))
                self.sent[k] += m
            for dst, c, data in msgs:
                chunks[dst][c] = chunks[dst][c] + data
        for s in range(N - 1):  # all-gather of the reduced chunks
            msgs = []
            for k in range(N):
                c = (k + 1 - s) % N
                msgs.append(((k + 1) % N, c, chunks[k][c].copy()))
                self.sent[k] += m
            for dst, c, data in msgs:
                chunks[dst][c] = data
        return [np.concatenate(chunks[k]) for k in range(N)]


def _check(N, *dims):
    for dm in dims:
        if dm % N:
            raise IndivisibleDimension(f"{dm} % {N}")


def emulate_layer(N, x, z, Wq, Wk, Wv, Wo, adapters, slot):
    """One attention layer's q/k/v/o base + LoRA under S-LoRA TP on N devices.

    x: B x h (replicated input of q/k/v); z: B x d (input of o, i.e. the
    attention output; column-partitioned across devices as Megatron leaves it);
    W*: h x d (Wo: d x h); adapters[a] = {'q': (A, B), 'k': ..., 'v': ..., 'o': ...}
    with A: in x r, B: r x out; slot[i] = adapter of token i or -1.

    Returns (outputs dict with full 'q','k','v' (assembled from column shards)
    and 'o' (after the final all-reduce), counters dict with elements sent per
    device by the LoRA all-gathers, the LoRA all-reduce and the base
    all-reduce)."""
    B, h = x.shape
    d = Wq.shape[1]
    _check(N, h, d)
    ranks = [adapters[a]["q"][0].shape[1] for a in range(len(adapters))]
    for r in ranks:
        _check(N, r)
    tok = [i for i in range(B) if slot[i] >= 0]
    sum_r = sum(ranks[slot[i]] for i in tok)
    dN, hN = d // N, h // N
    ring_ag = Ring(N)
    ring_lora_ar = Ring(N)
    ring_base_ar = Ring(N)
    out = {}
    # ---------------- q, k, v: column partition, all-gather of x A1 ---------
    for name, W in (("q", Wq), ("k", Wk), ("v", Wv)):
        # shrink on each device with its column shard of A1
        v_shard = []
        for k in range(N):
            parts = []
            for i in tok:
                A = adapters[slot[i]][name][0]
                rN = A.shape[1] // N
                parts.append(x[i] @ A[:, k * rN:(k + 1) * rN])
            v_shard.append(np.concatenate(parts) if parts else np.zeros(0))
        # all-gather: device k receives everybody's shard
        if N > 1 and sum_r > 0:
            gathered = ring_ag.all_gather(v_shard)
        else:  # one device, or no adapted token: nothing to exchange
            gathered = v_shard
        y_cols = []
        for k in range(N):
            g = gathered[k]
            m = g.size // N if N > 0 else 0
            yk = x @ W[:, k * dN:(k + 1) * dN]
            off = 0
            for i in tok:
                A, Bm = adapters[slot[i]][name]
                rN = A.shape[1] // N
                # token i's full v = concat over source devices of its rN slice
                vi = np.concatenate([g[src * m + off: src * m + off + rN] for src in range(N)])
                off += rN
                yk[i] = yk[i] + vi @ Bm[:, k * dN:(k + 1) * dN]
            y_cols.append(yk)
        out[name] = np.concatenate(y_cols, axis=1)
    # ---------------- o: row partition, all-reduce, fold into base ----------
    P = []
    u_part = []
    for k in range(N):
        zk = z[:, k * dN:(k + 1) * dN]
        P.append(zk @ Wo[k * dN:(k + 1) * dN, :])
        parts = []
        for i in tok:
            A = adapters[slot[i]]["o"][0]
            parts.append(zk[i] @ A[k * dN:(k + 1) * dN, :])
        u_part.append(np.concatenate(parts) if parts else np.zeros(0))
    if N > 1 and sum_r > 0:
        u = ring_lora_ar.all_reduce(u_part)
    else:  # one device, or no adapted token: nothing to exchange
        u = u_part
    for k in range(N):
        off = 0
        for i in tok:
            Bm = adapters[slot[i]]["o"][1]
            r = Bm.shape[0]
            ui = u[k][off:off + r]
            off += r
            P[k][i, k * hN:(k + 1) * hN] += ui @ Bm[:, k * hN:(k + 1) * hN]  # add_2 fold
    if N > 1:
        final = ring_base_ar.all_reduce([p.ravel() for p in P])
        out["o"] = final[0].reshape(B, h)
    else:
        out["o"] = P[0]
    counters = {
        "lora_allgather_sent": ring_ag.sent,
        "lora_allreduce_sent": ring_lora_ar.sent,
        "base_allreduce_sent": ring_base_ar.sent,
        "sum_r": sum_r,
    }
    return out, counters


def shard_elements(N, h, d, r, n_proj_col=3):
    """Per-device weight elements of one adapter's shards and of the base
    weights under the partition above (memory optimality)."""
    _check(N, h, d, r)
    per_dev = []
    for _k in range(N):
        e = 0
        for _p in range(n_proj_col):
            e += h * (r // N) + r * (d // N) + h * (d // N)  # A1, B1, W1 shards
        e += (d // N) * r + r * (h // N) + (d // N) * h      # A2, B2, W2 shards
        per_dev.append(e)
    total = n_proj_col * (h * r + r * d + h * d) + (d * r + r * h + d * h)
    return per_dev, total
