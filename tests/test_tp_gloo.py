"""World-size-2 multi-process test of the S-LoRA TP orchestration
(paper_2311_03285_b200/tp.py) over torch.distributed gloo on CPU.

The compute steps are an in-test CPU emulation that writes/reads the C ABI's
documented v layout ([proj][segment][token][r/div], v_blocks rank blocks);
the collectives are real (gloo all_gather_into_tensor / all_reduce).  The
assembled result must equal the single-device oracle, and the exchanged
element counts must equal P:337."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

H, T, N = 64, 10, 2
RANKS = [8, 16, 4]
TOK = np.array([0, 1, 0, -1, 2, 2, 1, 0, 2, 1])


class EmuOps:
    """CPU stand-in for the library's shrink/expand on TP rank k."""

    def __init__(self, k, W):
        self.k, self.W = k, W
        self.segs = []                      # (adapter, tokens, vrow_off) first-appearance order
        order = []
        for a in TOK:
            if a >= 0 and a not in order:
                order.append(int(a))
        off = 0
        for a in order:
            toks = [i for i in range(T) if TOK[i] == a]
            self.segs.append((a, toks, off))
            off += len(toks) * RANKS[a]
        self.NR = off

    def v_elems(self, projs, div):
        return len(projs) * self.NR // div

    def shrink(self, layer, projs, x, ldx, v, stream):
        k, P = self.k, H // N
        for pi, pname in enumerate(projs):
            p = "qkvo".index(pname)
            div = N if p < 3 else 1
            for a, toks, voff in self.segs:
                r = RANKS[a]
                A = self.W[a][p][0]
                rl = r // div
                base = pi * self.NR // div + voff // div
                for ti, tok in enumerate(toks):
                    if p < 3:
                        val = x[tok].double().numpy() @ A[:, k * rl:(k + 1) * rl]
                    else:
                        val = x[tok].double().numpy() @ A[k * P:(k + 1) * P, :]
                    v[base + ti * rl: base + (ti + 1) * rl] = torch.from_numpy(val).float()

    def expand(self, layer, projs, v, vb, ys, ldys, stream):
        k, P = self.k, H // N
        names = [c for c in "qkvo" if c in projs]
        stride = len(names) * self.NR // vb
        for pi, pname in enumerate(names):
            p = "qkvo".index(pname)
            y = ys[p]
            for a, toks, voff in self.segs:
                r = RANKS[a]
                rb = r // vb
                B = self.W[a][p][1]
                base = pi * self.NR // vb + voff // vb
                for ti, tok in enumerate(toks):
                    full = np.array([float(v[(j // rb) * stride + base + ti * rb + (j % rb)]) for j in range(r)])
                    y[tok] += torch.from_numpy(full @ B[:, k * P:(k + 1) * P]).to(y.dtype)


def weights():
    rng = np.random.default_rng(3)
    return [[(rng.standard_normal((H, r)) / 8, rng.standard_normal((r, H)) / 4) for _ in range(4)] for r in RANKS]


def worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=N)
    try:
        from paper_2311_03285_b200.tp import TPLoraLayer
        import oracle
        W = weights()
        rng = np.random.default_rng(9)
        x = rng.standard_normal((T, H))
        z = rng.standard_normal((T, H))
        yin = [rng.standard_normal((T, H)) for _ in range(3)]
        base = [rng.standard_normal((T, H)) for _ in range(N)]
        P = H // N
        tpl = TPLoraLayer(EmuOps(rank, W))
        tpl.buffers_for()
        ysh = [torch.from_numpy(yin[p][:, rank * P:(rank + 1) * P].copy()) for p in range(3)]
        tpl.qkv(0, torch.from_numpy(x), H, ysh, [P] * 3)
        bp = torch.from_numpy(base[rank].copy())
        tpl.o(0, torch.from_numpy(z[:, rank * P:(rank + 1) * P].copy()), P, bp, H)
        dist.all_reduce(bp)                                   # the base layer's own all-reduce
        ids = [0, 1, 2]
        slot = np.array([a if a >= 0 else -1 for a in TOK])
        errs = []
        for p in range(3):
            ref = oracle.lora_apply(x, yin[p], [W[a][p][0] for a in ids], [W[a][p][1] for a in ids], slot)
            errs.append(float(np.abs(ysh[p].numpy() - ref[:, rank * P:(rank + 1) * P]).max()))
        ref = oracle.lora_apply(z, sum(base), [W[a][3][0] for a in ids], [W[a][3][1] for a in ids], slot)
        errs.append(float(np.abs(bp.numpy() - ref).max()))
        NR = sum(RANKS[a] for a in TOK if a >= 0)
        q.put((rank, errs, dict(tpl.sent_elems), NR))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_tp_orchestration_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, port, q)) for r in range(N)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(N)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, errs, sent, NR in res:
        assert max(errs) < 1e-5, (rank, errs)
        # all-gather 3(N-1)Br/N, all-reduce 2(N-1)Br/N (B r -> sum of ranks)
        assert sent["allgather"] == 3 * (N - 1) * NR // N
        assert sent["allreduce"] == 2 * (N - 1) * NR // N


class FakePool:
    """Records what LibraryTP hands the library (no device)."""
    tp_size = N

    def __init__(self, rank):
        self.tp_rank = rank
        self.opened = None

    def tp_init(self, uid, rank, size):
        self.init = (rank, size)

    def tp_p2p_export(self):
        return bytes([self.tp_rank + 1]) * 64

    def tp_p2p_open(self, handles):
        self.opened = [bytes(h) for h in handles]


def p2p_worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=N)
    try:
        from paper_2311_03285_b200 import slora as sl
        from paper_2311_03285_b200.tp import LibraryTP
        sl.tp_unique_id = lambda: b"u" * 128  # rank 0's NCCL id draw (no device here)
        pool = FakePool(rank)
        tpl = LibraryTP(pool)
        tpl.enable_p2p()
        q.put((rank, pool.init, pool.opened, tpl.p2p))
    finally:
        dist.destroy_process_group()


def test_tp_p2p_handle_exchange_world_size_2_gloo():
    """NEXT-3 host logic: every rank exports its exchange-region handle, the handles are
    all-gathered over torch.distributed and every rank opens the SAME list in rank order (the
    kernel indexes peers by rank)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=p2p_worker, args=(r, port, q)) for r in range(N)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(N))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(N)]
    for rank, init, opened, on in res:
        assert init == (rank, N) and on
        assert opened == want, (rank, opened)
