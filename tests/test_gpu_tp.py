"""S-LoRA tensor parallelism with N logical ranks on ONE GPU:
N pools (one per tp_rank, each holding only its shards in H/N pages), the
split shrink/expand kernels through the C ABI, and the collectives done by
plain torch ops (cat = all-gather, sum = all-reduce).  The assembled result
must match the single-device fp64 oracle.  Mark: gpu."""
import numpy as np
import pytest

from oracle import to_f64
from synth import workload as wl
from gpu_helpers import TOL, normalized_err, to_device

pytestmark = pytest.mark.gpu


def setup(cfg, batch, N, layers=1):
    from paper_2311_03285_b200 import Batch, Pool
    pools, batches, weights = [], [], {}
    for a in batch.unique:
        r = batch.ranks[a]
        weights[a] = [wl.adapter_weights(cfg, a, l, p, r) for l in range(layers) for p in range(4)]
    for k in range(N):
        need = sum(layers * 8 * r for r in batch.ranks.values())
        pool = Pool(cfg.hidden, layers, need + 64, dtype=cfg.dtype, device=0, tp_size=N, tp_rank=k,
                    order="shuffle", seed=k + 1)
        for a in batch.unique:
            host = np.concatenate([np.concatenate([A.ravel(), B.ravel()]) for A, B in weights[a]])
            pool.adapter_load(a, batch.ranks[a], host)
        b = Batch(pool)
        b.prepare(batch.token_adapter)
        pools.append(pool)
        batches.append(b)
    return pools, batches, weights


def oracle_ref(cfg, batch, weights, x, y_in, layer, proj):
    import oracle
    ids = batch.unique
    slot = np.array([ids.index(a) if a >= 0 else -1 for a in batch.token_adapter])
    return oracle.lora_apply(to_f64(x, cfg.dtype), y_in,
                             [to_f64(weights[a][layer * 4 + proj][0], cfg.dtype) for a in ids],
                             [to_f64(weights[a][layer * 4 + proj][1], cfg.dtype) for a in ids], slot)


@pytest.mark.parametrize("N,name", [(2, "c2"), (4, "c3"), (8, "c4")])
def test_tp_sharded_matches_oracle(N, name):
    import torch
    cfg = wl.CONFIGS[name]
    if name == "c4":
        cfg = wl.Config(cfg.name, cfg.index, cfg.hidden, cfg.n_adapters, cfg.rank_list, cfg.dtype, 1.0, 64,
                        tp=8, num_layers=1)
    batch = wl.make_batch(cfg)
    T, H = batch.T, cfg.hidden
    P = H // N
    pools, batches, weights = setup(cfg, batch, N)
    x = wl.activations(cfg, T, H, 1)
    xd = to_device(x, cfg.dtype)
    # ---- q, k, v: shrink (A1 column shard) -> all-gather -> expand (B1 col shard)
    n_local = batches[0].v_elems("qkv", N)
    v_local = [torch.empty(n_local, dtype=torch.float32, device="cuda") for _ in range(N)]
    for k in range(N):
        batches[k].shrink(0, "qkv", xd, H, v_local[k])
    v_all = torch.cat(v_local)                      # all-gather (rank-major blocks)
    yin = [wl.activations(cfg, T, H, 10 + p) for p in range(3)]
    yshard = [[to_device(np.ascontiguousarray(yin[p][:, k * P:(k + 1) * P]), cfg.dtype) for p in range(3)]
              for k in range(N)]
    for k in range(N):
        ys = yshard[k] + [None]
        batches[k].expand(0, "qkv", v_all, N, ys, [P, P, P, 0])
    torch.cuda.synchronize()
    for p in range(3):
        got = np.concatenate([yshard[k][p].double().cpu().numpy() for k in range(N)], axis=1)
        ref = oracle_ref(cfg, batch, weights, x, to_f64(yin[p], cfg.dtype), 0, p)
        assert normalized_err(got, ref) <= TOL[cfg.dtype], p
    # ---- o: shrink (A2 row shard, x column shard) -> all-reduce -> expand into
    #         column slice k of the base partial sum, then the base all-reduce
    z = wl.activations(cfg, T, H, 20)
    n_o = batches[0].v_elems("o", 1)
    u_part = []
    for k in range(N):
        zk = to_device(np.ascontiguousarray(z[:, k * P:(k + 1) * P]), cfg.dtype)
        u = torch.empty(n_o, dtype=torch.float32, device="cuda")
        batches[k].shrink(0, "o", zk, P, u)
        u_part.append(u)
    u_sum = torch.stack(u_part).sum(0)              # all-reduce of the B x r partials
    base = [wl.activations(cfg, T, H, 30 + k) for k in range(N)]   # base partial sums P_k
    base_d = [to_device(b, cfg.dtype) for b in base]
    for k in range(N):
        ys = [None, None, None, base_d[k][:, k * P:(k + 1) * P]]
        batches[k].expand(0, "o", u_sum, 1, ys, [0, 0, 0, H])   # fold into slice k (add_2)
    torch.cuda.synchronize()
    got = sum(base_d[k].double().cpu().numpy() for k in range(N))   # base all-reduce
    yin_o = sum(to_f64(b, cfg.dtype) for b in base)
    ref = oracle_ref(cfg, batch, weights, z, yin_o, 0, 3)
    assert normalized_err(got, ref) <= TOL[cfg.dtype]
    # exchanged LoRA elements match P:337 (per device: all-gather receives
    # 3(N-1)/N * sum_r, all-reduce 2(N-1)/N * sum_r)
    NR = batches[0].info()["sum_rank_tokens"]
    assert n_local * N == 3 * NR and n_o == NR
