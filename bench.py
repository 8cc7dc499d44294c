#!/usr/bin/env python
"""Benchmark of the S-LoRA hot path on B200 (BASELINE.json metric:
"LoRA-layer tokens/s and achieved HBM GB/s vs peak at 1/2/4/8 B200").

One STEP = one pass of the whole hot path over one synthetic batch:
  a4 batch descriptor (slora_batch_prepare: group by adapter, pack units,
     upload), then for each of the model's layers
  a5+a7 q/k/v fused shrink->expand (one launch) and o fused shrink->expand
     (one launch) -- on N > 1 GPUs the library's TP calls (slora_tp_lora_qkv:
     shrink -> NCCL all-gather -> expand; slora_tp_lora_o: shrink -> NCCL
     all-reduce -> expand into the base partial, a6 + a8 fold).
value = adapted tokens x layers / step time (LoRA-layer tokens/s, i.e.
T / per-layer LoRA time), whole job.  Default workload: BASELINE configs[2]
decode (Llama-7B h=4096, 2000 adapters, ranks {64,32,16,8} round-robin,
Zipf alpha=1, decode batch 64, fp16) -- the north_star's ">= 70% of HBM"
target.  Weights of 32 layers (~3.5 GB) rotate through the timed region, far
larger than the 126 MB L2 (no flush needed; stated in config).  The line also
nests the other BASELINE configs measured the same way ("secondary"), each
with its own roofline, and the two NEXT-2 ablations ("ablations").

--impl reference: the fp64 CPU oracle (oracle/), timed on host cores on a
bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import workload as wl  # noqa: E402

METRIC = "LoRA-layer tokens/s and achieved HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, help="c1 | c2 | c2-mixed | c3 | c4 (default: c2)")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the nested secondary configs / ablations")
    ap.add_argument("--profile-steps", type=int, default=0, help="untimed steps only (for ncu)")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph replay")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ setup
class Workload:
    def __init__(self, cfg, layers, tp, rank, device, stream, order=None, kv_tokens=16, tp_path=None):
        import torch
        from paper_2311_03285_b200 import Batch, Pool
        self.cfg, self.L, self.N, self.k = cfg, layers, tp, rank
        # the TP calls (slora_tp_*) serve the layers when N > 1, or on one GPU with SLORA_BENCH_TP=1
        self.tp_path = (tp > 1) if tp_path is None else tp_path
        self.batch = wl.make_batch(cfg)
        b = self.batch
        self.T, self.H = b.T, cfg.hidden
        self.P = self.H // tp
        es = wl.elem_bytes(cfg.dtype)
        need = sum(layers * 8 * r for r in b.ranks.values())
        # KV pages of every request interleaved with adapter pages; order: page placement
        kv_pages = 2 * kv_tokens * layers * len(b.requests)
        order = order or os.environ.get("SLORA_BENCH_ORDER", "shuffle")
        self.pool = Pool(self.H, layers, need + kv_pages + 64, dtype=cfg.dtype, device=device, tp_size=tp,
                         tp_rank=rank, order=order, seed=1234 + rank, max_adapters=max(256, len(b.ranks) + 8))
        rid = 0
        reqs = list(b.requests)
        load_s, load_bytes = 0.0, 0
        for i, a in enumerate(b.unique):
            if rid < len(reqs) and kv_tokens:
                self.pool.kv_alloc(rid, kv_tokens)
                rid += 1
            host = wl.adapter_host_buffer(cfg, a, layers)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.pool.adapter_load(a, b.ranks[a], host, stream=stream)
            torch.cuda.synchronize()
            load_s += time.perf_counter() - t0
            load_bytes += host.nbytes
        # a2: host -> pool adapter load (pageable numpy buffer -> library's pinned
        # staging -> H2D -> page scatter), synchronous per adapter
        self.load = {"adapters": len(b.unique), "bytes": int(load_bytes), "ms": round(1e3 * load_s, 3),
                     "GBps": round(load_bytes / max(load_s, 1e-9) / 1e9, 2),
                     "note": "full (unsharded) host tensors of all layers; this rank copies its 1/N shard"}
        while rid < len(reqs) and kv_tokens:
            self.pool.kv_alloc(rid, kv_tokens)
            rid += 1
        torch.cuda.synchronize()
        self.tpl = None
        if self.tp_path:  # the library's NCCL communicator (bootstrapped over torch.distributed)
            from paper_2311_03285_b200.tp import LibraryTP
            self.tpl = LibraryTP(self.pool)
        self.dbatch = Batch(self.pool)
        self.dbatch.prepare(b.token_adapter, stream=stream)
        # a4: batch descriptor (grouping, work lists, LPT schedule, upload), host time per prepare
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            self.dbatch.prepare(b.token_adapter, stream=stream)
        self.prepare_us = round((time.perf_counter() - t0) / 20 * 1e6, 1)
        torch.cuda.synchronize()
        td = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[cfg.dtype]
        self.td = td
        dev = f"cuda:{device}"
        g = torch.Generator(device=dev).manual_seed(5 + rank)
        # activations resident in HBM: x per layer, y per (layer, proj)
        self.x = torch.randn((layers, self.T, self.H), generator=g, device=dev).to(td)
        if not self.tp_path:
            self.y = torch.randn((layers, 4, self.T, self.H), generator=g, device=dev).to(td)
        else:
            self.y = torch.randn((layers, 3, self.T, self.P), generator=g, device=dev).to(td)
            self.z = torch.randn((layers, self.T, self.P), generator=g, device=dev).to(td)
            self.base = torch.randn((layers, self.T, self.H), generator=g, device=dev).to(td)
        self.es = es
        # algorithmic bytes per step: unique-adapter weight shards
        # + x once per call + y read+write; tables excluded (KB-sized)
        Tad = int((b.token_adapter >= 0).sum())
        wbytes = sum(r * 2 * self.P * es for r in b.ranks.values())  # per projection, this rank's shard
        if tp == 1:
            self.bytes_qkv = 3 * wbytes + Tad * self.H * es + 3 * 2 * Tad * self.H * es
            self.bytes_o = wbytes + Tad * self.H * es + 2 * Tad * self.H * es
        else:
            self.bytes_qkv = 3 * wbytes + Tad * self.H * es + 3 * 2 * Tad * self.P * es
            self.bytes_o = wbytes + Tad * self.P * es + 2 * Tad * self.P * es
        self.Tad = Tad
        self.flops_layer = sum(4 * 2 * r * 2 * self.H // tp for r in
                               [b.ranks[a] for a in b.token_adapter if a >= 0])

    graph = None

    def close(self):
        import torch
        self.graph = None
        self.dbatch.close()
        self.pool.close()
        del self.x, self.y
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def capture(self, stream):
        """Capture the layer sequence (launches + the library's NCCL calls)
        into a CUDA graph; the per-step batch_prepare stays outside (host work
        + descriptor upload), as in a serving loop that replays a decode graph
        every iteration."""
        import torch
        self.dbatch.prepare(self.batch.token_adapter, stream=stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        with torch.cuda.graph(g, stream=cs):
            self.layers(torch.cuda.current_stream())
        torch.cuda.synchronize()
        self.graph = g

    def rotating_maps(self, n, seed=99):
        """n decode token maps over the resident adapters, each a different batch with the SAME
        work: adapters permuted within each rank class (so segment sizes per rank are kept) and
        token order shuffled -- a serving loop's batch changes every iteration."""
        rng = np.random.default_rng(seed)
        tok = self.batch.token_adapter
        ads = sorted(set(int(a) for a in tok if a >= 0))
        maps = []
        for _ in range(n):
            perm = {}
            for r in sorted(set(self.batch.ranks[a] for a in ads)):
                cls = [a for a in ads if self.batch.ranks[a] == r]
                for a, b2 in zip(cls, rng.permutation(cls)):
                    perm[a] = int(b2)
            m = np.array([perm[int(a)] if a >= 0 else -1 for a in tok], np.int64)
            maps.append(m[rng.permutation(len(m))])
        return maps

    def step(self, stream, events=None, token_map=None):
        """One step: prepare + all layers.  events: list to append
        (start, end, kind) CUDA event pairs around each launch."""
        b = self.dbatch
        b.prepare(self.batch.token_adapter if token_map is None else token_map, stream=stream)
        if self.graph is not None and events is None:
            self.graph.replay()
            return
        self.layers(stream, events)

    def packed_calls(self):
        """The step's 2 x L fused calls packed once for slora_lora_apply_many (single GPU)."""
        if getattr(self, "_packed", None) is None:
            from paper_2311_03285_b200 import Batch
            H = self.H
            calls = []
            for l in range(self.L):
                ys = [self.y[l, p] for p in range(4)]
                calls.append((l, "qkv", self.x[l], H, ys, [H] * 4))
                calls.append((l, "o", self.x[l], H, ys, [H] * 4))
            self._packed = Batch.make_calls(calls)
        return self._packed

    def layers(self, stream, events=None):
        import torch
        b = self.dbatch
        H, P = self.H, self.P
        for l in range(self.L):
            e0 = torch.cuda.Event(enable_timing=True) if events is not None else None
            if e0:
                e0.record(stream)
            if not self.tp_path:
                ys = [self.y[l, p] for p in range(4)]
                b.apply(l, "qkv", self.x[l], H, ys, [H] * 4, stream=stream)
            else:
                self.tpl.qkv(b, l, self.x[l], H, [self.y[l, p] for p in range(3)], [P, P, P], stream=stream)
            if e0:
                e1 = torch.cuda.Event(enable_timing=True); e1.record(stream)
                e2 = torch.cuda.Event(enable_timing=True); e2.record(stream)
            if not self.tp_path:
                b.apply(l, "o", self.x[l], H, ys, [H] * 4, stream=stream)
            else:
                self.tpl.o(b, l, self.z[l], P, self.base[l], H, stream=stream)
            if e0:
                e3 = torch.cuda.Event(enable_timing=True); e3.record(stream)
                events.append((e0, e1, "qkv"))
                events.append((e2, e3, "o"))


def timed_steps(W, stream, steps, ws):
    """K steps bracketed by barrier + synchronize; per-step CUDA events on the
    launching stream (between steps: the prepare is part of a step).  Returns
    (mean ms, per-step ms list), max over ranks for the mean."""
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        W.step(stream)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    ms = ev[0].elapsed_time(ev[steps]) / steps
    if ws > 1:
        tt = torch.tensor([ms], device=f"cuda:{torch.cuda.current_device()}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return ms, per


def lora_comm_overhead(W, stream, steps):
    """P:532 ("S-LoRA with and without LoRA communication"): the TP step replayed from a graph
    with the library's collectives (slora_tp_lora_qkv / _o) and from a graph of the same shrink
    and expand kernels with the exchange steps left out (slora_lora_shrink / _expand on
    workspaces: results not meaningful, timing only).  Device time per step of each."""
    import torch
    b, N, k, H, P = W.dbatch, W.N, W.k, W.H, W.P
    vloc = torch.zeros(b.v_elems("qkv", N), dtype=torch.float32, device="cuda")
    vall = torch.zeros(b.v_elems("qkv", 1), dtype=torch.float32, device="cuda")
    u = torch.zeros(b.v_elems("o", 1), dtype=torch.float32, device="cuda")

    def nocomm():
        st = torch.cuda.current_stream()
        for l in range(W.L):
            b.shrink(l, "qkv", W.x[l], H, vloc, stream=st)
            b.expand(l, "qkv", vall, N, [W.y[l, p] for p in range(3)], [P] * 3, stream=st)
            b.shrink(l, "o", W.z[l], P, u, stream=st)
            ys = W.base[l][:, k * P:(k + 1) * P]
            b.expand(l, "o", u, 1, [None, None, None, ys], [0, 0, 0, H], stream=st)

    def timed(replay):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for _ in range(2):
            replay()
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(steps):
            b.prepare(W.batch.token_adapter, stream=stream)
            replay()
        ev[1].record(stream)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / steps

    nocomm()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        nocomm()
    with_ms = timed(W.graph.replay)
    without_ms = timed(g.replay)
    return {"with_lora_comm_ms": round(with_ms, 4), "without_lora_comm_ms": round(without_ms, 4),
            "overhead": round(with_ms / without_ms - 1.0, 4),
            "note": "P:532: the same TP step with and without the q/k/v all-gather and o all-reduce of the LoRA "
                    "intermediate (graph replays, device time per step)"}


def tp_p2p_step(W, stream, steps, nccl_ms):
    """NEXT-3: the TP step through slora_tp_fused_qkv / _o (one kernel per call: the v exchange
    by NVLink peer stores + system-scope counters instead of NCCL), graph replay, device time."""
    import torch
    W.tpl.enable_p2p()
    W.dbatch.prepare(W.batch.token_adapter, stream=stream)
    torch.cuda.synchronize()
    W.layers(torch.cuda.current_stream())  # eager once (builds nothing new: prepare did)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        W.layers(torch.cuda.current_stream())
    for _ in range(2):
        W.dbatch.prepare(W.batch.token_adapter, stream=stream)
        g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(steps):
        W.dbatch.prepare(W.batch.token_adapter, stream=stream)
        g.replay()
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    return {"ms_per_step": round(ms, 4), "vs_nccl_path": round(ms / nccl_ms, 3), "launches_per_layer": 2,
            "note": "slora_tp_fused_qkv/_o: shrink -> peer stores of v into every rank's exchange region -> "
                    "expand in one kernel per call (NCCL path: 4 kernels + 2 collectives per layer)"}


def base_lora_overlap(W, stream, steps=10, wl_layers=8):
    """P:631 ("the use of multiple CUDA streams to parallelize base model and LoRA
    computations"): the decode step's base projections (y = x W for q,k,v,o of every layer:
    cuBLAS GEMMs, T x 4096 x 4096 fp16, 8 distinct weight sets cycled, 1 GB) on one stream and
    the LoRA step (the captured graph) on another.  Reported: each alone, both concurrently,
    and the fraction of the LoRA time hidden under the base GEMMs.  The LoRA deltas go to their
    own y buffers here (a real layer adds them into the base output afterwards: T x d adds)."""
    import torch
    H, T, L = W.H, W.T, W.L
    td = W.td
    g = torch.Generator(device="cuda").manual_seed(11)
    Wb = torch.randn((wl_layers, 4, H, H), generator=g, device="cuda").to(td).mul_(1.0 / np.sqrt(H))
    yb = torch.empty((4, T, H), dtype=td, device="cuda")
    s_base = torch.cuda.Stream()

    def base():
        for l in range(L):
            for p in range(4):
                torch.matmul(W.x[l], Wb[l % wl_layers, p], out=yb[p])

    def timed(fn_list):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        evs = []
        for fn, st in fn_list:
            st.wait_event(e0) if st is not stream else None
            with torch.cuda.stream(st):
                for _ in range(steps):
                    fn()
            ev = torch.cuda.Event()
            ev.record(st)
            evs.append(ev)
        for ev in evs:
            stream.wait_event(ev)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    lora = lambda: W.step(stream)  # noqa: E731  prepare + graph replay (stream is current inside timed)
    base()  # cuBLAS handle / workspace for this stream, then the base step as a graph (no host launch cost)
    torch.cuda.synchronize()
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=s_base):
        base()
    base_g = gb.replay
    res = {}
    for _ in range(2):  # the second round is reported (first-use costs in the first)
        res["base"] = timed([(base_g, s_base)])
        res["lora"] = timed([(lora, stream)])
        res["both"] = timed([(base_g, s_base), (lora, stream)])
    t_base, t_lora, t_both = res["base"], res["lora"], res["both"]
    del Wb, yb, gb
    torch.cuda.empty_cache()
    return {"base_ms": round(t_base, 4), "lora_ms": round(t_lora, 4), "both_ms": round(t_both, 4),
            "lora_hidden_fraction": round(max(0.0, min(1.0, (t_base + t_lora - t_both) / t_lora)), 3),
            "note": "per step: 32 layers x q,k,v,o base GEMMs (torch.matmul / cuBLAS, replayed from a graph) on one "
                    "stream, the LoRA step graph on another; hidden = (base + lora - both) / lora"}


def rotating_steps(W, stream, steps):
    """Like timed_steps, but every step prepares a different batch (re-drawn token maps over
    the resident adapters) and replays the SAME graph: the launches read the descriptors
    prepare just rewrote (fixed-address call headers).  Also the host time per step."""
    import torch
    maps = W.rotating_maps(8)
    for m in maps[:3]:
        W.step(stream, token_map=m)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    t0 = time.perf_counter()
    for i in range(steps):
        W.step(stream, token_map=maps[i % len(maps)])
    host_ms = (time.perf_counter() - t0) * 1e3 / steps
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    W.dbatch.prepare(W.batch.token_adapter, stream=stream)
    torch.cuda.synchronize()
    return {"ms_per_step": round(ms, 4), "host_ms_per_step": round(host_ms, 4), "batches": len(maps),
            "note": "every step: slora_batch_prepare of a different decode batch (adapters permuted within each "
                    "rank class, token order shuffled: same work, new descriptors) + replay of the one captured "
                    "graph; host time includes prepare waiting for the previous step's upload"}


def roofline_of(W, ms, stream, serialized=True):
    """Roofline of the step: algorithmic bytes / time per step (the launches
    run back to back, prepare included: a conservative average launch
    duration); serialized per-launch durations from a separate pass."""
    import torch
    peaks, peak_kind = measured_peaks()
    bytes_step = (W.bytes_qkv + W.bytes_o) * W.L
    achieved = bytes_step / (ms / 1e3) / 1e9
    r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
         "frac": round(achieved / peaks["hbm_gbs"], 4),
         "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
         "alg_bytes_per_launch": {"qkv": W.bytes_qkv, "o": W.bytes_o},
         "avg_launch_us_in_step": round(1e3 * ms / (2 * W.L), 2),
         "frac_of_8TBs_spec": round(achieved / 8000.0, 4)}
    if serialized:
        events = []
        for _ in range(3):
            W.step(stream, events=events)
        torch.cuda.synchronize()
        dur = {"qkv": [], "o": []}
        for a, b, kind in events:
            dur[kind].append(a.elapsed_time(b))
        r["serialized_launch_us"] = {"qkv": round(1e3 * float(np.mean(dur["qkv"])), 2),
                                     "o": round(1e3 * float(np.mean(dur["o"])), 2)}
        r["serialized_kernel_ms_per_step"] = round((sum(dur["qkv"]) + sum(dur["o"])) / 3, 4)
    return r


def measure(name, layers, steps, warmup, stream, graph=True):
    """A secondary config measured like the headline (graph replay, events)."""
    import torch
    cfg = wl.CONFIGS[name]
    W = Workload(cfg, layers, 1, 0, torch.cuda.current_device(), stream)
    for _ in range(max(3, warmup)):
        W.step(stream)
    if graph:
        W.capture(stream)
        for _ in range(2):
            W.step(stream)
    ms, per = timed_steps(W, stream, steps, 1)
    out = {"workload": cfg.name, "dtype": cfg.dtype, "hidden": cfg.hidden, "layers": layers, "tokens": W.T,
           "adapted_tokens": W.Tad, "unique_adapters": len(W.batch.ranks),
           "ms_per_step": round(ms, 4), "value": round(W.Tad * layers / (ms / 1e3), 1), "unit": UNIT,
           "p10_p50_p90_ms": [round(float(v), 4) for v in np.percentile(per, [10, 50, 90])],
           "mbgmm_segments": W.dbatch.info()["mbgmm_segments"],
           "roofline": roofline_of(W, ms, stream, serialized=False)}
    W.close()
    return out


def measure_mlp(stream, layers=8, steps=10):
    """NEXT-4 secondary: C2's decode batch with LoRA on all seven Llama-7B projections
    (q,k,v,o 4096 -> 4096; MLP gate/up 4096 -> 11008, down 11008 -> 4096: stored rows over 3
    pages), 4 fused calls per layer grouped by input width, graph replay like the headline.
    Weight CONTENT is immaterial to the timing: one host buffer per rank serves every adapter
    of that rank (the parity of these shapes is tests/test_gpu_proj_shapes.py)."""
    import torch
    from paper_2311_03285_b200 import Batch, Pool
    cfg = wl.CONFIGS["c2-mlp"]
    dims = wl.proj_dims(cfg)
    b0 = wl.make_batch(cfg)
    H, es = cfg.hidden, wl.elem_bytes(cfg.dtype)
    units = sum(-(-i // H) + -(-o // H) for i, o in dims)
    need = sum(layers * r * units for r in b0.ranks.values())
    pool = Pool(H, layers, need + 64, dtype=cfg.dtype, device=torch.cuda.current_device(), order="shuffle",
                seed=1234, max_adapters=len(b0.ranks) + 8, proj_dims=dims)
    bufs = {r: wl.adapter_host_buffer(cfg, 100_000 + r, layers, rank=r) for r in set(b0.ranks.values())}
    for a in b0.unique:
        pool.adapter_load(a, b0.ranks[a], bufs[b0.ranks[a]], stream=stream)
    torch.cuda.synchronize()
    b = Batch(pool)
    b.prepare(b0.token_adapter, stream=stream)
    T = b0.T
    td = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[cfg.dtype]
    g = torch.Generator(device="cuda").manual_seed(9)
    calls = [(0, 1, 2), (3,), (4, 5), (6,)]
    xs = {c: torch.randn((layers, T, dims[c[0]][0]), generator=g, device="cuda").to(td) for c in calls}
    ys = [torch.randn((layers, T, o), generator=g, device="cuda").to(td) for _, o in dims]
    ld = [o for _, o in dims]

    def run_layers():
        for l in range(layers):
            for c in calls:
                b.apply(l, list(c), xs[c][l], dims[c[0]][0], [y[l] for y in ys], ld,
                        stream=torch.cuda.current_stream())

    def step():
        b.prepare(b0.token_adapter, stream=stream)
        gr.replay()

    run_layers()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(gr, stream=cs):
        run_layers()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(stream)
    for i in range(steps):
        step()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[steps]) / steps
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    Tad = int((b0.token_adapter >= 0).sum())
    wb = sum(sum(r * (i + o) * es for i, o in dims) for r in b0.ranks.values())
    act = sum(Tad * dims[c[0]][0] * es for c in calls) + sum(2 * Tad * o * es for _, o in dims)
    bytes_step = layers * (wb + act)
    peaks, kind = measured_peaks()
    achieved = bytes_step / (ms / 1e3) / 1e9
    out = {"workload": cfg.name, "dtype": cfg.dtype, "hidden": H, "proj_dims": [list(d) for d in dims],
           "layers": layers, "tokens": T, "adapted_tokens": Tad, "unique_adapters": len(b0.ranks),
           "calls_per_layer": ["q,k,v", "o", "gate,up", "down"],
           "ms_per_step": round(ms, 4), "value": round(Tad * layers / (ms / 1e3), 1), "unit": UNIT,
           "p10_p50_p90_ms": [round(float(v), 4) for v in np.percentile(per, [10, 50, 90])],
           "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": round(achieved / peaks["hbm_gbs"], 4), "alg_bytes_per_layer": int(wb + act),
                        "peak_source": f"{kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)"},
           "note": "value counts adapted tokens x layers (each layer = 7 LoRA'd projections); 8 layers of "
                   "adapter pages (%.1f GB) rotate, >> L2" % (layers * wb / 1e9)}
    b.close()
    pool.close()
    del xs, ys
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def traffic_record(cfg_name):
    """Measured DRAM bytes per launch of the hot kernel: a STATIC record from
    the committed ncu capture (profiles/ncu_summary.json), not this run."""
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        if prof.get("workload") == cfg_name:
            return {"per_launch_bytes": prof.get("dram_bytes_per_launch"), "source":
                    "static: profiles/ncu_summary.json (ncu --set full of one layer, committed)"}
    except Exception:
        pass
    return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2311_03285_b200 import launch_count

    ws, rank, local = dist_env()
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    name = args.workload or "c2"
    cfg = wl.CONFIGS[name]
    layers = args.layers or cfg.num_layers
    if name == "c0":
        layers = 1
    stream = torch.cuda.current_stream()
    tp_path = ws > 1 or os.environ.get("SLORA_BENCH_TP") == "1"
    W = Workload(cfg, layers, ws, rank, local, stream, tp_path=tp_path)
    if args.profile_steps:
        for _ in range(args.profile_steps):
            W.step(stream)
        torch.cuda.synchronize()
        return
    warm = max(3, args.warmup)
    for _ in range(warm):
        W.step(stream)
    torch.cuda.synchronize()
    # host enqueue cost of one eager step (Python + ctypes + launches); under TP also the exchange
    # of one step as counted by the library from its NCCL call arguments (graph replays bypass the host)
    tp0 = W.tpl.stats() if W.tpl else None
    lc0 = launch_count()
    th0 = time.perf_counter()
    W.step(stream)
    host_ms = (time.perf_counter() - th0) * 1e3
    launches_per_step = launch_count() - lc0
    host_many_ms = None
    if not tp_path:  # the same eager step through one slora_lora_apply_many call
        pk = W.packed_calls()
        W.dbatch.apply_many(pk, stream=stream)
        torch.cuda.synchronize()
        th0 = time.perf_counter()
        W.dbatch.prepare(W.batch.token_adapter, stream=stream)
        W.dbatch.apply_many(pk, stream=stream)
        host_many_ms = (time.perf_counter() - th0) * 1e3
        torch.cuda.synchronize()
    tp1 = W.tpl.stats() if W.tpl else None
    torch.cuda.synchronize()
    use_graph = not args.no_graph
    if use_graph:
        W.capture(stream)
        for _ in range(2):
            W.step(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    # ---- timed region: K steps, CUDA events on the launching stream.  No
    # per-launch events inside (they would serialize the programmatic
    # dependent launches); per-launch durations come from a separate pass.
    n0 = launch_count()
    ms, per = timed_steps(W, stream, args.steps, ws)
    launches = launch_count() - n0
    ck = clocks.stop()
    tokens_step = W.Tad * layers
    value = tokens_step / (ms / 1e3)  # TP: the N ranks serve the same tokens together (strong scaling)
    roofline = roofline_of(W, ms, stream)
    roofline["kernel"] = (f"mbgmv_kernel<{cfg.dtype}, kFused> (persistent warp-specialized gather-shrink-expand)"
                          if not tp_path else f"mbgmv_kernel<{cfg.dtype}, kShrink/kExpand> + NCCL (per GPU)")
    roofline["traffic"] = traffic_record(cfg.name) if not tp_path else None
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": warm, "ms_per_step": round(ms, 4), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype,
           "data": "synthetic (seeded; random-init adapters; Zipf adapter popularity)",
           "config": {"workload": cfg.name, "hidden": cfg.hidden, "ranks": list(cfg.rank_list),
                      "n_adapters": cfg.n_adapters, "alpha": cfg.alpha, "tokens": W.T,
                      "adapted_tokens": W.Tad, "unique_adapters": len(W.batch.ranks), "layers": layers,
                      "projections": "q,k,v,o", "parallelism": f"tp{ws}",
                      "l2": "inputs larger than L2 (adapter pages of all layers ~%.2f GB rotate)" %
                            (layers * (W.bytes_qkv + W.bytes_o) / 1e9),
                      "step": "batch_prepare + layers x (qkv, o)" + (" through slora_tp_lora_qkv/_o" if tp_path
                                                                     else " fused applies"),
                      "launch": "CUDA graph replay of the layer launches (PDL edges; TP: with the library's "
                                "NCCL calls); prepare per step" if use_graph else "eager launches"},
           "p10_p50_p90_ms": [round(float(v), 4) for v in np.percentile(per, [10, 50, 90])],
           "gpu_launches": int(launches_per_step * args.steps if use_graph else launches),
           "host_enqueue_ms_eager_step": round(host_ms, 3),
           "host_enqueue_ms_eager_step_apply_many": None if host_many_ms is None else round(host_many_ms, 3),
           "clocks": ck,
           "batch_prepare_host_us": W.prepare_us, "adapter_load": W.load, "roofline": roofline}
    if W.tpl:
        st = {k: tp1[k] - tp0[k] for k in tp1}
        NR = sum(W.batch.ranks[a] for a in W.batch.token_adapter if a >= 0)
        out["tp_exchange_per_step"] = dict(st, P337_allgather_elems=3 * (ws - 1) * NR // ws * layers,
                                           P337_allreduce_elems=2 * (ws - 1) * NR // ws * layers,
                                           source="counts from the arguments passed to ncclAllGather/"
                                                  "ncclAllReduce (slora_tp_get_stats)")
    if use_graph and tp_path:
        try:
            out["lora_comm"] = lora_comm_overhead(W, stream, max(5, args.steps // 2))
        except Exception as e:
            out["lora_comm"] = {"error": f"{type(e).__name__}: {e}"}
        # NEXT-3 device-initiated exchange: one rank here; across GPUs only on request (unmeasured there)
        if ws == 1 or os.environ.get("SLORA_BENCH_TP_P2P") == "1":
            try:
                out["tp_device_initiated"] = tp_p2p_step(W, stream, max(5, args.steps // 2), ms)
            except Exception as e:
                out["tp_device_initiated"] = {"error": f"{type(e).__name__}: {e}"}
    if use_graph and not tp_path and W.dbatch.info()["mbgmm_segments"] == 0:
        rot = rotating_steps(W, stream, args.steps)
        rot["vs_fixed_batch"] = round(rot["ms_per_step"] / ms, 3)
        out["rotating_batch"] = rot
    if not args.no_e2e:
        out["e2e"] = run_e2e(W, stream, max(3, args.steps // 2))
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, W.batch, budget_s=8.0)
    if ws == 1 and not tp_path and not args.no_secondary and use_graph:
        try:
            out["base_lora_overlap"] = base_lora_overlap(W, stream)
        except Exception as e:
            out["base_lora_overlap"] = {"error": f"{type(e).__name__}: {e}"}
        try:
            out["adapter_io"] = run_adapter_io(W, stream)
        except Exception as e:  # reported, never silently dropped
            out["adapter_io"] = {"error": f"{type(e).__name__}: {e}"}
    W.close()
    if ws == 1 and not tp_path and not args.no_secondary and name == "c2":
        sec = {}
        for sname, sl in (("c2-mixed", 32), ("c2-uniform", 32), ("c1", 32), ("c3", 40), ("c4", 8)):
            try:
                sec[sname] = measure(sname, sl, 10, 3, stream)
            except Exception as e:  # reported, never silently dropped
                sec[sname] = {"error": f"{type(e).__name__}: {e}"}
        sec["c4"]["note"] = "70B shapes unsharded on one GPU (the TP8 config's N=1 point); 8 layers (670 MB of " \
                            "adapter pages rotate, >> L2)"
        sec["c3"]["note"] = "13B shapes unsharded on one GPU (the TP4 config's N=1 point), 40 layers"
        try:
            sec["c2-mlp"] = measure_mlp(stream)
        except Exception as e:
            sec["c2-mlp"] = {"error": f"{type(e).__name__}: {e}"}
        out["secondary"] = sec
        try:
            out["ablations"] = run_ablations(stream)
        except Exception as e:
            out["ablations"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_adapter_io(W, stream, n_adapters=16):
    """NEXT-1: adapter loads on the library's loader thread + copy stream
    (slora_adapter_prefetch), alone and overlapped with the decode step.

    A second set of adapters (the ranks of the batch's first n_adapters, new ids, all layers)
    is loaded into a pool of its own on the same GPU: from page-locked host buffers (the
    loader's H2D reads them directly) and from pageable numpy buffers (packed by the loader's
    host threads into pinned staging).  Then the pinned set is prefetched while the step's
    graph is replayed: hidden = 1 - (T_both - T_steps) / T_load, with T_both the wall time
    until the steps and the loads are both done."""
    import torch
    from paper_2311_03285_b200 import Pool
    cfg, L = W.cfg, W.L
    ranks = [W.batch.ranks[a] for a in W.batch.unique][:n_adapters]
    ids = [1_000_000 + i for i in range(len(ranks))]
    need = sum(L * 8 * r for r in ranks)
    pool = Pool(W.H, L, need + 16, dtype=cfg.dtype, device=torch.cuda.current_device(), max_adapters=len(ids) + 8)
    by_rank = {r: wl.adapter_host_buffer(cfg, 100_000 + r, L, rank=r) for r in set(ranks)}  # content is immaterial
    hosts = [by_rank[r].copy() for r in ranks]
    td = torch.int16 if cfg.dtype == "bf16" else None
    pinned = [(torch.from_numpy(h.view(np.int16)) if td else torch.from_numpy(h)).pin_memory() for h in hosts]
    nbytes = sum(h.nbytes for h in hosts)

    def load_all(bufs):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, r, hb in zip(ids, ranks, bufs):
            pool.adapter_prefetch(i, r, hb)
        for i in ids:
            pool.adapter_wait(i)
        t = time.perf_counter() - t0
        for i in ids:
            pool.adapter_evict(i, stream=stream)
        torch.cuda.synchronize()
        return t

    # the serving loop's compute stream at high priority, the library's copy stream at the lowest:
    # the LoRA kernels' CTAs are scheduled ahead of the loader's scatter kernels
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -5)
    stream = torch.cuda.Stream(priority=hi)
    ctx = torch.cuda.stream(stream)
    ctx.__enter__()
    load_all(pinned)  # warm-up (first-touch of staging, thread start)
    t_pinned = min(load_all(pinned) for _ in range(2))
    t_pageable = load_all(hosts)
    # steps alone: enough graph replays to outlast the load
    step_ms = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(3):
        W.step(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / 3
    k = max(8, int(np.ceil(1.5 * t_pinned * 1e3 / step_ms)))

    def steps(n):
        e0.record(stream)
        for _ in range(n):
            W.step(stream)
        e1.record(stream)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps(k)
    torch.cuda.synchronize()
    t_steps = time.perf_counter() - t0
    gpu_steps_alone = e0.elapsed_time(e1)
    # overlapped: prefetch the set, replay the steps meanwhile
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, r, hb in zip(ids, ranks, pinned):
        pool.adapter_prefetch(i, r, hb)
    steps(k)
    for i in ids:
        pool.adapter_wait(i)
    torch.cuda.synchronize()
    t_both = time.perf_counter() - t0
    gpu_steps_both = e0.elapsed_time(e1)
    st = pool.loader_stats()
    for i in ids:
        pool.adapter_evict(i, stream=stream)
    pool.close()
    ctx.__exit__(None, None, None)
    hidden = 1.0 - (t_both - t_steps) / t_pinned
    return {"adapters": len(ids), "bytes": int(nbytes), "layers": L,
            "pinned_GBps": round(nbytes / t_pinned / 1e9, 2), "pinned_ms": round(1e3 * t_pinned, 2),
            "pageable_GBps": round(nbytes / t_pageable / 1e9, 2), "pageable_ms": round(1e3 * t_pageable, 2),
            "overlap": {"steps": k, "steps_alone_ms": round(1e3 * t_steps, 2), "both_ms": round(1e3 * t_both, 2),
                        "hidden_fraction": round(max(0.0, min(1.0, hidden)), 3),
                        "step_ms_alone": round(gpu_steps_alone / k, 4), "step_ms_while_loading":
                            round(gpu_steps_both / k, 4)},
            "loader": {"loads": st["loads"], "direct_loads": st["direct_loads"]},
            "note": "slora_adapter_prefetch on the library's loader thread and copy stream; pinned = page-locked "
                    "host_w read by the H2D directly, pageable = numpy packed into pinned staging; a separate "
                    "pool on the same GPU; steps on a high-priority stream; hidden = 1 - (T_both - T_steps) / T_load"}


def run_ablations(stream):
    """NEXT-2: the S-LoRA-bmm and no-unify-mem kernel-level
    ablations, timed on the C2 decode batch (bench_ablations.py)."""
    import bench_ablations
    return bench_ablations.run(stream)


def run_e2e(W, stream, steps):
    """Same metric through the public API with HOST buffers: every step copies
    the step's activations H2D from pinned memory (x of all layers and the y
    outputs they update; under TP also z and the base partials), prepares the
    batch from the host token map, runs the layers and reads every updated
    output back D2H."""
    import torch
    if not W.tp_path:
        return run_e2e_pipelined(W, stream, steps)
    ins = [W.x, W.y] + ([W.z, W.base] if W.tp_path else [])
    outs = [W.y] + ([W.base] if W.tp_path else [])
    hin = [t.cpu().pin_memory() for t in ins]
    hout = [torch.empty_like(t, device="cpu").pin_memory() for t in outs]
    bi = sum(t.numel() * t.element_size() for t in hin) + W.T * 8
    bo = sum(t.numel() * t.element_size() for t in hout)

    def one():
        for d, h in zip(ins, hin):
            d.copy_(h, non_blocking=True)
        W.step(stream)
        for h, d in zip(hout, outs):
            h.copy_(d, non_blocking=True)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        one()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    return {"value": round(W.Tad * W.L / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(bi),
            "d2h_bytes_per_step": int(bo), "ms_per_step": round(ms, 4)}


def run_e2e_pipelined(W, stream, steps, chunk=4):
    """e2e on one GPU with the host<->device copies pipelined by groups of `chunk` layers: a
    copy-in stream moves group g's x and y from pinned host memory while the compute stream runs
    group g-1 (one slora_lora_apply_many call per group: q/k/v, o of each layer) and a copy-out
    stream returns group g-2's y.  A group's buffers are refilled for the next step only after
    their copy-out (per-group events).  Same bytes as the serial form; the step ends when its
    last output is on the host."""
    import torch
    from paper_2311_03285_b200 import Batch
    L, H = W.L, W.H
    hx = W.x.cpu().pin_memory()
    hy = W.y.cpu().pin_memory()
    hyo = torch.empty_like(W.y, device="cpu").pin_memory()
    bi = hx.numel() * hx.element_size() + hy.numel() * hy.element_size() + W.T * 8
    bo = hyo.numel() * hyo.element_size()
    groups = [(g, min(g + chunk, L)) for g in range(0, L, chunk)]
    calls = []
    for a, b in groups:
        cl = []
        for l in range(a, b):
            ys = [W.y[l, p] for p in range(4)]
            cl += [(l, "qkv", W.x[l], H, ys, [H] * 4), (l, "o", W.x[l], H, ys, [H] * 4)]
        calls.append(Batch.make_calls(cl))
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    n = len(groups)
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_c = [torch.cuda.Event() for _ in range(n)]
    ev_out = [torch.cuda.Event() for _ in range(n)]
    started = [False]

    def one():
        W.dbatch.prepare(W.batch.token_adapter, stream=stream)
        for i, (a, b) in enumerate(groups):
            if started[0]:
                s_in.wait_event(ev_out[i])  # the group's previous outputs are on the host
            with torch.cuda.stream(s_in):
                W.x[a:b].copy_(hx[a:b], non_blocking=True)
                W.y[a:b].copy_(hy[a:b], non_blocking=True)
            ev_in[i].record(s_in)
        for i, (a, b) in enumerate(groups):
            stream.wait_event(ev_in[i])
            W.dbatch.apply_many(calls[i], stream=stream)
            ev_c[i].record(stream)
            s_out.wait_event(ev_c[i])
            with torch.cuda.stream(s_out):
                hyo[a:b].copy_(W.y[a:b], non_blocking=True)
            ev_out[i].record(s_out)
        started[0] = True
        stream.wait_event(ev_out[n - 1])  # the step is done when its last output is on the host

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        one()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    return {"value": round(W.Tad * W.L / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(bi),
            "d2h_bytes_per_step": int(bo), "ms_per_step": round(ms, 4),
            "note": f"groups of {chunk} layers: pinned H2D of x, y on a copy stream || slora_lora_apply_many "
                    "(q/k/v, o of each layer) || D2H of y on another copy stream; eager launches (no graph)"}


# --------------------------------------------------------------- oracle arm
def oracle_sample(cfg, batch):
    """One layer (q,k,v,o deltas) of the workload's batch, oracle inputs."""
    import oracle
    ids = batch.unique
    slot = np.array([ids.index(a) if a >= 0 else -1 for a in batch.token_adapter], np.int64)
    T, H = batch.T, cfg.hidden
    x = oracle.to_f64(wl.activations(cfg, T, H, 100), cfg.dtype)
    proj = []
    for p in range(4):
        As, Bs = [], []
        for a in ids:
            A, B = wl.adapter_weights(cfg, a, 0, p, batch.ranks[a])
            As.append(oracle.to_f64(A, cfg.dtype))
            Bs.append(oracle.to_f64(B, cfg.dtype))
        y = oracle.to_f64(wl.activations(cfg, T, H, 200 + p), cfg.dtype)
        proj.append((As, Bs, y))
    return x, slot, proj


def oracle_layer(x, slot, proj, nthreads):
    import oracle
    for As, Bs, y in proj:
        oracle.lora_apply(x, y, As, Bs, slot, nthreads=nthreads)


def _time_loop(fn, budget_s):
    fn()
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        fn()
        n += 1
    return (time.perf_counter() - t0) / max(n, 1), n


def cpu_baseline(cfg, batch, budget_s=8.0):
    """The oracle as it stands on the host cores: the LoRA delta
    of one layer on all cores and on one thread, and the full layer
    x.W + delta (base GEMM in the oracle's naive fp64 loops) on a bounded
    token sample."""
    import oracle
    cores = os.cpu_count() or 1
    x, slot, proj = oracle_sample(cfg, batch)
    Tad = int((slot >= 0).sum())
    dt, n = _time_loop(lambda: oracle_layer(x, slot, proj, cores), budget_s)
    dt1, n1 = _time_loop(lambda: oracle_layer(x, slot, proj, 1), budget_s / 2)
    # full layer on the first 8 tokens: base x.W (h x d, W ~ N(0, 1/h)) + delta, 4 projections
    Ts = min(8, batch.T)
    rng = np.random.default_rng(7)
    Ws = [rng.standard_normal((cfg.hidden, cfg.hidden)) / np.sqrt(cfg.hidden) for _ in range(4)]
    xs, ss = x[:Ts], slot[:Ts]

    def full():
        for (As, Bs, y), Wp in zip(proj, Ws):
            base = oracle.base_forward(xs, Wp, nthreads=cores)
            oracle.lora_apply(xs, base, As, Bs, ss, nthreads=cores)

    dtf, nf = _time_loop(full, budget_s / 2)
    Tads = int((ss >= 0).sum())
    return {"value": round(Tad / dt, 2), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} repetitions of one layer's q,k,v,o deltas of the {cfg.name} batch "
                      f"({Tad} tokens, {len(batch.ranks)} adapters), fp64 C oracle, {cores} threads",
            "one_thread_value": round(Tad / dt1, 2),
            "full_layer_value": round(Tads / dtf, 2),
            "full_layer_sample": f"{nf} repetitions of x.W + delta for q,k,v,o on the batch's first {Ts} tokens "
                                 f"(W: {cfg.hidden}x{cfg.hidden} fp64, naive loops), {cores} threads"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    name = args.workload or "c2"
    cfg = wl.CONFIGS[name]
    batch = wl.make_batch(cfg)
    cores = os.cpu_count() or 1
    x, slot, proj = oracle_sample(cfg, batch)
    Tad = int((slot >= 0).sum())
    for _ in range(max(3, args.warmup)):
        oracle_layer(x, slot, proj, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_layer(x, slot, proj, cores)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    value = Tad / (ms / 1e3)
    sample = (f"each step = one layer's q,k,v,o deltas of the {cfg.name} batch ({Tad} tokens, "
              f"{len(batch.ranks)} adapters), fp64 C oracle on {cores} host threads")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (seeded)",
           "config": {"workload": cfg.name, "hidden": cfg.hidden, "ranks": list(cfg.rank_list),
                      "tokens": batch.T, "layers": 1, "parallelism": "host threads"},
           "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
