"""CPU fp64 oracle for S-LoRA heterogeneous batched LoRA (arXiv 2311.03285).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs may import, call, link or
execute anything under oracle/.  The product path (paper_2311_03285_b200/)
never imports it, and this package imports nothing from the product path.

Contents
  slora_oracle.{h,c}  plain C, fp64, naive loops: Eq. lora_factored
                      per token, the padded baseline and the
                      base forward xW.  Built to liboracle.so.
  pool_model.py       reference model of Unified Paging.
  tp_emulation.py     S-LoRA tensor parallelism emulated on N logical devices
                      (Fig. lora_tp) with counted payloads.
  (this file)         ctypes loader + exact decoding of stored fp32/fp16/bf16
                      values to fp64.

Parity pins (tests/test_oracle_pins.py): merged-weight equivalence (Eq. lora
= Eq. lora_factored), base-only reduction, integer brute force,
rank-1 closed form, permutation and padding invariance, FLOP identity, TP
emulation vs single device and the P:337 communication formula.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "slora_oracle.c")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (fp contraction off: each a*b+c is two
    roundings, in the order the source states)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-pthread", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.POINTER(ctypes.c_int64)
        _lib.oracle_lora_apply.argtypes = [ctypes.c_int64] * 3 + [d, d, ctypes.c_int64, i64, d, i64, i64,
                                                                  d, d, i64, d, ctypes.c_int, i64]
        _lib.oracle_lora_apply.restype = ctypes.c_int
        _lib.oracle_padded_apply.argtypes = [ctypes.c_int64] * 3 + [d, d, ctypes.c_int64, i64, d, i64, i64,
                                                                    d, d, i64, d, i64]
        _lib.oracle_padded_apply.restype = ctypes.c_int
        _lib.oracle_base_forward.argtypes = [ctypes.c_int64] * 3 + [d, d, d, ctypes.c_int]
        _lib.oracle_base_forward.restype = ctypes.c_int
    return _lib


# ----------------------------------------------------------------- decoding
def to_f64(raw: np.ndarray, dtype: str) -> np.ndarray:
    """Exact conversion of stored values to fp64.
    fp32 / fp16: numpy's widening conversion is exact.
    bf16: stored as uint16 bit patterns; bits << 16 is the fp32 with the same
    value, then widened exactly."""
    if dtype == "f32":
        return np.asarray(raw, dtype=np.float32).astype(np.float64)
    if dtype == "f16":
        return np.asarray(raw, dtype=np.float16).astype(np.float64)
    if dtype == "bf16":
        bits = np.asarray(raw, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
        return bits.view(np.float32).astype(np.float64)
    raise ValueError(dtype)


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _pack(adapters_A, adapters_B):
    ranks = np.array([a.shape[1] for a in adapters_A], dtype=np.int64)
    A_off = np.zeros(len(adapters_A), dtype=np.int64)
    B_off = np.zeros(len(adapters_A), dtype=np.int64)
    oa = ob = 0
    for i, (A, B) in enumerate(zip(adapters_A, adapters_B)):
        A_off[i], B_off[i] = oa, ob
        oa += A.size
        ob += B.size
    A_all = np.concatenate([np.ascontiguousarray(A, np.float64).ravel() for A in adapters_A]) \
        if adapters_A else np.zeros(1)
    B_all = np.concatenate([np.ascontiguousarray(B, np.float64).ravel() for B in adapters_B]) \
        if adapters_B else np.zeros(1)
    return ranks, A_off, B_off, A_all, B_all


def lora_apply(x, y_in, adapters_A, adapters_B, slot, scale=None, nthreads=1, return_flops=False):
    """out_i = y_in_i + scale_a * (x_i A_a) B_a, slot -1 -> y_in_i.

    x: T x h fp64; y_in: T x d fp64; adapters_A[a]: h x r_a; adapters_B[a]:
    r_a x d; slot: length-T int (adapter index or -1)."""
    x = np.ascontiguousarray(x, np.float64)
    y_in = np.ascontiguousarray(y_in, np.float64)
    T, h = x.shape
    d = y_in.shape[1]
    ranks, A_off, B_off, A_all, B_all = _pack(adapters_A, adapters_B)
    sc = np.ones(len(ranks)) if scale is None else np.ascontiguousarray(scale, np.float64)
    sl = np.ascontiguousarray(slot, np.int64)
    out = np.empty((T, d), np.float64)
    fl = np.zeros(1, np.int64)
    rc = lib().oracle_lora_apply(T, h, d, _dp(x), _dp(y_in), len(ranks), _ip(ranks), _dp(sc),
                                 _ip(A_off), _ip(B_off), _dp(A_all), _dp(B_all), _ip(sl), _dp(out),
                                 int(nthreads), _ip(fl))
    if rc != 0:
        raise ValueError("oracle_lora_apply: bad arguments")
    return (out, int(fl[0])) if return_flops else out


def padded_apply(x, y_in, adapters_A, adapters_B, slot, scale=None):
    """Padded baseline; returns (out, flops)."""
    x = np.ascontiguousarray(x, np.float64)
    y_in = np.ascontiguousarray(y_in, np.float64)
    T, h = x.shape
    d = y_in.shape[1]
    ranks, A_off, B_off, A_all, B_all = _pack(adapters_A, adapters_B)
    sc = np.ones(len(ranks)) if scale is None else np.ascontiguousarray(scale, np.float64)
    sl = np.ascontiguousarray(slot, np.int64)
    out = np.empty((T, d), np.float64)
    fl = np.zeros(1, np.int64)
    rc = lib().oracle_padded_apply(T, h, d, _dp(x), _dp(y_in), len(ranks), _ip(ranks), _dp(sc),
                                   _ip(A_off), _ip(B_off), _dp(A_all), _dp(B_all), _ip(sl), _dp(out),
                                   _ip(fl))
    if rc != 0:
        raise ValueError("oracle_padded_apply: bad arguments")
    return out, int(fl[0])


def base_forward(x, W, nthreads=1):
    """h = xW."""
    x = np.ascontiguousarray(x, np.float64)
    W = np.ascontiguousarray(W, np.float64)
    T, h = x.shape
    d = W.shape[1]
    out = np.empty((T, d), np.float64)
    if lib().oracle_base_forward(T, h, d, _dp(x), _dp(W), _dp(out), int(nthreads)) != 0:
        raise ValueError("oracle_base_forward: bad arguments")
    return out
