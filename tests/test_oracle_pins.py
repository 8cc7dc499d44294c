"""Pins for the CPU oracle (oracle/): what the paper and the mathematics fix,
independent of the oracle's own code.

Each test says which plausible oracle mistake it would catch.
P:L = /root/reference/PAPER.md line L (documentation only; not read here).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import tp_emulation as tpe

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def rand_problem(rng, T, h, d, ranks, p_none=0.0):
    x = rng.standard_normal((T, h))
    y = rng.standard_normal((T, d))
    As = [rng.standard_normal((h, r)) / np.sqrt(h) for r in ranks]
    Bs = [rng.standard_normal((r, d)) / np.sqrt(r) for r in ranks]
    slot = rng.integers(0, len(ranks), size=T)
    if p_none:
        slot = np.where(rng.random(T) < p_none, -1, slot)
    return x, y, As, Bs, slot


# --------------------------------------------------------------------- O1
def test_merged_weight_equivalence():
    """Eq. lora = Eq. lora_factored: x(W + sAB) = xW + s(xA)B.
    The right side is computed by numpy matmul on the merged weight, a
    different association order than the oracle's loops.  Catches a dropped
    term, a wrong sign, a transposed A or B, scale applied twice/never."""
    rng = np.random.default_rng(1)
    for trial in range(100):
        h = int(rng.integers(1, 65))
        d = int(rng.integers(1, 65))
        n_ad = int(rng.integers(1, 5))
        ranks = [int(rng.integers(1, 17)) for _ in range(n_ad)]
        T = int(rng.integers(1, 9))
        x, _, As, Bs, slot = rand_problem(rng, T, h, d, ranks)
        W = rng.standard_normal((h, d))
        scale = rng.uniform(0.25, 2.0, size=n_ad)
        base = oracle.base_forward(x, W)
        out = oracle.lora_apply(x, base, As, Bs, slot, scale)
        ref = np.stack([x[i] @ (W + scale[slot[i]] * (As[slot[i]] @ Bs[slot[i]])) for i in range(T)])
        err = np.abs(out - ref).max() / max(np.abs(ref).max(), 1e-300)
        assert err <= 1e-12, (trial, err)
        # base forward itself against numpy's matmul (h = xW)
        assert np.abs(base - x @ W).max() <= 1e-12 * max(np.abs(x @ W).max(), 1.0)


# --------------------------------------------------------------------- O2
def test_base_only_reductions():
    """No adapter, A = 0 or B = 0 => output is exactly y_in.
    Catches a delta applied to tokens without an adapter or garbage init."""
    rng = np.random.default_rng(2)
    x, y, As, Bs, _ = rand_problem(rng, 12, 32, 24, [4, 8])
    out = oracle.lora_apply(x, y, As, Bs, np.full(12, -1))
    assert np.array_equal(out, y)
    zA = [np.zeros_like(A) for A in As]
    zB = [np.zeros_like(B) for B in Bs]
    slot = np.arange(12) % 2
    assert np.array_equal(oracle.lora_apply(x, y, zA, Bs, slot), y)
    assert np.array_equal(oracle.lora_apply(x, y, As, zB, slot), y)
    # mixed: only adapted rows change
    slot = np.array([0, -1] * 6)
    out = oracle.lora_apply(x, y, As, Bs, slot)
    assert np.array_equal(out[1::2], y[1::2])
    assert not np.array_equal(out[0::2], y[0::2])


# --------------------------------------------------------------------- O3
def test_integer_brute_force_exact():
    """Integer inputs at C0 shapes: fp64 is exact, so the oracle must equal
    Python-int brute force EXACTLY (S:44 naive triple loop).  Catches any
    index, sign, transposition or bound error, bit for bit."""
    rng = np.random.default_rng(3)
    h = d = 256
    ranks = [4, 8, 4, 8]
    T = 16
    x = rng.integers(-3, 4, size=(T, h))
    y = rng.integers(-3, 4, size=(T, d))
    As = [rng.integers(-3, 4, size=(h, r)) for r in ranks]
    Bs = [rng.integers(-3, 4, size=(r, d)) for r in ranks]
    slot = np.array([0] * 5 + [1] + [2] * 7 + [-1] * 3)
    scale = np.array([1.0, 2.0, 0.5, 1.0])
    out = oracle.lora_apply(x.astype(float), y.astype(float), [A.astype(float) for A in As],
                            [B.astype(float) for B in Bs], slot, scale)
    for i in range(T):
        a = int(slot[i])
        for c in range(d):
            want = Fraction(int(y[i, c]))
            if a >= 0:
                acc = 0
                for j in range(ranks[a]):
                    vj = sum(int(x[i, k]) * int(As[a][k, j]) for k in range(h))
                    acc += vj * int(Bs[a][j, c])
                want += Fraction(scale[a]).limit_denominator(4) * acc
            assert out[i, c] == float(want), (i, c)


# --------------------------------------------------------------------- O4
def test_rank1_closed_form():
    """A = e_p (h x 1), B = e_q^T (1 x d) => delta_i = x_i[p] at column q,
    zero elsewhere.  h != d and p != q catch swapped operands."""
    h, d, p, q = 48, 40, 7, 31
    rng = np.random.default_rng(4)
    x = rng.standard_normal((5, h))
    y = rng.standard_normal((5, d))
    A = np.zeros((h, 1)); A[p, 0] = 1.0
    B = np.zeros((1, d)); B[0, q] = 1.0
    out = oracle.lora_apply(x, y, [A], [B], np.zeros(5, int))
    want = y.copy()
    want[:, q] += x[:, p]
    assert np.array_equal(out, want)


# --------------------------------------------------------------------- O5
def test_permutation_invariance():
    """Permuting tokens permutes outputs bit-exactly.  Catches state
    leaking between tokens (e.g. an accumulator not reset)."""
    rng = np.random.default_rng(5)
    x, y, As, Bs, slot = rand_problem(rng, 40, 64, 48, [8, 16, 64, 32], p_none=0.2)
    out = oracle.lora_apply(x, y, As, Bs, slot)
    perm = rng.permutation(40)
    out_p = oracle.lora_apply(x[perm], y[perm], As, Bs, slot[perm])
    assert np.array_equal(out_p, out[perm])
    # thread count does not change a single bit
    out_t = oracle.lora_apply(x, y, As, Bs, slot, nthreads=7)
    assert np.array_equal(out_t, out)


# --------------------------------------------------------------- O6 + O7
def test_padding_invariance_and_flop_identity():
    """Zero padding to r_max adds exact zeros and the executed-
    operation counters satisfy the S:222 identity
        unpadded = sum_i (2 S_i h r_i + 2 S_i r_i d),  padded uses r_max.
    Catches loops that run to the wrong bound or skip the expand half."""
    rng = np.random.default_rng(6)
    h, d = 64, 40
    ranks = [8, 16, 64, 32]
    for trial in range(20):
        T = int(rng.integers(1, 30))
        x, y, As, Bs, slot = rand_problem(rng, T, h, d, ranks, p_none=0.1)
        out, fl = oracle.lora_apply(x, y, As, Bs, slot, return_flops=True)
        outp, flp = oracle.padded_apply(x, y, As, Bs, slot)
        assert np.array_equal(out, outp)
        used = [int(s) for s in slot if s >= 0]
        assert fl == sum(2 * h * ranks[a] + 2 * ranks[a] * d for a in used)
        rmax = max([ranks[a] for a in used], default=1)
        assert flp == len(used) * (2 * h * rmax + 2 * rmax * d)
        all_equal = len({ranks[a] for a in used}) <= 1
        assert (fl == flp) == all_equal


# --------------------------------------------------------------------- O8
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_tp_emulation_matches_single_device(N):
    """S-LoRA TP emulated on N devices equals the single-device
    oracle within 1e-9, and the traffic the emulated ring collectives
    actually generated equals the P:337 formula exactly."""
    rng = np.random.default_rng(100 + N)
    h = d = 64
    ranks = [8, 16, 64, 32, 8]
    B = 12
    x = rng.standard_normal((B, h))
    z = rng.standard_normal((B, d))
    W = {p: rng.standard_normal((h, d)) / np.sqrt(h) for p in "qkvo"}
    ads = [{p: (rng.standard_normal((h, r)) / np.sqrt(h), rng.standard_normal((r, d)) / np.sqrt(r))
            for p in "qkvo"} for r in ranks]
    slot = rng.integers(0, len(ranks), size=B)
    slot[3] = -1
    out, cnt = tpe.emulate_layer(N, x, z, W["q"], W["k"], W["v"], W["o"], ads, slot)
    for p in "qkv":
        ref = oracle.lora_apply(x, oracle.base_forward(x, W[p]), [a[p][0] for a in ads],
                                [a[p][1] for a in ads], slot)
        assert np.abs(out[p] - ref).max() <= 1e-9 * np.abs(ref).max()
    ref = oracle.lora_apply(z, oracle.base_forward(z, W["o"]), [a["o"][0] for a in ads],
                            [a["o"][1] for a in ads], slot)
    assert np.abs(out["o"] - ref).max() <= 1e-9 * np.abs(ref).max()
    sum_r = sum(ranks[s] for s in slot if s >= 0)
    assert cnt["sum_r"] == sum_r
    for k in range(N):
        assert cnt["lora_allgather_sent"][k] == 3 * (N - 1) * sum_r // N
        assert cnt["lora_allreduce_sent"][k] == 2 * (N - 1) * sum_r // N
        assert cnt["base_allreduce_sent"][k] == 2 * (N - 1) * B * h // N
    if N == 1:
        assert cnt["lora_allgather_sent"] == [0] and cnt["base_allreduce_sent"] == [0]


def test_tp_indivisible():
    """N must divide h and r (reading R3)."""
    rng = np.random.default_rng(9)
    h = 64
    ads = [{p: (rng.standard_normal((h, 6)), rng.standard_normal((6, h))) for p in "qkvo"}]
    W = np.zeros((h, h))
    with pytest.raises(tpe.IndivisibleDimension):
        tpe.emulate_layer(4, np.zeros((2, h)), np.zeros((2, h)), W, W, W, W, ads, [0, 0])
    with pytest.raises(tpe.IndivisibleDimension):
        tpe.emulate_layer(4, np.zeros((2, 66)), np.zeros((2, 66)), *[np.zeros((66, 66))] * 4, [], [-1, -1])


def test_comm_golden_example_and_ratio():
    """S:352 example evaluated by the emulation's own counters at full
    h = 4096 (uniform r = 8, N = 2, B = 16): base 65536, LoRA 320 elements;
    and the ratio 5r/(2h) = 5/1024 ~ 0.488% as an exact rational."""
    g = GOLD["comm_cost_example"]
    N, B, h, r = g["N"], g["B"], g["h"], g["r"]
    rng = np.random.default_rng(10)
    W = np.zeros((h, h))
    ads = [{p: (rng.standard_normal((h, r)) * 1e-3, rng.standard_normal((r, h)) * 1e-3) for p in "qkvo"}]
    _, cnt = tpe.emulate_layer(N, np.ones((B, h)), np.ones((B, h)), W, W, W, W, ads, [0] * B)
    lora = cnt["lora_allgather_sent"][0] + cnt["lora_allreduce_sent"][0]
    base = cnt["base_allreduce_sent"][0]
    assert base == g["base_elements"]
    assert lora == g["lora_elements"]
    gr = GOLD["comm_ratio_example"]
    assert Fraction(lora, base) == Fraction(gr["ratio_num"], gr["ratio_den"])
    assert abs(100 * lora / base - gr["ratio_percent_approx"]) < 1e-3


# --------------------------------------------------------------------- O9
@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_memory_optimality(N):
    """No replicated weight: per-device shard elements sum to the
    global count, each device holding exactly 1/N."""
    per, total = tpe.shard_elements(N, 4096, 4096, 64)
    assert sum(per) == total
    assert all(p * N == total for p in per)


def _ieee_value(bits, ebits, mbits):
    """IEEE-754 binary value of a bit pattern, from the definition
    (sign, biased exponent, fraction; subnormals; inf/nan), as a Fraction or
    float('inf')/-inf.  Independent of numpy's views."""
    sign = -1 if bits >> (ebits + mbits) & 1 else 1
    e = bits >> mbits & ((1 << ebits) - 1)
    m = bits & ((1 << mbits) - 1)
    bias = (1 << (ebits - 1)) - 1
    if e == (1 << ebits) - 1:
        return sign * float("inf") if m == 0 else float("nan")
    if e == 0:
        return sign * Fraction(m, 1 << mbits) * Fraction(2) ** (1 - bias)
    return sign * (1 + Fraction(m, 1 << mbits)) * Fraction(2) ** (e - bias)


@pytest.mark.parametrize("bits,expect", [(0x3F80, 1.0), (0xC040, -3.0), (0x0001, 2.0 ** -133),
                                         (0x7F7F, 3.3895313892515355e38), (0x4049, 3.140625),
                                         (0x8000, -0.0), (0x0080, 2.0 ** -126)])
def test_to_f64_bf16_bit_patterns(bits, expect):
    """oracle.to_f64 decodes bf16 storage (uint16 bit patterns) exactly: pinned
    to hand-derived values and to the IEEE definition with 8 exponent and 7
    fraction bits.  Catches a wrong shift (<< 15 / << 17), a byte swap, or
    decoding as fp16."""
    got = oracle.to_f64(np.array([bits], np.uint16), "bf16")[0]
    assert got == expect and np.signbit(got) == np.signbit(expect)
    assert Fraction(got) == _ieee_value(bits, 8, 7)


def test_to_f64_bf16_sampled_patterns_against_definition():
    """Every 97th of the 65536 bf16 patterns (all exponents, signs, subnormals,
    inf/nan) decodes to the IEEE definition, checked with exact rationals."""
    pats = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    with np.errstate(invalid="ignore"):  # nan patterns
        got = oracle.to_f64(pats, "bf16")
    for b in range(0, 1 << 16, 97):  # a spread sample checked with exact rationals
        v = _ieee_value(b, 8, 7)
        if isinstance(v, float):
            assert np.isinf(got[b]) if not np.isnan(v) else np.isnan(got[b])
        else:
            assert Fraction(got[b]) == v, hex(b)


@pytest.mark.parametrize("bits", [0x3C00, 0x0001, 0x7BFF, 0xC200, 0x0400])
def test_to_f64_f16_bit_patterns(bits):
    got = oracle.to_f64(np.array([bits], np.uint16).view(np.float16), "f16")[0]
    assert Fraction(got) == _ieee_value(bits, 5, 10)


def test_bf16_round_to_nearest_even_ties():
    """synth.round_to (the storage rounding both sides read) rounds fp32 to
    bf16 to nearest, ties to even: 1 + 2^-8 is halfway between 1 (even
    fraction 0) and 1 + 2^-7 (odd) -> 1; 1 + 3*2^-8 is halfway between
    1 + 2^-7 (odd) and 1 + 2^-6 (even) -> 1 + 2^-6; just above a tie rounds up."""
    from synth import workload as wl
    xs = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, 1 + 2 ** -8 + 2 ** -20, -(1 + 2 ** -8)], np.float32)
    b = wl.round_to(xs, "bf16")
    assert [int(v) for v in b] == [0x3F80, 0x3F82, 0x3F81, 0xBF80]
    assert list(oracle.to_f64(b, "bf16")) == [1.0, 1 + 2 ** -6, 1 + 2 ** -7, -1.0]
