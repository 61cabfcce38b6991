"""GPU parity of the stand-alone splitters (tmg_split_low_i64 /
tmg_split_high_i64, k_split_i64.cu) with the reference's split_low_i64 /
split_high_i64 (products.hpp:68-79, split.cpp:66-158).

The cases are the reference's own (test_products.cpp:52-176) at the chunk
widths an int64 holds, checked against a Python-integer restatement of
chunk_big (split.cpp:41-61) and, at product sizes, against the C oracle's
split (oracle.c, the float pipeline's chunk_store).  Bit-exact.
"""
from dataclasses import replace

import numpy as np
import pytest

import paper_1703_00640_b200 as tm
from oracle import port

pytestmark = pytest.mark.gpu

FULL, LOW, HIGH = tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH
EXACT = tm.Backend.EXACT


def lg_ceil(n):
    return (n - 1).bit_length()


def chunk_big(u, b, count, balanced):
    """split.cpp:41-61 on Python ints."""
    out, carry = [], 0
    half, full = 1 << (b - 1), 1 << b
    for i in range(count):
        x = ((u >> (i * b)) & (full - 1)) + carry
        if balanced and i + 1 < count and x > half:
            out.append(x - full)
            carry = 1
        else:
            out.append(x)
            carry = 0
    return out


def reassemble(chunks, b):
    acc = 0
    for c in reversed([int(c) for c in chunks]):
        acc = (acc << b) + c
    return acc


def rand_bits(rng, n):
    return int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1)


def test_low_split_documented_example(ctx):
    # test_products.cpp:52-64 (the reference tests' manual_params defaults to an
    # unsigned split, test_products.cpp:19-20)
    p = tm.manual_params(6, 2, 3, FULL, EXACT, signed_split=False)
    assert tm.split_low_i64(13, p, ctx).tolist() == [1, 3, 0]
    # balanced: 3 > 2^{b-1} becomes -1 and carries into the top chunk
    assert tm.split_low_i64(13, replace(p, signed_split=True), ctx).tolist() == [1, -1, 1]


def test_high_split_aligns_to_the_top(ctx):
    # test_products.cpp:66-78
    p = tm.manual_params(10, 4, 3, HIGH, EXACT, signed_split=False)
    assert tm.split_high_i64(1023, p, ctx).tolist() == [0, 12, 15, 15]


def test_splits_reassemble_the_operand(ctx):
    # test_products.cpp:80-120 (the cells an int64 chunk holds)
    rng = np.random.default_rng(0x5EED)
    for b, N in ((4, 3), (6, 17), (13, 40), (31, 9), (62, 41)):
        for balanced in (False, True):
            n = N * b - 1
            p = tm.manual_params(n, b, N, FULL, EXACT, balanced)
            for _ in range(20):
                u = rand_bits(rng, n)
                w = tm.split_low_i64(u, p, ctx)
                assert len(w) == N and reassemble(w, b) == u
                assert w.tolist() == chunk_big(u, b, N, balanced)
            assert reassemble(tm.split_low_i64(0, p, ctx), b) == 0
    for balanced in (False, True):
        b, N = 6, 33
        n = (N + 1) * b - lg_ceil(N) - 2
        p = tm.manual_params(n, b, N, HIGH, EXACT, balanced)
        sigma = (N + 1) * b - n
        for _ in range(20):
            u = rand_bits(rng, n)
            w = tm.split_high_i64(u, p, ctx)
            assert len(w) == N + 1 and reassemble(w, b) == u << sigma
            assert w.tolist() == chunk_big(u << sigma, b, N + 1, balanced)
    p = tm.manual_params(10000, 16, 625, FULL, EXACT, True)
    u = rand_bits(rng, 10000)
    assert reassemble(tm.split_low_i64(u, p, ctx), 16) == u


def test_balanced_chunks_stay_in_their_window(ctx):
    # test_products.cpp:122-141
    rng = np.random.default_rng(0xBA1A)
    b, N = 8, 25
    p = tm.manual_params(N * b, b, N, FULL, EXACT, True)
    half, full = 1 << (b - 1), 1 << b
    for _ in range(50):
        w = tm.split_low_i64(rand_bits(rng, N * b), p, ctx)
        assert np.all(w[:-1] > -half) and np.all(w[:-1] <= half)
        assert 0 <= w[-1] <= full


def test_machine_word_splits_match_the_big_splits(ctx):
    # test_products.cpp:143-163
    rng = np.random.default_rng(0x1DEA)
    for b in (4, 14, 21, 62):
        N = 19
        n = N * b - 2
        for balanced in (False, True):
            p = tm.manual_params(n, b, N, FULL, EXACT, balanced)
            for _ in range(10):
                u = rand_bits(rng, n)
                assert tm.split_low_i64(u, p, ctx).tolist() == chunk_big(u, b, N, balanced)
    wide = tm.manual_params(300, 100, 3, FULL, EXACT)
    with pytest.raises(tm.InputOutOfRange, match="too large for int64"):
        tm.split_low_i64(5, wide, ctx)


def test_splits_reject_out_of_range(ctx):
    # test_products.cpp:165-177; the operand range check runs on the device
    p = tm.manual_params(12, 4, 3, LOW, EXACT, signed_split=False)
    for bad_u in (1 << 12, 1 << 13):
        with pytest.raises(tm.InputOutOfRange, match="outside"):
            ctx.split_i64(np.array([bad_u], dtype=np.uint64), p)
    with pytest.raises(tm.InputOutOfRange):
        tm.split_low_i64(-1, p, ctx)
    # a good split after a refused one
    assert tm.split_low_i64(0xABC, p, ctx).tolist() == chunk_big(0xABC, 4, 3, False)
    bad = replace(p, n=13)
    with pytest.raises(tm.InputOutOfRange, match="N b >= n"):
        tm.split_low_i64(1, bad, ctx)
    high = replace(tm.manual_params(10, 4, 3, HIGH, EXACT), n=15)
    with pytest.raises(tm.InputOutOfRange, match=r"\(N\+1\) b"):
        tm.split_high_i64(1, high, ctx)


@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 777, 1 << 26])
@pytest.mark.parametrize("mode", [FULL, LOW, HIGH])
def test_product_sized_splits_match_the_oracle(ctx, n, mode):
    """At the products' own parameters: the oracle's chunk_store restatement
    (doubles, exact for these b), both balancings."""
    rng = np.random.default_rng(n + int(mode))
    nl = (n + 63) // 64
    u = rng.integers(0, 2**64, nl, dtype=np.uint64)
    if n % 64:
        u[-1] &= np.uint64((1 << (n % 64)) - 1)
    p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
    high = mode == HIGH
    count = p.N + 1 if high else p.N
    lead = (p.N + 1) * p.b - n if high else 0
    for balanced in (True, False):
        w = ctx.split_i64(u, replace(p, signed_split=balanced), high=high)
        ref = port.split(u, n, p.b, count, balanced, lead)
        assert np.array_equal(w, ref.astype(np.int64))


@pytest.mark.parametrize("b", [12, 13, 19])
def test_split_carry_chains_through_half_windows(ctx, b):
    """Windows equal to 2^{b-1} pass their carry-in on: stretches of them
    across warp and block boundaries, with a generating, a killing or no
    window below, and one that reaches chunk 0."""
    rng = np.random.default_rng(b)
    N = 5000
    n = N * b
    half = 1 << (b - 1)
    digs = [int(x) for x in rng.integers(0, 1 << b, N)]
    for start, length, below in ((0, 40, None), (100, 700, half + 1), (1000, 31, half - 1),
                                 (2040, 300, (1 << b) - 1), (4000, 999, 0)):
        for j in range(start, start + length):
            digs[j] = half
        if below is not None:
            digs[start - 1] = below
    u = sum(d << (i * b) for i, d in enumerate(digs))
    p = tm.manual_params(n, b, N, FULL, EXACT, True)
    assert tm.split_low_i64(u, p, ctx).tolist() == chunk_big(u, b, N, True)
