"""GPU parity of the stand-alone FP64 cyclic convolution
(tmg_cyclic_convolve_f64) with the reference's cyclic_convolve_f64
(convolution.hpp:64-67, convolution.cpp:175-203).

Integer-valued operands small enough for FP64 to hold every coefficient are
checked exactly: the rounded result must equal the oracle's (rfft * rfft ->
irfft on pocketfft, itself cross-checked against a direct integer sum at
small lengths), with a residual below the products' 0.25 tripwire.  Real-valued
operands are compared within TOL * sum|f| * max|g| (a forward-error bound of
a double-precision FFT convolution; FFTW and this transform differ in
operation order, so bit equality is not defined for them).
"""
import numpy as np
import pytest

import paper_1703_00640_b200 as tm
from oracle import port

pytestmark = pytest.mark.gpu
TOL = 64 * 2.0**-52  # relative to sum|f| max|g|


def direct(f, g):
    n = len(f)
    idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
    return (np.asarray(f, dtype=object)[None, :] * np.asarray(g, dtype=object)[idx]).sum(axis=1)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 12, 60, 243, 1000, 4096])
def test_direct_lengths_exact_on_integers(ctx, n):
    rng = np.random.default_rng(n)
    f = rng.integers(-2000, 2000, n)
    g = rng.integers(-2000, 2000, n)
    out = ctx.cyclic_convolve_f64(f, g)
    if n <= 1000:
        assert [int(x) for x in out] == [int(x) for x in direct(f, g)]
    else:
        assert np.array_equal(out, np.rint(port.cyclic_convolve(f.astype(float), g.astype(float))))


# multi-pass plans: the lengths select_params picks for the products (two- and
# three-pass, compiled and generic column shapes), and other smooth lengths
@pytest.mark.parametrize("n", [5120, 6144, 8192, 20480, 81920, 100352, 5 * 7 * 3 * 4 * 1024,
                               327680, 1310720, 5898240, 7077888, 22937600])
def test_transform_lengths_exact_on_integers(ctx, n):
    rng = np.random.default_rng(n)
    f = rng.integers(-2048, 2049, n).astype(np.float64)
    g = rng.integers(-2048, 2049, n).astype(np.float64)
    out = ctx.cyclic_convolve_f64(f, g)
    ref = port.cyclic_convolve(f, g)
    r = np.rint(out)
    assert np.array_equal(r, np.rint(ref))
    assert np.max(np.abs(out - r)) < 0.25
    assert ctx.last_kernel_count() >= 5  # absmax, pack, first column pass, row pass, last column pass


@pytest.mark.parametrize("n", [4096, 12288, 1 << 20, 5898240])
def test_real_operands_within_fft_tolerance(ctx, n):
    rng = np.random.default_rng(n + 1)
    f = rng.standard_normal(n)
    g = rng.standard_normal(n) * 1e3
    out = ctx.cyclic_convolve_f64(f, g)
    ref = port.cyclic_convolve(f, g)
    bound = TOL * np.sum(np.abs(f)) * np.max(np.abs(g))
    assert np.max(np.abs(out - ref)) <= bound


def test_identity_and_shift(ctx):
    """f (*) delta = f and f (*) delta_5 = f shifted, to FFT accuracy relative
    to ||f|| ||g||, whatever the operands' relative magnitudes (the packed
    transform balances them by a power of two first)."""
    n = 1 << 16
    rng = np.random.default_rng(5)
    f = rng.integers(-1000, 1000, n).astype(np.float64)
    for amp in (1.0, 2.0**-40, 3.0e9):
        e = np.zeros(n)
        e[0] = amp
        bound = 64 * 2.0**-52 * np.linalg.norm(f) * amp
        assert np.max(np.abs(ctx.cyclic_convolve_f64(f, e) - amp * f)) <= bound
        assert np.max(np.abs(ctx.cyclic_convolve_f64(e, f) - amp * f)) <= bound
        e[0], e[5] = 0.0, amp
        assert np.max(np.abs(ctx.cyclic_convolve_f64(f, e) - amp * np.roll(f, 5))) <= bound
    assert not ctx.cyclic_convolve_f64(f, np.zeros(n)).any()


def test_length_errors_follow_make_plan(ctx):
    # test_convolution.cpp:144 (176 = 16 * 11 is not smooth)
    with pytest.raises(tm.UnsupportedLength, match="smooth length, got 176"):
        ctx.cyclic_convolve_f64(np.zeros(176), np.zeros(176))
    with pytest.raises(tm.UnsupportedLength, match="positive"):
        ctx.cyclic_convolve_f64(np.zeros(0), np.zeros(0))
    with pytest.raises(tm.UnsupportedLength, match="multiples of 4"):
        ctx.cyclic_convolve_f64(np.zeros(3**11), np.zeros(3**11))
    with pytest.raises(tm.PlanMismatch):
        ctx.cyclic_convolve_f64(np.zeros(8), np.zeros(16))
    # odd smooth lengths up to 32768 are summed directly
    n = 3**9
    rng = np.random.default_rng(9)
    f = rng.integers(-100, 100, n).astype(np.float64)
    g = rng.integers(-100, 100, n).astype(np.float64)
    assert np.array_equal(ctx.cyclic_convolve_f64(f, g), np.rint(port.cyclic_convolve(f, g)))


def test_products_after_a_convolution_are_unaffected(ctx):
    """The convolution shares the context's workspace with the products."""
    n = 1 << 20
    rng = np.random.default_rng(3)
    nl = n // 64
    u = rng.integers(0, 2**64, nl, dtype=np.uint64)
    v = rng.integers(0, 2**64, nl, dtype=np.uint64)
    P = port.limbs_to_int(port.oracle_full(u, v))
    ctx.cyclic_convolve_f64(np.ones(81920), np.ones(81920))
    p = tm.select_params(n, tm.Mode.LOW, policy=tm.Policy.ACCURATE)
    assert tm.from_limbs(ctx.product_limbs(tm.Mode.LOW, u, v, p)) == P & ((1 << n) - 1)
    ctx.cyclic_convolve_f64(np.ones(100352), np.ones(100352))
    p = tm.select_params(n, tm.Mode.FULL, policy=tm.Policy.ACCURATE)
    assert tm.from_limbs(ctx.product_limbs(tm.Mode.FULL, u, v, p)) == P
