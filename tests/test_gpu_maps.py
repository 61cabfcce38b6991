"""GPU parity of the stand-alone ring-change maps (tmg_alpha_star_f64,
tmg_beta_star_f64, tmg_gamma_dagger_f64, tmg_delta_dagger_f64; k_maps.cu)
with the reference's maps_f64.hpp functions as restated in oracle/oracle.c
(maps_f64.cpp:48-384).

The GPU evaluates the series coefficients on the fly from their closed forms;
the reference reads tables rounded from long double.  The two differ in the
last ulps of a coefficient, so values are compared within
TOL = 8 eps * max(|in|, |ref|) -- the leading row has coefficient 1 exactly
and row r is smaller by about 2^{-r b}, which keeps the difference to a few
eps of the largest input.  What the products need from the maps -- the same
integers after rounding -- is checked exactly by assembling the reference's
low and high pipelines (products_f64.cpp:123-171) from the stand-alone entry
points and comparing with the exact product.
"""
import ctypes

import numpy as np
import pytest

import paper_1703_00640_b200 as tm
from oracle import port

pytestmark = pytest.mark.gpu
EPS = 2.0**-52
LOW, HIGH = tm.Mode.LOW, tm.Mode.HIGH


def tol(*arrays):
    return 8 * EPS * max(float(np.max(np.abs(a))) for a in arrays)


def digits(rng, b, count, top=False):
    d = rng.integers(-(1 << (b - 1)) + 1, (1 << (b - 1)) + 1, count).astype(np.float64)
    if top:
        d[-1] = float(rng.integers(0, (1 << b) + 1))
    return d


def shapes():
    out = [(64, 12, 4), (100, 8, 5), (1000, 14, 4), (4099, 13, 3)]
    for lg in (16, 20, 24):
        for mode in (LOW, HIGH):
            p = tm.select_params(1 << lg, mode, policy=tm.Policy.ACCURATE)
            out.append((p.N, p.b, p.lam))
    return sorted(set(out))


@pytest.mark.parametrize("N,b,lam", shapes())
def test_alpha_and_beta_star(ctx, N, b, lam):
    rng = np.random.default_rng(N + b)
    x = digits(rng, b, N)
    ref = x.copy()
    port.lib().orc_alpha_star_inplace(port._pd(port.coeff_table("alpha", lam, N, b)), lam, N, port._pd(ref))
    out = ctx.alpha_star_f64(N, b, lam, x)
    assert np.max(np.abs(out - ref)) <= tol(x, ref)
    # beta* on convolution-sized values
    w = np.rint(rng.standard_normal(N) * 2.0 ** (2 * b - 2) * np.sqrt(N))
    refb = np.empty(N)
    port.lib().orc_beta_star(port._pd(port.coeff_table("beta", lam, N, b)), lam, N, b, port._pd(w), port._pd(refb))
    outb = ctx.beta_star_f64(N, b, lam, w)
    assert np.max(np.abs(outb - refb)) <= tol(w, refb)


@pytest.mark.parametrize("N,b,lam", shapes())
def test_gamma_and_delta_dagger(ctx, N, b, lam):
    rng = np.random.default_rng(N + b + 1)
    x = digits(rng, b, N + 1, top=True)
    ref = x.copy()
    au = ctypes.c_double(0.0)
    port.lib().orc_gamma_dagger_inplace(port._pd(port.coeff_table("gamma", lam, N, b)), lam, N, b, port._pd(ref),
                                        ctypes.byref(au))
    out, aux = ctx.gamma_dagger_f64(N, b, lam, x)
    assert np.max(np.abs(out - ref[:N])) <= tol(x, ref[:N])
    assert abs(aux - au.value) <= 8 * EPS * abs(au.value)
    w = np.rint(rng.standard_normal(N) * 2.0 ** (2 * b - 2) * np.sqrt(N))
    a2 = au.value * au.value
    refd = np.empty(N + 1)
    port.lib().orc_delta_dagger(port._pd(port.coeff_table("delta", lam, N, b)), lam, N, b, port._pd(w), a2,
                                port._pd(refd))
    outd = ctx.delta_dagger_f64(N, b, lam, w, a2)
    assert np.max(np.abs(outd - refd)) <= tol(w, refd, np.array([a2]))


@pytest.mark.parametrize("lg", [16, 20, 22])
def test_low_pipeline_from_the_entry_points(ctx, lg):
    """products_f64.cpp:123-143 assembled on the GPU: split, alpha*, cyclic
    convolution, beta*; the oracle's checked rounding and recombination then
    give the exact low product."""
    n = 1 << lg
    rng = np.random.default_rng(lg)
    u = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
    v = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
    p = tm.select_params(n, LOW, policy=tm.Policy.ACCURATE)
    a = ctx.alpha_star_f64(p.N, p.b, p.lam, ctx.split_i64(u, p).astype(np.float64))
    c = ctx.alpha_star_f64(p.N, p.b, p.lam, ctx.split_i64(v, p).astype(np.float64))
    w = ctx.cyclic_convolve_f64(a, c)
    low = ctx.beta_star_f64(p.N, p.b, p.lam, w)
    t, max_err, _ = port._accumulate(low, p.b, p.b, (p.N * p.b + p.b + 128) // 64 + 4)
    assert max_err < 0.25
    assert t & ((1 << p.b) - 1) == 0
    P = port.limbs_to_int(port.oracle_full(u, v))
    assert (t >> p.b) & ((1 << n) - 1) == P & ((1 << n) - 1)


@pytest.mark.parametrize("lg", [16, 20, 22])
def test_high_pipeline_from_the_entry_points(ctx, lg):
    """products_f64.cpp:145-171 assembled on the GPU: top-aligned split,
    gamma-dagger, cyclic convolution, delta-dagger; rounding, recombination
    and round(t / 2^s) by the oracle; the result is an admissible high
    product."""
    n = 1 << lg
    rng = np.random.default_rng(lg + 100)
    u = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
    v = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
    p = tm.select_params(n, HIGH, policy=tm.Policy.ACCURATE)
    sigma = (p.N + 1) * p.b - n
    a, au = ctx.gamma_dagger_f64(p.N, p.b, p.lam, ctx.split_i64(u, p, high=True).astype(np.float64))
    c, av = ctx.gamma_dagger_f64(p.N, p.b, p.lam, ctx.split_i64(v, p, high=True).astype(np.float64))
    w = ctx.cyclic_convolve_f64(a, c)
    h = ctx.delta_dagger_f64(p.N, p.b, p.lam, w, au * av)
    t, max_err, _ = port._accumulate(h, p.b, p.b, ((p.N + 1) * p.b + p.b + 128) // 64 + 4)
    assert max_err < 0.25
    wv = port._round_even_shift(t, 2 * p.b + sigma)
    assert port.is_valid_high(u, v, n, wv)


def test_map_argument_errors(ctx):
    with pytest.raises(tm.InputOutOfRange):
        ctx.alpha_star_f64(0, 12, 4, np.zeros(0))
    with pytest.raises(tm.Unsupported):
        ctx.alpha_star_f64(64, 12, 9, np.zeros(64))  # lambda above the GPU limit
    with pytest.raises(tm.Unsupported):
        ctx.gamma_dagger_f64(6, 8, 1, np.zeros(7))   # N b < 64
    with pytest.raises(tm.PlanMismatch):
        ctx.beta_star_f64(64, 12, 4, np.zeros(63))
