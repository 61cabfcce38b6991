"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Full and low products must be bit-exact with the exact product (GMP, the
reference's own bignum dependency, cross-checked against Python ints and the
oracle's Karatsuba in test_oracle.py).  High products must satisfy
|uv - 2^n w| < 2^n with 0 <= w <= 2^n (the reference's admissible set), and
are compared with the oracle port's value.  Inputs where the float pipeline
cannot certify the rounding must raise ConvolutionPrecisionFailure, like the
reference (products_f64.cpp:16-27).

Covers BASELINE.json configs 1-5 plus the reference tests' edge cases.
"""
import json
import os

import numpy as np
import pytest

import paper_1703_00640_b200 as tm
from oracle import port

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TRIP = 0.25  # reference tripwire (products_f64.cpp:22)


def sp(n, mode):
    """The accurate policy's parameters (Numerics) -- an explicit
    opt-in; select_params' default is the reference's params.cpp."""
    return tm.select_params(n, mode, policy=tm.Policy.ACCURATE)


def _check(mode, u, v, n, r):
    P = port.limbs_to_int(port.oracle_full(u, v))
    if mode == tm.Mode.FULL:
        assert r == P
    elif mode == tm.Mode.LOW:
        assert r == P & ((1 << n) - 1)
    else:
        assert 0 <= r <= (1 << n)
        assert abs(P - (r << n)) < (1 << n)


def _rand(rng, n):
    nl = (n + 63) // 64
    a = rng.integers(0, 2**64, nl, dtype=np.uint64)
    if n % 64:
        a[-1] &= np.uint64((1 << (n % 64)) - 1)
    return a


@pytest.mark.parametrize("n", [4096, 5001, 8192, 20011, 65536, 100003, 105078, 262144, 1000000, 1 << 22,
                               4748529])
def test_random_products_match_exact(ctx, n):
    rng = np.random.default_rng(n)
    for _ in range(3):
        u, v = _rand(rng, n), _rand(rng, n)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = sp(n, mode)
            r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
            _check(mode, u, v, n, r)
            assert ctx.last_stats.max_round_err <= TRIP


def test_golden_vectors(ctx):
    """Committed known answers (tools/make_golden.py): exact, or the same
    precision failure the reference raises for boundary-digit operands."""
    gold = json.load(open(os.path.join(GOLD, "products.json")))
    exact = failed = 0
    for e in gold["vectors"]:
        n = e["n"]
        nl = (n + 63) // 64
        u = port.int_to_limbs(int(e["u"], 16), nl)
        v = port.int_to_limbs(int(e["v"], 16), nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = sp(n, mode)
            try:
                r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
            except tm.ConvolutionPrecisionFailure:
                assert not e["tag"].startswith("uniform"), e["tag"]
                failed += 1
                continue
            if mode == tm.Mode.FULL:
                assert format(r, "x") == e["full"], (e["tag"], n)
            elif mode == tm.Mode.LOW:
                assert format(r, "x") == e["low"], (e["tag"], n)
            else:
                assert format(r, "x") in e["high_set"], (e["tag"], n)
            exact += 1
    assert exact > 300


def test_reference_cli_examples(ctx):
    gold = json.load(open(os.path.join(GOLD, "products.json")))
    mode = {"mul": tm.Mode.FULL, "mullo": tm.Mode.LOW, "mulhi": tm.Mode.HIGH}
    for c in gold["cli"]:
        r = tm.multiply(mode[c["cmd"]], int(c["u"], 16), int(c["v"], 16), n=c["n"], ctx=ctx)
        assert format(r, "x") in c["expect"], c


def test_gpu_agrees_with_port_on_tripwire(ctx):
    """Where the oracle port certifies with a margin, the GPU must too; where
    the port trips far above the wire, the GPU must trip as well."""
    gold = json.load(open(os.path.join(GOLD, "products.json")))
    for e in gold["vectors"]:
        n = e["n"]
        if n < 4096:
            continue
        nl = (n + 63) // 64
        u = port.int_to_limbs(int(e["u"], 16), nl)
        v = port.int_to_limbs(int(e["v"], 16), nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW):
            p = sp(n, mode)
            try:
                pe = port.product(mode.name.lower(), u, v, n, p.b, p.N, p.lam).max_err
            except port.ConvolutionPrecisionFailure:
                pe = None
            try:
                ctx.product_limbs(mode, u, v, p)
                ge = ctx.last_stats.max_round_err
            except tm.ConvolutionPrecisionFailure:
                ge = None
            if pe is not None and pe < 0.18:
                assert ge is not None, (e["tag"], n, mode, pe)


def test_commutativity_and_consistency(ctx):
    rng = np.random.default_rng(11)
    n = 200000
    u, v = _rand(rng, n), _rand(rng, n)
    pl, pf, ph = (sp(n, m) for m in (tm.Mode.LOW, tm.Mode.FULL, tm.Mode.HIGH))
    lo = tm.from_limbs(ctx.product_limbs(tm.Mode.LOW, u, v, pl))
    assert lo == tm.from_limbs(ctx.product_limbs(tm.Mode.LOW, v, u, pl))
    fu = tm.from_limbs(ctx.product_limbs(tm.Mode.FULL, u, v, pf))
    assert fu == tm.from_limbs(ctx.product_limbs(tm.Mode.FULL, v, u, pf))
    assert lo == fu & ((1 << n) - 1)
    hi = tm.from_limbs(ctx.product_limbs(tm.Mode.HIGH, u, v, ph))
    assert hi in ((fu >> n), (fu >> n) + 1)
    # deterministic
    assert hi == tm.from_limbs(ctx.product_limbs(tm.Mode.HIGH, u, v, ph))


@pytest.mark.parametrize("n", [5001, 300007])
def test_structured_operands(ctx, n):
    nl = (n + 63) // 64
    vals = [0, 1, 2, 3, 1 << (n // 2), 1 << (n - 1), (1 << (n - 1)) + 1, (1 << (n - 1)) - 1,
            (1 << n) - 1, (1 << n) - 2]
    for a in vals:
        for b_ in (vals[0], vals[1], vals[-2], a):
            u, v = port.int_to_limbs(a, nl), port.int_to_limbs(b_, nl)
            for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
                r = tm.from_limbs(ctx.product_limbs(mode, u, v, sp(n, mode)))
                _check(mode, u, v, n, r)


@pytest.mark.parametrize("n", [(1 << 20) + 3, 3 << 20])
def test_carry_chains_across_blocks(esc_ctx, n):
    """Products whose limbs hold long runs of zeros and all-ones: a carry
    (or borrow) into a carry block walks through many limbs and across
    blocks (k_carry_patch for full and low, k_carry_apply for high).  The
    structured spectra may refuse at the policy's b: escalation recomputes."""
    nl = (n + 63) // 64
    M = (1 << n) - 1
    rng = np.random.default_rng(11)
    r0 = port.limbs_to_int(_rand(rng, n))
    cases = [(M, M), (M, (1 << (n // 2)) + 1), ((1 << (n - 1)) + (1 << (n // 3)), M - M // 3),
             (M, 1 << (n - 1)), (r0, M), (M ^ (1 << (n // 2)), M), ((1 << n) - (1 << 1000), M - 5)]
    for a, b_ in cases:
        u, v = port.int_to_limbs(a, nl), port.int_to_limbs(b_, nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            r = tm.from_limbs(esc_ctx.product_limbs(mode, u, v, sp(n, mode)))
            _check(mode, u, v, n, r)


def test_unsigned_wide_chunks_trip(ctx):
    """test_products.cpp:408-416: b = 30 unsigned chunks overflow the exact
    integer range and must be refused."""
    p = tm.manual_params(3840, 30, 128, tm.Mode.LOW, tm.Backend.FFT, signed_split=False, lam=4)
    top = (1 << 3840) - 1
    with pytest.raises(tm.ConvolutionPrecisionFailure):
        tm.low_product(top, top, p, ctx)


def test_unsigned_split_products(ctx):
    n = 20000
    rng = np.random.default_rng(5)
    u, v = _rand(rng, n), _rand(rng, n)
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        ref = sp(n, mode)
        b = ref.b - 4
        cover = -(-n // b)
        N = next(x for x in range(cover + (4 if mode == tm.Mode.HIGH else 0), 4 * cover)
                 if all(q in (2, 3, 5, 7) for q in _factors(x)) and x % 4 == 0)
        p = tm.manual_params(n, b, N, mode, tm.Backend.FFT, signed_split=False)
        r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
        _check(mode, u, v, n, r)


def _factors(x):
    out = []
    for q in (2, 3, 5, 7):
        while x % q == 0:
            out.append(q)
            x //= q
    if x > 1:
        out.append(x)
    return out


def test_input_out_of_range(ctx):
    p = sp(8192, tm.Mode.LOW)
    with pytest.raises(tm.InputOutOfRange):
        tm.low_product(1 << 8192, 3, p, ctx)
    with pytest.raises(tm.InputOutOfRange):
        tm.full_product(3, 5, p, ctx)  # params built for a different mode


def test_fallback_below_cutoff(ctx):
    rng = np.random.default_rng(6)
    for n in (1, 7, 64, 65, 1000, 4095):
        u, v = _rand(rng, n), _rand(rng, n)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = sp(n, mode)
            assert p.mode == tm.Mode.ORACLE_FALLBACK
            r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
            P = port.limbs_to_int(u) * port.limbs_to_int(v)
            if mode == tm.Mode.FULL:
                assert r == P
            elif mode == tm.Mode.LOW:
                assert r == P & ((1 << n) - 1)
            else:
                assert r == P >> n  # oracle_high_set(...).front()


def test_device_path_matches_host_path(ctx):
    import torch
    n = 1 << 20
    rng = np.random.default_rng(9)
    u, v = _rand(rng, n), _rand(rng, n)
    p = sp(n, tm.Mode.LOW)
    host = ctx.product_limbs(tm.Mode.LOW, u, v, p)
    du = torch.from_numpy(u.view(np.int64)).cuda()
    dv = torch.from_numpy(v.view(np.int64)).cuda()
    out = torch.zeros(len(host), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
    ctx.check()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), host)


_CHAIN_SNIPPET = """
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1703_00640_b200 as tm
from oracle import port
sp = lambda n, m: tm.select_params(n, m, policy=tm.Policy.ACCURATE)
ctx = tm.Context(0)
bad = 0
for n in (1 << 20, 1 << 22):
    nl = n // 64
    rng = np.random.default_rng(n)
    p = sp(n, tm.Mode.LOW)
    for rep in range(4):
        a = rng.integers(0, 2**64, nl, dtype=np.uint64)
        b = rng.integers(0, 2**64, nl, dtype=np.uint64)
        bufs = [torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b)]
        bufs += [torch.zeros(nl, dtype=torch.int64, device="cuda") for _ in range(6)]
        torch.cuda.synchronize()
        # x_{k+2} = x_k x_{k+1} mod 2^n, each product reading the previous outputs
        for k in range(6):
            ctx.product_device(p, bufs[k].data_ptr(), bufs[k + 1].data_ptr(), bufs[k + 2].data_ptr(), 1)
        ctx.check()
        M = (1 << n) - 1
        xs = [port.limbs_to_int(a), port.limbs_to_int(b)]
        for k in range(6):
            xs.append(xs[k] * xs[k + 1] & M)
        got = [port.limbs_to_int(t.cpu().numpy().view(np.uint64)) for t in bufs]
        bad += sum(g != x for g, x in zip(got, xs))
# a multi-pass product, then fused small products reading its output
n1, n2 = 1 << 20, 1 << 16
p1, p2 = sp(n1, tm.Mode.LOW), sp(n2, tm.Mode.LOW)
rng = np.random.default_rng(5)
for rep in range(4):
    a = rng.integers(0, 2**64, n1 // 64, dtype=np.uint64)
    b = rng.integers(0, 2**64, n1 // 64, dtype=np.uint64)
    da, db = (torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b))
    o1 = torch.zeros(n1 // 64, dtype=torch.int64, device="cuda")
    o2 = torch.zeros(n2 // 64, dtype=torch.int64, device="cuda")
    o3 = torch.zeros(n2 // 64, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ctx.product_device(p1, da.data_ptr(), db.data_ptr(), o1.data_ptr(), 1)
    ctx.product_device(p2, o1.data_ptr(), db.data_ptr(), o2.data_ptr(), 1)
    ctx.product_device(p2, o2.data_ptr(), o1.data_ptr(), o3.data_ptr(), 1)
    ctx.check()
    x1 = port.limbs_to_int(a) * port.limbs_to_int(b) % (1 << n1)
    m2 = (1 << n2) - 1
    x2 = (x1 & m2) * (port.limbs_to_int(b) & m2) & m2
    x3 = x2 * (x1 & m2) & m2
    got = [port.limbs_to_int(t.cpu().numpy().view(np.uint64)) for t in (o1, o2, o3)]
    bad += sum(g != x for g, x in zip(got, (x1, x2, x3)))
print("bad", bad)
print("ok" if bad == 0 else "mismatch")
"""


def test_chained_device_products():
    """Device-pointer products chained output -> input on one stream with no
    synchronisation in between: each product's operands are the previous
    ones' outputs, which kernels still in flight may be writing, so k_zstat
    must not read them before its predecessor completes."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CHAIN_SNIPPET], cwd=root, env=dict(os.environ),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-500:] + r.stderr[-2000:]


# --------------------------------------------------------------------------
# BASELINE.json configurations


def test_config1_low_2p20_seed1(ctx):
    n = 1 << 20
    u, v = port.config_operands(1, n // 64)
    p = sp(n, tm.Mode.LOW)
    r = ctx.product_limbs(tm.Mode.LOW, u, v, p)
    assert np.array_equal(r, port.oracle_low(u, v, n))
    assert ctx.last_stats.max_round_err < TRIP


def test_config2_high_2p24_seed2(ctx):
    n = 1 << 24
    u, v = port.config_operands(2, n // 64, force_top_bit=True)
    p = sp(n, tm.Mode.HIGH)
    w = tm.from_limbs(ctx.product_limbs(tm.Mode.HIGH, u, v, p))
    assert port.is_valid_high(u, v, n, w)
    assert ctx.last_stats.max_round_err < TRIP
    # the oracle port at the same parameters lands on the same value unless
    # t / 2^s sits within rounding noise of a half-integer
    pw = port.high_product(u, v, n, p.b, p.N, p.lam).value
    assert pw in port.oracle_high_set(u, v, n)
    assert w == pw


def test_config3_full_low_high_2p26_seed3(ctx):
    n = 1 << 26
    u, v = port.config_operands(3, n // 64)
    P = port.limbs_to_int(port.oracle_full(u, v))
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        p = sp(n, mode)
        r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
        if mode == tm.Mode.FULL:
            assert r == P
        elif mode == tm.Mode.LOW:
            assert r == P & ((1 << n) - 1)
        else:
            assert abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)
        assert ctx.last_stats.max_round_err < TRIP


def test_config3_reference_params_trip_like_the_reference(ctx):
    """At the reference's own b = 13 for n = 2^26 the FP64 error passes its
    0.25 tripwire; the GPU either refuses like the reference or,
    if it certifies, is exact."""
    n = 1 << 26
    u, v = port.config_operands(3, n // 64)
    p = tm.select_params(n, tm.Mode.LOW, policy=tm.Policy.REFERENCE)
    assert p.b == 13
    try:
        r = ctx.product_limbs(tm.Mode.LOW, u, v, p)
    except tm.ConvolutionPrecisionFailure:
        return
    assert np.array_equal(r, port.oracle_low(u, v, n))


def test_config4_batched_low_2p16_seed4(ctx):
    n, count = 1 << 16, 4096
    nl = n // 64
    w = port.mt19937_64(4, 2 * count * nl).reshape(count, 2, nl)
    u = np.ascontiguousarray(w[:, 0, :])
    v = np.ascontiguousarray(w[:, 1, :])
    p = sp(n, tm.Mode.LOW)
    out, flags = ctx.product_batched(p, u, v, return_flags=True)
    assert not flags.any()
    for i in range(count):
        assert np.array_equal(out[i], port.oracle_low(u[i], v[i], n)), i
    assert ctx.last_stats.max_round_err < TRIP


@pytest.fixture(scope="module")
def esc_ctx():
    c = tm.Context(0, escalation=2)
    yield c
    c.close()


def _stress_operand(pattern, nl):
    if pattern == "ones":
        return np.full(nl, np.uint64(0xFFFFFFFFFFFFFFFF))
    u = np.zeros(nl, dtype=np.uint64)
    u[0::2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return u


@pytest.mark.parametrize("pattern", ["ones", "alternating"])
@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.HIGH])
def test_config5_stress_2p28(ctx, pattern, mode):
    """BASELINE config 5: u = v = 2^n - 1 and alternating all-ones / zero
    limbs at n = 2^28, on the default path (no escalation) at the
    reference's own parameters (the accurate policy picks the same ones
    here).  The alternating pattern concentrates the spectrum on a few
    lines; the result must certify at the first attempt, below the wire
    (low <= 1/4, high < 1/4), and be exact."""
    n = 1 << 28
    u = _stress_operand(pattern, n // 64)
    v = u.copy()
    p = tm.select_params(n, mode)
    assert (p.b, p.N, p.lam) == (12, 22937600, 5)
    assert sp(n, mode) == p
    r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
    st = ctx.last_stats
    print(f"stress {pattern} {mode.name}: b={p.b} N={p.N} residual {st.max_round_err:.4f}")
    assert st.attempts == 1 and not st.escalated
    if mode == tm.Mode.LOW:
        assert st.max_round_err <= TRIP
    else:
        assert st.max_round_err < TRIP
    _check(mode, u, v, n, r)


def test_escalation_recovers_refused_alternating_product(esc_ctx, ctx):
    """2^24 alternating limbs at b = 13 refuse on the GPU and in the
    reference-order port alike; escalation (an opt-in of this library)
    recomputes at b - 1 and returns the exact low product."""
    n = 1 << 24
    u = _stress_operand("alternating", n // 64)
    p = tm.select_params(n, tm.Mode.LOW)
    with pytest.raises(tm.ConvolutionPrecisionFailure):
        ctx.product_limbs(tm.Mode.LOW, u, u, p)
    r = esc_ctx.product_limbs(tm.Mode.LOW, u, u, p)
    assert np.array_equal(r, port.oracle_low(u, u, n))
    assert esc_ctx.last_stats.escalated and esc_ctx.last_stats.max_round_err < TRIP


# --------------------------------------------------------------------------
# Certify / refuse parity with the reference at its own parameters
# (Policy.REFERENCE = params.cpp, the default) on the default context: where
# the oracle port -- the reference's pipeline in its operation order,
# convolution.cpp:186-192 -- certifies, the GPU must certify too, be exact,
# and stay within one 1/16 of the port's residual; where the port refuses,
# the GPU may refuse or certify, and a certified result must be exact.
SLACK = 0.0625


def _ref_parity(ctx, mode, u, v, n, p=None):
    p = p or tm.select_params(n, mode)
    assert p == tm.select_params(n, mode, policy=tm.Policy.REFERENCE)
    try:
        pe = port.product(mode.name.lower(), u, v, n, p.b, p.N, p.lam).max_err
    except port.ConvolutionPrecisionFailure:
        pe = None
    try:
        r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
        ge = ctx.last_stats.max_round_err
    except tm.ConvolutionPrecisionFailure:
        r, ge = None, None
    if pe is not None:
        assert ge is not None, (mode.name, n, "port certifies at", pe, "GPU refuses")
        assert ge <= pe + SLACK, (mode.name, n, ge, pe)
    if r is not None:
        _check(mode, u, v, n, r)
        assert ge <= TRIP
    return pe, ge


def test_reference_fft_products_8192_seed14(ctx):
    """test_products.cpp:371-391: n = 8192, mt19937_64(0x14), ten random pairs
    through low / high / full, then the all-ones operand (low, full)."""
    n = 8192
    for u, v in port.random_bits_pairs(0x14, n, 10):
        for mode in (tm.Mode.LOW, tm.Mode.HIGH, tm.Mode.FULL):
            _ref_parity(ctx, mode, u, v, n)
    top = _stress_operand("ones", n // 64)
    for mode in (tm.Mode.LOW, tm.Mode.FULL):
        pe, ge = _ref_parity(ctx, mode, top, top, n)
        assert pe is not None and ge is not None


def test_reference_fft_products_5001_seed15(ctx):
    """test_products.cpp:393-406: n = 5001 (covering slack), mt19937_64(0x15),
    six random pairs through low and high."""
    n = 5001
    for u, v in port.random_bits_pairs(0x15, n, 6):
        for mode in (tm.Mode.LOW, tm.Mode.HIGH):
            _ref_parity(ctx, mode, u, v, n)


def test_reference_policy_config1(ctx):
    n = 1 << 20
    u, v = port.config_operands(1, n // 64)
    _ref_parity(ctx, tm.Mode.LOW, u, v, n)


def test_reference_policy_config2(ctx):
    n = 1 << 24
    u, v = port.config_operands(2, n // 64, force_top_bit=True)
    _ref_parity(ctx, tm.Mode.HIGH, u, v, n)


@pytest.mark.parametrize("mode", [tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH])
def test_reference_policy_config3(ctx, mode):
    n = 1 << 26
    u, v = port.config_operands(3, n // 64)
    _ref_parity(ctx, mode, u, v, n)


def test_reference_policy_config4(ctx):
    """4096 x 2^16 low products at the reference's parameters in one batch:
    per-product flags agree with the port's certify / refuse on a sample,
    every certified product exact."""
    n, count = 1 << 16, 4096
    nl = n // 64
    w = port.mt19937_64(4, 2 * count * nl).reshape(count, 2, nl)
    u = np.ascontiguousarray(w[:, 0, :])
    v = np.ascontiguousarray(w[:, 1, :])
    p = tm.select_params(n, tm.Mode.LOW)
    out, flags = ctx.product_batched(p, u, v, return_flags=True)
    for i in range(count):
        if not flags[i]:
            assert np.array_equal(out[i], port.oracle_low(u[i], v[i], n)), i
    for i in range(0, count, 64):
        try:
            port.product("low", u[i], v[i], n, p.b, p.N, p.lam)
            assert not flags[i], i
        except port.ConvolutionPrecisionFailure:
            pass


@pytest.mark.parametrize("pattern", ["ones", "alternating"])
@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.HIGH])
def test_reference_policy_config5(ctx, pattern, mode):
    n = 1 << 28
    u = _stress_operand(pattern, n // 64)
    pe, ge = _ref_parity(ctx, mode, u, u.copy(), n)
    assert ge is not None  # the default path certifies config 5


# --------------------------------------------------------------------------
# plan shapes: every radix placement of the multi-pass row/column transforms


def _plan_shape_lengths(limit):
    """Smooth lengths whose row length C (largest even divisor <= 4096) and
    column length A differ in radix structure: radix 4/8 before odd radices,
    odd C/2 schedules, forward/inverse stage tables that do and do not share."""
    seen, out = set(), []
    for N in sorted(2**a * 3**b * 5**c * 7**d for a in range(2, 21) for b in range(4)
                    for c in range(3) for d in range(3)):
        if not (8193 <= N <= (1 << 20)):
            continue
        C = next(c for c in range(4096, 15, -1) if c % 2 == 0 and N % c == 0)
        key = (C, min(N // C, 64))
        if key not in seen:
            seen.add(key)
            out.append(N)
    rng = np.random.default_rng(11)
    return [int(x) for x in rng.choice(out, size=min(limit, len(out)), replace=False)]


@pytest.mark.parametrize("N", _plan_shape_lengths(48))
def test_plan_shapes_exact(ctx, N):
    rng = np.random.default_rng(N)
    for mode, b, Nn in ((tm.Mode.LOW, 12, N), (tm.Mode.FULL, 16, N // 2)):
        n = Nn * b - 5
        p = tm.manual_params(n, b, Nn, mode)
        nl = (n + 63) // 64
        u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        v = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        r = ctx.product_limbs(mode, u, v, p)
        if mode == tm.Mode.LOW:
            assert np.array_equal(r, port.oracle_low(u, v, n)), (N, mode)
        else:
            assert np.array_equal(r, port.oracle_full(u, v)[:len(r)]), (N, mode)
        assert ctx.last_stats.max_round_err < TRIP


@pytest.mark.parametrize("b", [7, 8, 9, 10])
@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.HIGH])
def test_multipass_series_lengths(ctx, b, mode):
    """Multi-pass products at small chunk widths: lambda = 6..8 rows of the
    series maps (the carry kernel is instantiated per lambda)."""
    rng = np.random.default_rng(100 * b + int(mode))
    n = 1 << 17
    N = 1
    while N * b < n + 64:
        N *= 2
    p = tm.manual_params(n, b, N, mode)
    assert p.lam == max(4, (52 + b - 1) // b)
    nl = n // 64
    u = rng.integers(0, 2**64, nl, dtype=np.uint64)
    v = rng.integers(0, 2**64, nl, dtype=np.uint64)
    r = ctx.product_limbs(mode, u, v, p)
    assert ctx.last_stats.transform_length > 8192 and ctx.last_stats.passes >= 2
    _check(mode, u, v, n, tm.from_limbs(r))
    assert ctx.last_stats.max_round_err < TRIP


def test_wide_chunks_refuse_on_the_64_bit_window_path(ctx):
    """b > 32 takes the split kernel's 64-bit window path; at a multi-pass
    length such chunks overflow the exact double range and must refuse."""
    n, b, N = 40 * 6000, 40, 6144
    p = tm.manual_params(n, b, N, tm.Mode.FULL)
    rng = np.random.default_rng(5)
    nl = (n + 63) // 64
    u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
    with pytest.raises(tm.ConvolutionPrecisionFailure):
        ctx.product_limbs(tm.Mode.FULL, u, u, p)


@pytest.mark.parametrize("lg", [17, 18])
@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.FULL, tm.Mode.HIGH])
def test_batched_multipass_products(ctx, mode, lg):
    """Batches beyond the single-product cutoff (L > 8192): at 2^17 the low
    and high products (L = 10240) run the fused kernel one CTA per product
    (k_small_product_big), the full one (L = 12544) and every 2^18 product
    run multi-pass chains concurrently on the batch workspaces; every
    product exact, per-product flags zero."""
    n, count = 1 << lg, 24 if lg == 17 else 10
    nl = n // 64
    w = port.mt19937_64(17 + int(mode), 2 * count * nl).reshape(count, 2, nl)
    u = np.ascontiguousarray(w[:, 0, :])
    v = np.ascontiguousarray(w[:, 1, :])
    p = sp(n, mode)
    out, flags = ctx.product_batched(p, u, v, return_flags=True)
    assert ctx.last_stats.transform_length > 8192
    assert not flags.any()
    for i in range(count):
        _check(mode, u[i], v[i], n, tm.from_limbs(out[i]))
    assert ctx.last_stats.max_round_err < TRIP


# Column lengths with compile-time column passes (k_multipass.cu kColCtShapes):
# 1728 = 12^3 and 1440 = 12 x 12 x 10 (prime-factor radices), 1792 = 16 x 16 x 7,
# 1400 = 8 x 5 x 5 x 7; each row length 4096.
_COLCT = [1728, 1440, 1792, 1400]


@pytest.mark.parametrize("A", _COLCT)
def test_compiled_column_shapes_exact(ctx, A):
    rng = np.random.default_rng(A)
    for mode, b, Nn in ((tm.Mode.LOW, 8, A * 4096), (tm.Mode.FULL, 10, A * 2048)):
        n = Nn * b - 5
        p = tm.manual_params(n, b, Nn, mode)
        assert p.transform_length == A * 4096
        nl = (n + 63) // 64
        u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        v = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        r = ctx.product_limbs(mode, u, v, p)
        if mode == tm.Mode.LOW:
            assert np.array_equal(r, port.oracle_low(u, v, n)), (A, mode)
        else:
            assert np.array_equal(r, port.oracle_full(u, v)[:len(r)]), (A, mode)
        assert ctx.last_stats.max_round_err < TRIP


def _opt_ctx(*opts):
    c = tm.Context(0)
    for o, v in opts:
        c.set_option(o, v)
    return c


def _config3_all_modes(c, n=1 << 26):
    u, v = port.config_operands(3, (n + 63) // 64)
    P = port.limbs_to_int(port.oracle_full(u, v))
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        r = tm.from_limbs(c.product_limbs(mode, u, v, sp(n, mode)))
        if mode == tm.Mode.FULL:
            assert r == P
        elif mode == tm.Mode.LOW:
            assert r == P & ((1 << n) - 1)
        else:
            assert abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)
        assert c.last_stats.max_round_err < TRIP


def test_generic_passes_at_compiled_lengths():
    """TMG_OPT_GENERIC_COLUMN_PASSES: the runtime-dispatched column passes
    (radix-16/4/3 schedules of 1728 and 1440) give the same products as the
    compiled prime-factor ones (BASELINE config 3 lengths)."""
    c = _opt_ctx((tm._native.TMG_OPT_GENERIC_COLUMN_PASSES, 1))
    _config3_all_modes(c)
    c.close()


def test_generic_row_pass():
    """TMG_OPT_GENERIC_ROW_PASS: the runtime-dispatched row pass (k_mid) in
    place of the compiled C = 4096 one, two- and three-pass plans."""
    c = _opt_ctx((tm._native.TMG_OPT_GENERIC_ROW_PASS, 1))
    _config3_all_modes(c, 1 << 22)
    c.close()
    c = _opt_ctx((tm._native.TMG_OPT_GENERIC_ROW_PASS, 1), (tm._native.TMG_OPT_FORCE_THREE_PASS, 1))
    _config3_all_modes(c, 1 << 22)
    assert c.last_stats.passes == 3
    c.close()


@pytest.mark.parametrize("kernels", [0, 2, 3])
@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 448])
def test_carry_in_from_the_lanes_ticket(n, kernels):
    """TMG_OPT_PATCH_SCAN_MAX = 0: full, low and high products take the
    carry-ins the last block of k_carry_lanes (TMG_OPT_CARRY_KERNELS 2) or
    of k_carry_runs (3) scans -- the two-kernel path above 4096 carry blocks
    -- instead of k_carry_patch's own scan; 0: whatever the size picks."""
    c = _opt_ctx((tm._native.TMG_OPT_PATCH_SCAN_MAX, 0), (tm._native.TMG_OPT_CARRY_KERNELS, kernels))
    _config3_all_modes(c, n)
    c.close()


@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 448, 1 << 24])
def test_lookback_carry_path(n):
    """TMG_OPT_LOOKBACK_CARRY: the single-pass decoupled look-back carry
    (k_carry) and the high product's k_high_agg -- the path the library takes
    beyond 2^32 carry bits -- give the same products."""
    c = _opt_ctx((tm._native.TMG_OPT_LOOKBACK_CARRY, 1))
    _config3_all_modes(c, n)
    c.close()


def test_lookback_carry_structured_operands():
    """Long carry chains through the look-back carry (all-ones operands)."""
    c = _opt_ctx((tm._native.TMG_OPT_LOOKBACK_CARRY, 1))
    n = (1 << 20) + 3
    nl = (n + 63) // 64
    M = (1 << n) - 1
    for a, b_ in ((M, M), (M, 1 << (n - 1)), ((1 << n) - (1 << 1000), M - 5)):
        u, v = port.int_to_limbs(a, nl), port.int_to_limbs(b_, nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            try:
                r = tm.from_limbs(c.product_limbs(mode, u, v, sp(n, mode)))
            except tm.ConvolutionPrecisionFailure:
                continue
            _check(mode, u, v, n, r)
    c.close()


def test_check_clears_a_refused_status(ctx):
    """A refused device-pointer product raises at the next tmg_check, and the
    check after it -- of good products only -- passes: the status word is
    cleared before the error is reported."""
    import torch
    bad = tm.manual_params(3840, 30, 128, tm.Mode.LOW, tm.Backend.FFT, signed_split=False, lam=4)
    top = np.full(60, np.uint64(0xFFFFFFFFFFFFFFFF))
    n = 1 << 20
    good = sp(n, tm.Mode.LOW)
    rng = np.random.default_rng(3)
    u, v = _rand(rng, n), _rand(rng, n)
    dt = torch.from_numpy(top.view(np.int64)).cuda()
    dtout = torch.zeros(60, dtype=torch.int64, device="cuda")
    du = torch.from_numpy(u.view(np.int64)).cuda()
    dv = torch.from_numpy(v.view(np.int64)).cuda()
    out = torch.zeros(n // 64, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    c = tm.Context(0)
    c.product_device(bad, dt.data_ptr(), dt.data_ptr(), dtout.data_ptr(), 1)
    with pytest.raises(tm.ConvolutionPrecisionFailure):
        c.check()
    c.product_device(good, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
    c.check()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), port.oracle_low(u, v, n))
    c.close()


def test_contexts_sharing_one_stream_chain():
    """Two contexts on one caller stream, each product reading the previous
    one's output (written by the other context's kernels, still in flight):
    device-pointer products wait for their predecessor before reading."""
    import torch
    n = 1 << 20
    nl = n // 64
    s = torch.cuda.Stream()
    c1, c2 = tm.Context(0), tm.Context(0)
    c1.set_stream(s.cuda_stream)
    c2.set_stream(s.cuda_stream)
    p = sp(n, tm.Mode.LOW)
    rng = np.random.default_rng(17)
    a, b = _rand(rng, n), _rand(rng, n)
    bufs = [torch.from_numpy(x.view(np.int64)).cuda() for x in (a, b)]
    bufs += [torch.zeros(nl, dtype=torch.int64, device="cuda") for _ in range(8)]
    torch.cuda.synchronize()
    for k in range(8):
        (c1 if k % 2 == 0 else c2).product_device(p, bufs[k].data_ptr(), bufs[k + 1].data_ptr(),
                                                   bufs[k + 2].data_ptr(), 1)
    c1.check()
    c2.check()
    M = (1 << n) - 1
    xs = [port.limbs_to_int(a), port.limbs_to_int(b)]
    for k in range(8):
        xs.append(xs[k] * xs[k + 1] & M)
    got = [port.limbs_to_int(t.cpu().numpy().view(np.uint64)) for t in bufs]
    assert got == xs
    c1.close()
    c2.close()


def test_plan_cache_distinguishes_every_param_field(ctx):
    """Params equal in (n, b, N, lambda, mode) but not in signed_split or p
    must not share a cached plan: the unsigned split after the signed one is
    still exact, and a wrong p is refused on a would-be cache hit."""
    n = 20000
    rng = np.random.default_rng(23)
    u, v = _rand(rng, n), _rand(rng, n)
    ps = tm.manual_params(n, 10, 2048, tm.Mode.LOW, tm.Backend.FFT, signed_split=True)
    pu = tm.manual_params(n, 10, 2048, tm.Mode.LOW, tm.Backend.FFT, signed_split=False)
    for p in (ps, pu):
        assert np.array_equal(ctx.product_limbs(tm.Mode.LOW, u, v, p), port.oracle_low(u, v, n))
    from dataclasses import replace
    with pytest.raises(tm.Error):
        ctx.product_limbs(tm.Mode.LOW, u, v, replace(ps, p=ps.p + 7))


def test_batched_graph_replay(ctx):
    """Repeated multi-pass batch shapes run eagerly, then are captured, then
    replayed as a CUDA graph; every call uploads new operands into the same
    device buffers and must still be exact.  A larger batch in between
    reallocates the workspaces, which must invalidate the captured graph."""
    n, count = 1 << 18, 10
    nl = n // 64
    p = sp(n, tm.Mode.LOW)
    # reps 0-2: eager, capture, replay; the larger batch before rep 3
    # reallocates; reps 3-5: eager, capture, replay again
    for rep in range(6):
        if rep == 3:
            # grows the batch workspaces (and the context's operand buffers)
            nb = 1 << 20
            wb = port.mt19937_64(99, 2 * 4 * (nb // 64)).reshape(4, 2, nb // 64)
            ub, vb = np.ascontiguousarray(wb[:, 0, :]), np.ascontiguousarray(wb[:, 1, :])
            pb = sp(nb, tm.Mode.LOW)
            outb = ctx.product_batched(pb, ub, vb)
            for i in range(4):
                _check(tm.Mode.LOW, ub[i], vb[i], nb, tm.from_limbs(outb[i]))
        w = port.mt19937_64(40 + rep, 2 * count * nl).reshape(count, 2, nl)
        u = np.ascontiguousarray(w[:, 0, :])
        v = np.ascontiguousarray(w[:, 1, :])
        out, flags = ctx.product_batched(p, u, v, return_flags=True)
        assert not flags.any()
        for i in range(count):
            _check(tm.Mode.LOW, u[i], v[i], n, tm.from_limbs(out[i]))


def test_batched_full_2p16_compiled_small_kernel(ctx):
    """Full products of 2^16 bits (L = 6144) run the fused kernel with the
    compile-time 8 x 8 x 8 x 12 schedule (k_small_6144); a batch is exact."""
    n, count = 1 << 16, 64
    nl = n // 64
    w = port.mt19937_64(61, 2 * count * nl).reshape(count, 2, nl)
    u, v = np.ascontiguousarray(w[:, 0, :]), np.ascontiguousarray(w[:, 1, :])
    p = sp(n, tm.Mode.FULL)
    out, flags = ctx.product_batched(p, u, v, return_flags=True)
    assert ctx.last_stats.transform_length == 6144
    assert not flags.any()
    for i in range(count):
        _check(tm.Mode.FULL, u[i], v[i], n, tm.from_limbs(out[i]))


@pytest.mark.parametrize("n", [1 << 26, (1 << 26) - 4099])
def test_first_pass_premap_matches_split_premap(ctx, n):
    """k_f1d_ct (the first column pass pre-maps the split's stored digits)
    against TMG_OPT_PREMAP_IN_SPLIT (k_zgen pre-maps, k_f1_ct reads the
    coefficients): same arithmetic in the same order, so identical products
    and identical rounding residuals; both exact against GMP.  Seeded random
    operands and the alternating / all-ones structured ones."""
    old = _opt_ctx((tm._native.TMG_OPT_PREMAP_IN_SPLIT, 1))
    nl = (n + 63) // 64
    rng = np.random.default_rng(n)
    alt = np.array([~0 if i % 2 == 0 else 0 for i in range(nl)], dtype=np.int64).view(np.uint64)
    ones = np.full(nl, ~np.uint64(0), dtype=np.uint64)
    if n % 64:
        alt[-1] &= np.uint64((1 << (n % 64)) - 1)
        ones[-1] &= np.uint64((1 << (n % 64)) - 1)
    for u, v in ((_rand(rng, n), _rand(rng, n)), (alt, ones)):
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = sp(n, mode)
            try:
                a = ctx.product_limbs(mode, u, v, p)
            except tm.ConvolutionPrecisionFailure:
                with pytest.raises(tm.ConvolutionPrecisionFailure):
                    old.product_limbs(mode, u, v, p)
                continue
            ea = ctx.last_stats.max_round_err
            b = old.product_limbs(mode, u, v, p)
            assert np.array_equal(a, b), mode
            assert ea == old.last_stats.max_round_err, mode
            _check(mode, u, v, n, tm.from_limbs(a))
    old.close()


@pytest.mark.parametrize("kernels", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [1 << 20, (1 << 22) + 448, 1 << 24])
def test_carry_kernel_paths(n, kernels):
    """TMG_OPT_CARRY_KERNELS: the single-pass look-back k_carry_lb (1),
    k_carry_lanes + k_carry_patch (2), k_carry_runs + k_carry_patch (3) and
    the single-pass k_carry_runs (4; 5 here: with TMG_OPT_GENERIC_RUNS, the
    chunk width a run-time value) at sizes where the default takes another;
    random and structured (long carry chains) operands, every path identical
    to the default and exact."""
    opts = [(tm._native.TMG_OPT_CARRY_KERNELS, min(kernels, 4))]
    if kernels == 5:
        opts.append((tm._native.TMG_OPT_GENERIC_RUNS, 1))
    c = _opt_ctx(*opts)
    _config3_all_modes(c, n)
    nl = (n + 63) // 64
    M = (1 << n) - 1
    for a, b_ in ((M, M), (M, 1 << (n - 1)), ((1 << n) - (1 << 1000), M - 5)):
        u, v = port.int_to_limbs(a, nl), port.int_to_limbs(b_, nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            r1 = c.product_limbs(mode, u, v, sp(n, mode))
            r0 = tm.default_context(0).product_limbs(mode, u, v, sp(n, mode))
            assert np.array_equal(r0, r1)
            _check(mode, u, v, n, tm.from_limbs(r0))
    c.close()


@pytest.mark.parametrize("n", [1 << 18, 1 << 20, (1 << 22) + 448])
def test_split_carry_in_paths(n):
    """TMG_OPT_SPLIT_AGGREGATES: the split's block carry-ins composed from
    k_zstat's aggregates, against the default look-back inside k_zgen for
    one-wave grids; random operands and long balanced-carry chains (windows
    equal to 2^{b-1} over many blocks: limbs 0x8080...)."""
    c = _opt_ctx((tm._native.TMG_OPT_SPLIT_AGGREGATES, 1))
    _config3_all_modes(c, n)
    nl = (n + 63) // 64
    M = (1 << n) - 1
    chain = int.from_bytes(bytes([0x80]) * (nl * 8), "little") & M
    for a, b_ in ((M, M), (chain, chain), (chain, M - 5)):
        u, v = port.int_to_limbs(a, nl), port.int_to_limbs(b_, nl)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            try:
                r0 = tm.default_context(0).product_limbs(mode, u, v, sp(n, mode))
            except tm.ConvolutionPrecisionFailure:
                # a structured spectrum the policy's b cannot certify: the
                # other path refuses it the same way
                with pytest.raises(tm.ConvolutionPrecisionFailure):
                    c.product_limbs(mode, u, v, sp(n, mode))
                continue
            r1 = c.product_limbs(mode, u, v, sp(n, mode))
            assert np.array_equal(r0, r1)
            _check(mode, u, v, n, tm.from_limbs(r0))
    c.close()


@pytest.mark.parametrize("n", [1 << 24, (1 << 24) + 12345])
def test_split_by_runs_carry_chains(n):
    """k_zsplit (the split by runs, default from about 2^23 bits) against
    the block-scan split k_zgen (TMG_OPT_SPLIT_KERNEL = 1) and GMP: random
    operands with stretches of windows equal to 2^{b-1} -- the windows through
    which a run's carry-in comes from further below (carry_below) -- placed
    across run, block and tile-row boundaries, both with a carry arriving at
    the stretch (the window below it above 2^{b-1}) and without."""
    c = _opt_ctx((tm._native.TMG_OPT_SPLIT_KERNEL, 1))
    rng = np.random.default_rng(n & 0xffff)
    nl = (n + 63) // 64
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        p = sp(n, mode)
        b, N = p.b, p.N
        lead = (N + 1) * b - n if mode == tm.Mode.HIGH else 0
        ops = []
        for carry_first in (False, True):
            x = int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1)
            # stretches [j1, j2) of chunks (of the operand shifted up by lead)
            for j1, length in ((31, 3), (8190, 70), (4096 * 3 - 40, 100), (8192 * 5 + 33, 64), (100000, 1)):
                for j in range(j1, j1 + length):
                    pos = j * b - lead
                    if pos < 0 or pos + b > n:
                        continue
                    x &= ~(((1 << b) - 1) << pos)
                    x |= (1 << (b - 1)) << pos
                pos = (j1 - 1) * b - lead
                if carry_first and pos >= 0:
                    x |= ((1 << b) - 1) << pos  # all ones: above 2^{b-1}, a carry enters the stretch
            ops.append(port.int_to_limbs(x, nl))
        u, v = ops
        r0 = tm.default_context(0).product_limbs(mode, u, v, p)
        r1 = c.product_limbs(mode, u, v, p)
        assert np.array_equal(r0, r1)
        _check(mode, u, v, n, tm.from_limbs(r0))
    c.close()


@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.HIGH])
def test_split_by_runs_long_half_window_stretches(mode):
    """Carry walks that leave a run's row segment and its block: stretches of
    several thousand to a million windows equal to 2^{b-1} (one of them down
    to chunk 0), with and without a carry arriving below them; the carry into
    a segment's first chunk then comes from the block's per-segment warp walk
    (k_zsplit).  Against the block-scan split k_zgen and GMP; the second
    operand is random so that the product certifies."""
    n = 1 << 24
    c = _opt_ctx((tm._native.TMG_OPT_SPLIT_KERNEL, 1))
    rng = np.random.default_rng(77 + int(mode))
    nl = n // 64
    # the 2^26 products' chunk width and length (b = 12, N = 5 898 240): the
    # long runs of equal digits concentrate the spectrum, and 2^24's own b = 13
    # refuses them; one bit less certifies all but the longest
    p26 = sp(1 << 26, mode)
    p = tm.manual_params(n, p26.b, p26.N, mode, lam=p26.lam)
    b, N = p.b, p.N
    lead = (N + 1) * b - n if mode == tm.Mode.HIGH else 0
    v = _rand(rng, n)
    refused = 0
    for stretches, carry in ((((0, 20000),), False), (((5000, 1200000),), True),
                             (((3, 9000), (40000, 300000), (700001, 2500)), True)):
        x = int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1)
        off = -(-lead // b)  # first chunk that holds operand bits (the high split is top-aligned)
        for j1, length in stretches:
            lo = max((j1 + off) * b - lead, 0)
            hi = min((j1 + off + length) * b - lead, n - (n % b) - b)
            # whole windows [lo, hi) (aligned to the chunk grid) set to 2^{b-1}
            lo += (-(lo + lead)) % b
            hi -= (hi + lead) % b
            k = (hi - lo) // b
            pat = (((1 << (b * k)) - 1) // ((1 << b) - 1)) << (b - 1)
            x &= ~(((1 << (hi - lo)) - 1) << lo)
            x |= pat << lo
            if carry and lo >= b:
                x |= ((1 << b) - 1) << (lo - b)
        u = port.int_to_limbs(x & ((1 << n) - 1), nl)
        d = tm.default_context(0)
        try:
            r0 = d.product_limbs(mode, u, v, p)
        except tm.ConvolutionPrecisionFailure:
            # a million equal digits of full magnitude: the transform's coherent
            # error refuses the product (Numerics); the two splits
            # must then refuse alike, with the same residual
            e0 = d.last_stats.max_round_err
            with pytest.raises(tm.ConvolutionPrecisionFailure):
                c.product_limbs(mode, u, v, p)
            assert c.last_stats.max_round_err == e0
            refused += 1
            continue
        e0 = d.last_stats.max_round_err
        r1 = c.product_limbs(mode, u, v, p)
        assert np.array_equal(r0, r1) and c.last_stats.max_round_err == e0
        _check(mode, u, v, n, tm.from_limbs(r0))
        r2 = d.product_limbs(mode, v, u, p)
        assert np.array_equal(r0, r2)
    assert refused <= 1  # the first and the last operand certify (residuals 0.012 and 0.10)
    c.close()
