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


@pytest.mark.parametrize("n", [4096, 5001, 8192, 20011, 65536, 100003, 262144, 1000000, 1 << 22])
def test_random_products_match_exact(ctx, n):
    rng = np.random.default_rng(n)
    for _ in range(3):
        u, v = _rand(rng, n), _rand(rng, n)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = tm.select_params(n, mode)
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
            p = tm.select_params(n, mode)
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
            p = tm.select_params(n, mode)
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
    pl, pf, ph = (tm.select_params(n, m) for m in (tm.Mode.LOW, tm.Mode.FULL, tm.Mode.HIGH))
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
                r = tm.from_limbs(ctx.product_limbs(mode, u, v, tm.select_params(n, mode)))
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
            r = tm.from_limbs(esc_ctx.product_limbs(mode, u, v, tm.select_params(n, mode)))
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
        ref = tm.select_params(n, mode)
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
    p = tm.select_params(8192, tm.Mode.LOW)
    with pytest.raises(tm.InputOutOfRange):
        tm.low_product(1 << 8192, 3, p, ctx)
    with pytest.raises(tm.InputOutOfRange):
        tm.full_product(3, 5, p, ctx)  # params built for a different mode


def test_fallback_below_cutoff(ctx):
    rng = np.random.default_rng(6)
    for n in (1, 7, 64, 65, 1000, 4095):
        u, v = _rand(rng, n), _rand(rng, n)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = tm.select_params(n, mode)
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
    p = tm.select_params(n, tm.Mode.LOW)
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
ctx = tm.Context(0)
bad = 0
for n in (1 << 20, 1 << 22):
    nl = n // 64
    rng = np.random.default_rng(n)
    p = tm.select_params(n, tm.Mode.LOW)
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
p1, p2 = tm.select_params(n1, tm.Mode.LOW), tm.select_params(n2, tm.Mode.LOW)
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
    p = tm.select_params(n, tm.Mode.LOW)
    r = ctx.product_limbs(tm.Mode.LOW, u, v, p)
    assert np.array_equal(r, port.oracle_low(u, v, n))
    assert ctx.last_stats.max_round_err < TRIP


def test_config2_high_2p24_seed2(ctx):
    n = 1 << 24
    u, v = port.config_operands(2, n // 64, force_top_bit=True)
    p = tm.select_params(n, tm.Mode.HIGH)
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
        p = tm.select_params(n, mode)
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
    p = tm.select_params(n, tm.Mode.LOW)
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


@pytest.mark.parametrize("pattern", ["ones", "alternating"])
@pytest.mark.parametrize("mode", [tm.Mode.LOW, tm.Mode.HIGH])
def test_config5_stress_2p28(esc_ctx, pattern, mode):
    """BASELINE config 5: u = v = 2^n - 1 and alternating all-ones / zero
    limbs at n = 2^28.  The alternating pattern concentrates the spectrum on
    a few lines, outside the random-input error model the accurate policy
    uses; with escalation the product is recomputed at b - 1 when the first
    attempt refuses, and the result must be exact either way."""
    n = 1 << 28
    nl = n // 64
    if pattern == "ones":
        u = np.full(nl, np.uint64(0xFFFFFFFFFFFFFFFF))
    else:
        u = np.zeros(nl, dtype=np.uint64)
        u[0::2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    v = u.copy()
    p = tm.select_params(n, mode)
    r = tm.from_limbs(esc_ctx.product_limbs(mode, u, v, p))
    st = esc_ctx.last_stats
    print(f"stress {pattern} {mode.name}: first attempt b={p.b} residual {st.first_round_err:.4f}; "
          f"result from attempt {st.attempts} (b={st.b}, N={st.N}) residual {st.max_round_err:.4f}")
    assert st.max_round_err < TRIP
    assert st.attempts == 1 or (st.escalated and st.b < p.b and st.first_round_err >= TRIP)
    _check(mode, u, v, n, r)


def test_escalation_recovers_refused_alternating_product(esc_ctx, ctx):
    """2^22 alternating limbs: the accurate-policy b = 13 refuses on the GPU
    (and the reference refuses the same pattern at 2^24); escalation returns
    the exact low product."""
    n = 1 << 22
    u = np.zeros(n // 64, dtype=np.uint64)
    u[0::2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    p = tm.select_params(n, tm.Mode.LOW)
    try:
        r0 = ctx.product_limbs(tm.Mode.LOW, u, u, p)
        assert np.array_equal(r0, port.oracle_low(u, u, n))
    except tm.ConvolutionPrecisionFailure:
        pass
    r = esc_ctx.product_limbs(tm.Mode.LOW, u, u, p)
    assert np.array_equal(r, port.oracle_low(u, u, n))
    assert esc_ctx.last_stats.max_round_err < TRIP


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
    p = tm.select_params(n, mode)
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


_FALLBACK_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from oracle import port
ctx = tm.default_context(0)
n = 1 << 26
u, v = port.config_operands(3, n // 64)
P = port.limbs_to_int(port.oracle_full(u, v))
for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
    p = tm.select_params(n, mode)
    r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
    if mode == tm.Mode.FULL:
        assert r == P
    elif mode == tm.Mode.LOW:
        assert r == P & ((1 << n) - 1)
    else:
        assert abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)
print("ok")
"""


def test_generic_passes_at_compiled_lengths():
    """TMG_NO_COLCT: the runtime-dispatched column passes (radix-16/4/3
    schedules of 1728 and 1440) give the same products as the compiled
    prime-factor ones (BASELINE config 3 lengths)."""
    import subprocess
    import sys
    env = dict(os.environ, TMG_NO_COLCT="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FALLBACK_SNIPPET], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


_CARRY_SNIPPET = """
import sys
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from oracle import port
ctx = tm.Context(0)
for n in (1 << 20, (1 << 22) + 448):
    u, v = port.config_operands(3, (n + 63) // 64)
    P = port.limbs_to_int(port.oracle_full(u, v))
    assert tm.from_limbs(ctx.product_limbs(tm.Mode.FULL, u, v, tm.select_params(n, tm.Mode.FULL))) == P
    assert tm.from_limbs(ctx.product_limbs(tm.Mode.LOW, u, v, tm.select_params(n, tm.Mode.LOW))) == P % (1 << n)
    w = tm.from_limbs(ctx.product_limbs(tm.Mode.HIGH, u, v, tm.select_params(n, tm.Mode.HIGH)))
    assert 0 <= w <= (1 << n) and abs(P - (w << n)) < (1 << n)
print("ok")
"""


def test_carry_in_from_the_lanes_ticket():
    """TMG_PATCH_SCAN_MAX=0: full, low and high products take the carry-ins the
    last k_carry_lanes block scans (the path above 4096 carry blocks, n >~
    2^27) instead of k_carry_patch's own scan; the results must not change."""
    import subprocess
    import sys
    env = dict(os.environ, TMG_PATCH_SCAN_MAX="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CARRY_SNIPPET], cwd=root, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_batched_graph_replay(ctx):
    """Repeated multi-pass batch shapes run eagerly, then are captured, then
    replayed as a CUDA graph; every call uploads new operands into the same
    device buffers and must still be exact.  A larger batch in between
    reallocates the workspaces, which must invalidate the captured graph."""
    n, count = 1 << 18, 10
    nl = n // 64
    p = tm.select_params(n, tm.Mode.LOW)
    # reps 0-2: eager, capture, replay; the larger batch before rep 3
    # reallocates; reps 3-5: eager, capture, replay again
    for rep in range(6):
        if rep == 3:
            # grows the batch workspaces (and the context's operand buffers)
            nb = 1 << 20
            wb = port.mt19937_64(99, 2 * 4 * (nb // 64)).reshape(4, 2, nb // 64)
            ub, vb = np.ascontiguousarray(wb[:, 0, :]), np.ascontiguousarray(wb[:, 1, :])
            pb = tm.select_params(nb, tm.Mode.LOW)
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
    p = tm.select_params(n, tm.Mode.FULL)
    out, flags = ctx.product_batched(p, u, v, return_flags=True)
    assert ctx.last_stats.transform_length == 6144
    assert not flags.any()
    for i in range(count):
        _check(tm.Mode.FULL, u[i], v[i], n, tm.from_limbs(out[i]))
