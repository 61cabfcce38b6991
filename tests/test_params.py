"""Parameter selection and validation through the C ABI (host-only calls;
no GPU needed).  Mirrors /root/reference/proj/tests/test_products.cpp:179-274
plus the accuracy-aware policy of DESIGN.md."""
import json
import math
import os

import pytest

import paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import Backend, Mode, Policy

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_policy_pins_million_bit_rows():
    pins = json.load(open(os.path.join(GOLD, "params.json")))["reference_1e6"]
    for mode in ("low", "high", "full"):
        p = tm.select_params(1000000, Mode[mode.upper()], Backend.FFT, policy=Policy.REFERENCE)
        assert (p.b, p.N, p.lam, p.p) == tuple(pins[mode][k] for k in ("b", "N", "lambda", "p"))
        assert p.signed_split
        assert p.mode == Mode[mode.upper()]


def test_table1_truncated_row():
    # paper Table 1, n = 10^6: N = 2^11 * 35, b = 14, lambda = 4; full 2^14 * 3, b = 21
    lo = tm.select_params(1000000, Mode.LOW, policy=Policy.REFERENCE)
    assert lo.N == 2**11 * 35 and lo.b == 14 and lo.lam == 4
    fu = tm.select_params(1000000, Mode.FULL, policy=Policy.REFERENCE)
    assert fu.N == 2**14 * 3 and fu.b == 21


def test_fallback_cutoff():
    for c in json.load(open(os.path.join(GOLD, "params.json")))["fallback"]:
        p = tm.select_params(c["n"], Mode[c["mode"].upper()], Backend[c["backend"].upper()], c["cutoff"])
        expect = Mode.ORACLE_FALLBACK if c["mode_out"] == "fallback" else Mode[c["mode_out"].upper()]
        assert p.mode == expect
    tiny = tm.select_params(12, Mode.LOW, Backend.EXACT, 0)
    assert (tiny.b, tiny.N, tiny.p) == (4, 3, 20)


@pytest.mark.parametrize("n", [4096, 10001, 65536, 300000, 2154434, 1 << 26])
@pytest.mark.parametrize("mode", [Mode.FULL, Mode.LOW, Mode.HIGH])
@pytest.mark.parametrize("policy", [Policy.REFERENCE, Policy.ACCURATE])
def test_selected_params_validate(n, mode, policy):
    for backend in (Backend.EXACT, Backend.FFT):
        p = tm.select_params(n, mode, backend, policy=policy)
        assert p.mode == mode
        tm.validate_params(p)
        if backend == Backend.EXACT:
            assert p.N <= 4100 and not p.signed_split
        else:
            n_ = p.N
            for q in (2, 3, 5, 7):
                while n_ % q == 0:
                    n_ //= q
            assert n_ == 1 and p.signed_split


def test_validation_rejects_broken_shapes():
    good = tm.manual_params(12, 4, 3, Mode.LOW, Backend.EXACT, False)
    tm.validate_params(good)
    from dataclasses import replace
    for bad in (replace(good, p=good.p + 1), replace(good, b=3), replace(good, N=2),
                replace(good, n=13), replace(good, lam=0)):
        with pytest.raises(tm.InputOutOfRange):
            tm.validate_params(bad)
    high = tm.manual_params(10, 4, 3, Mode.HIGH, Backend.EXACT, False)
    tm.validate_params(high)
    with pytest.raises(tm.InputOutOfRange):
        tm.validate_params(replace(high, n=13))
    fft = tm.manual_params(44, 4, 11, Mode.LOW, Backend.FFT)
    with pytest.raises(tm.UnsupportedLength):
        tm.validate_params(fft)
    tm.validate_params(tm.manual_params(44, 4, 12, Mode.LOW, Backend.FFT))
    fb = tm.Params(n=8, mode=Mode.ORACLE_FALLBACK)
    tm.validate_params(fb)
    with pytest.raises(tm.InputOutOfRange):
        tm.validate_params(replace(fb, n=0))


def test_required_precision_and_lambda():
    assert tm.required_precision(Mode.FULL, 21, 49152) == 2 * 21 + 16 + 2
    assert tm.required_precision(Mode.LOW, 14, 71680) == 3 * 14 + 17 + 6
    assert tm.required_precision(Mode.HIGH, 14, 71680) == 3 * 14 + 17 + 9
    assert tm.default_lambda(Mode.LOW, Backend.FFT, 14, 65) == 4
    assert tm.default_lambda(Mode.LOW, Backend.FFT, 12, 65) == 5
    assert tm.default_lambda(Mode.FULL, Backend.FFT, 21, 60) == 0
    assert tm.default_lambda(Mode.LOW, Backend.EXACT, 4, 20) == (20 + 2 + 4 - 3) // (4 - 2)
    with pytest.raises(tm.InputOutOfRange):
        tm.default_lambda(Mode.LOW, Backend.FFT, 3, 20)


@pytest.mark.parametrize("n", [1 << 16, 1 << 20, 1000000, 1 << 24, 1 << 26, 1 << 28])
def test_accurate_policy_bounds_predicted_error(n):
    for mode in (Mode.FULL, Mode.LOW, Mode.HIGH):
        a = tm.select_params(n, mode, policy=Policy.ACCURATE)
        r = tm.select_params(n, mode, policy=Policy.REFERENCE)
        assert a.b <= r.b
        assert tm.predicted_sigma(a) <= 0.25 / 7 + 1e-12
        # reference budget still respected
        L = a.transform_length
        assert (2 if mode == Mode.FULL else 3) * a.b + 0.5 * math.log2(L) <= 50.5


def test_accurate_policy_at_benchmark_size():
    """At n = 2^26 the reference picks b = 13 for low/high, whose FP64 error
    exceeds its own 0.25 tripwire; the accurate policy drops to
    b = 12 and keeps the full product at the reference's b = 19."""
    n = 1 << 26
    assert tm.select_params(n, Mode.LOW, policy=Policy.REFERENCE).b == 13
    assert tm.select_params(n, Mode.LOW, policy=Policy.ACCURATE).b == 12
    assert tm.select_params(n, Mode.HIGH, policy=Policy.ACCURATE).b == 12
    full = tm.select_params(n, Mode.FULL, policy=Policy.ACCURATE)
    assert full.b == 19 and full.N == 1728 * 2048  # L = 1728 x 4096 (compiled 12^3 columns)
    assert tm.predicted_sigma(tm.select_params(n, Mode.LOW, policy=Policy.REFERENCE)) > 0.25 / 7


def test_output_limbs():
    assert tm.output_limbs(Mode.FULL, 64) == 2
    assert tm.output_limbs(Mode.LOW, 65) == 2
    assert tm.output_limbs(Mode.HIGH, 64) == 2
    assert tm.output_limbs(Mode.HIGH, 63) == 1


@pytest.mark.parametrize("n", list(range(4096, 4600, 37)) + [5001, 7777, 12345, 20011])
@pytest.mark.parametrize("mode", [Mode.FULL, Mode.LOW, Mode.HIGH])
def test_accurate_policy_lengths_suit_the_gpu(n, mode):
    """The accurate (GPU) policy only picks transform lengths divisible by 4
    (small n used to admit odd 2357-smooth N such as 175)."""
    p = tm.select_params(n, mode, policy=Policy.ACCURATE)
    assert p.transform_length % 4 == 0


def test_accurate_policy_prefers_compiled_column_schedules():
    """At n = 2^26 the GPU cost model counts the compiled three-stage column
    schedules (1728 = 12^3, 1440 = 12 x 12 x 10; prime-factor radices), so the
    full product takes L = 1728 x 4096 and the truncated ones 1440 x 4096."""
    n = 1 << 26
    full = tm.select_params(n, Mode.FULL, policy=Policy.ACCURATE)
    low = tm.select_params(n, Mode.LOW, policy=Policy.ACCURATE)
    high = tm.select_params(n, Mode.HIGH, policy=Policy.ACCURATE)
    assert full.transform_length == 1728 * 4096 and full.b == 19
    assert low.transform_length == 1440 * 4096 and low.b == 12
    assert high.transform_length == 1440 * 4096 and high.b == 12
    # the reference policy is untouched by the GPU cost model
    assert tm.select_params(n, Mode.LOW, policy=Policy.REFERENCE).b == 13
