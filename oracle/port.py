"""CPU oracle for the truncated-product hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference's float pipeline (arxiv 1703.00640 artifact,
/root/reference/proj/core/src/products_f64.cpp:106-171) on the CPU:

    split (split.cpp:66-102)  -> oracle.c orc_split
    alpha*/gamma+ (maps_f64.cpp:259-348) -> oracle.c
    real cyclic convolution    -> numpy.fft.rfft/irfft (pocketfft), standing in
                                  for the reference's FFTW r2c/c2r plans
                                  (convolution.cpp:175-195; FFTW 3 is not in
                                  this image)
    beta*/delta+ (maps_f64.cpp:269-384) -> oracle.c
    round_accumulate + SignedAccumulator (products_f64.cpp:16-102) -> oracle.c

plus independent exact products for checking (oracle_full / oracle_low /
oracle_high_set of oracle.hpp:20-35): GMP's mpn_mul (GMP 6.3.0, the
reference's own bignum dependency, through the system libgmp.so.10) and
oracle.c's hand-rolled Karatsuba restating oracle.cpp:69-130.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_gmp = None


class OracleError(Exception):
    pass


class ConvolutionPrecisionFailure(OracleError):
    """products_f64.cpp tripwires (errors.hpp:63-67)."""


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P64 = ctypes.POINTER(ctypes.c_uint64)
        PD = ctypes.POINTER(ctypes.c_double)
        PI64 = ctypes.POINTER(ctypes.c_int64)
        i64 = ctypes.c_int64
        L.orc_mt19937_64.argtypes = [ctypes.c_uint64, P64, i64]
        L.orc_split.argtypes = [P64, i64, ctypes.c_int, i64, ctypes.c_int, i64, PD]
        L.orc_coeff_table.argtypes = [ctypes.c_int, i64, i64, ctypes.c_int, PD]
        L.orc_alpha_star_inplace.argtypes = [PD, i64, i64, PD]
        L.orc_beta_star.argtypes = [PD, i64, i64, ctypes.c_int, PD, PD]
        L.orc_gamma_dagger_inplace.argtypes = [PD, i64, i64, ctypes.c_int, PD, PD]
        L.orc_delta_dagger.argtypes = [PD, i64, i64, ctypes.c_int, PD, ctypes.c_double, PD]
        L.orc_round_accumulate.argtypes = [PD, i64, ctypes.c_int, ctypes.c_int, P64, i64, PI64, PD, PD]
        L.orc_limb_mul.argtypes = [P64, i64, P64, i64, P64]
        _lib = L
    return _lib


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _pd(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
# limbs <-> int


def limbs_to_int(limbs) -> int:
    a = np.ascontiguousarray(limbs, dtype=np.uint64)
    return int.from_bytes(a.tobytes(), "little")


def int_to_limbs(x: int, nlimbs: int) -> np.ndarray:
    if x < 0:
        raise ValueError("negative")
    b = x.to_bytes(nlimbs * 8, "little")
    return np.frombuffer(b, dtype=np.uint64).copy()


# ---------------------------------------------------------------------------
# inputs (gen_inputs.cpp:76-83 uses std::mt19937_64 words in order)


def mt19937_64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().orc_mt19937_64(ctypes.c_uint64(seed), _p64(out), count)
    return out


def random_bits_pairs(seed: int, n: int, count: int):
    """The operand pairs of the reference's FFT product tests: u, v =
    testsup::random_bits(rng, n) in turn (test_support.hpp:17-22: ceil(n/64)
    mt19937_64 words, little-endian, low n bits) from std::mt19937_64(seed),
    as in test_products.cpp:371-406."""
    nl = (n + 63) // 64
    w = mt19937_64(seed, 2 * count * nl).reshape(count, 2, nl)
    if n % 64:
        w[:, :, -1] &= np.uint64((1 << (n % 64)) - 1)
    return [(w[i, 0].copy(), w[i, 1].copy()) for i in range(count)]


def config_operands(seed: int, nlimbs: int, force_top_bit: bool = False):
    """u = words[0:nl], v = words[nl:2nl] of mt19937_64(seed)."""
    w = mt19937_64(seed, 2 * nlimbs)
    u, v = w[:nlimbs].copy(), w[nlimbs:].copy()
    if force_top_bit:
        u[-1] |= np.uint64(1 << 63)
        v[-1] |= np.uint64(1 << 63)
    return u, v


# ---------------------------------------------------------------------------
# exact products


def _gmp_lib():
    global _gmp
    if _gmp is None:
        for name in ("libgmp.so.10", "/usr/lib/x86_64-linux-gnu/libgmp.so.10"):
            try:
                _gmp = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _gmp is None:
            raise OracleError("libgmp.so.10 not found")
        _gmp.__gmpn_mul.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long,
                                    ctypes.c_void_p, ctypes.c_long]
        _gmp.__gmpn_mul.restype = ctypes.c_uint64
    return _gmp


def gmp_mul(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Full product limbs (len(u) + len(v)) via GMP mpn_mul."""
    u = np.ascontiguousarray(u, dtype=np.uint64)
    v = np.ascontiguousarray(v, dtype=np.uint64)
    if len(u) < len(v):
        u, v = v, u
    r = np.zeros(len(u) + len(v), dtype=np.uint64)
    if len(v) == 0:
        return r
    _gmp_lib().__gmpn_mul(r.ctypes.data, u.ctypes.data, len(u), v.ctypes.data, len(v))
    return r


def limb_mul(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Karatsuba restatement of oracle.cpp:limb_mul (no GMP)."""
    u = np.ascontiguousarray(u, dtype=np.uint64)
    v = np.ascontiguousarray(v, dtype=np.uint64)
    r = np.zeros(len(u) + len(v), dtype=np.uint64)
    lib().orc_limb_mul(_p64(u), len(u), _p64(v), len(v), _p64(r))
    return r


def oracle_full(u, v) -> np.ndarray:
    return gmp_mul(u, v)


def oracle_low(u, v, n: int) -> np.ndarray:
    p = gmp_mul(u, v)
    nl = (n + 63) // 64
    out = p[:nl].copy()
    if n % 64:
        out[-1] &= np.uint64((1 << (n % 64)) - 1)
    return out


def oracle_high_set(u, v, n: int) -> list[int]:
    """All w in [0, 2^n] with |uv - 2^n w| < 2^n, ascending (oracle.hpp:27-31)."""
    p = limbs_to_int(gmp_mul(u, v))
    q, r = p >> n, p & ((1 << n) - 1)  # bit ops: divmod by 2^n is quadratic
    out = [q]
    if r != 0 and q + 1 <= (1 << n):
        out.append(q + 1)
    return out


def is_valid_high(u, v, n: int, w: int) -> bool:
    p = limbs_to_int(gmp_mul(u, v))
    return 0 <= w <= (1 << n) and abs(p - (w << n)) < (1 << n)


def low_int(p: int, n: int) -> int:
    return p & ((1 << n) - 1)


# ---------------------------------------------------------------------------
# the reference float pipeline


@dataclass
class Result:
    value: int
    max_err: float
    max_abs: float


def split(limbs, n: int, b: int, count: int, balanced: bool, lead: int = 0) -> np.ndarray:
    u = np.ascontiguousarray(limbs, dtype=np.uint64)
    out = np.empty(count, dtype=np.float64)
    if lib().orc_split(_p64(u), len(u), b, count, 1 if balanced else 0, lead, _pd(out)) != 0:
        raise OracleError("split: bad chunk width")
    return out


def coeff_table(fam: str, lam: int, N: int, b: int) -> np.ndarray:
    f = {"alpha": 0, "beta": 1, "gamma": 2, "delta": 3}[fam]
    t = np.empty(lam * N, dtype=np.float64)
    lib().orc_coeff_table(f, lam, N, b, _pd(t))
    return t


# Threads for the convolution FFTs.  None: numpy's pocketfft, one thread (the
# checker); an int: scipy's pocketfft with that many workers (the timed CPU
# baseline of bench.py, which uses every host thread it can).
FFT_WORKERS = None


# Where the 1/L of the convolution is applied.  "spectrum" is the reference's
# order (convolution.cpp:186-192): the product spectrum is multiplied by the
# rounded double 1.0/n and FFTW's unnormalised c2r plan runs on it.  "end"
# is pocketfft's normalised irfft (1/n on the outputs), kept for error
# studies: on structured operands it rounds less (Numerics).
SCALE_AT = "spectrum"


def cyclic_convolve(a: np.ndarray, c: np.ndarray) -> np.ndarray:
    """convolution.cpp:175-195: r2c of both inputs, pointwise product
    (re = a0 b0 - a1 b1, im = a0 b1 + a1 b0) times scale = 1.0 / n, c2r."""
    n = len(a)
    if FFT_WORKERS:
        import scipy.fft as sf
        fa = sf.rfft(a, workers=FFT_WORKERS)
        fc = sf.rfft(c, workers=FFT_WORKERS)
        if SCALE_AT == "end":
            return sf.irfft(fa * fc, n=n, workers=FFT_WORKERS)
        return sf.irfft((fa * fc) * (1.0 / n), n=n, norm="forward", workers=FFT_WORKERS)
    fa, fc = np.fft.rfft(a), np.fft.rfft(c)
    if SCALE_AT == "end":
        return np.fft.irfft(fa * fc, n=n)
    return np.fft.irfft((fa * fc) * (1.0 / n), n=n, norm="forward")


def _accumulate(vals: np.ndarray, scale: int, b: int, nout: int):
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    out = np.zeros(nout, dtype=np.uint64)
    sign = ctypes.c_int64(0)
    me = ctypes.c_double(0.0)
    ma = ctypes.c_double(0.0)
    st = lib().orc_round_accumulate(_pd(vals), len(vals), scale, b, _p64(out), nout,
                                    ctypes.byref(sign), ctypes.byref(me), ctypes.byref(ma))
    if st == 1:
        raise ConvolutionPrecisionFailure("float pipeline coefficient overflowed the exact-integer range")
    if st == 2:
        raise ConvolutionPrecisionFailure("float pipeline rounding tripwire: residual above a quarter")
    val = limbs_to_int(out)
    if sign.value < 0:
        val -= 1 << (64 * nout)
    return val, me.value, ma.value


def full_product(u, v, n: int, b: int, N: int, signed_split: bool = True) -> Result:
    """products_f64.cpp:106-121."""
    L = 2 * N
    a = np.zeros(L)
    c = np.zeros(L)
    a[:N] = split(u, n, b, N, signed_split)
    c[:N] = split(v, n, b, N, signed_split)
    w = cyclic_convolve(a, c)
    nout = (L * b + 128) // 64 + 4
    t, me, ma = _accumulate(w, 0, b, nout)
    if t < 0:
        raise ConvolutionPrecisionFailure("full product recombined negative")
    return Result(t, me, ma)


def low_product(u, v, n: int, b: int, N: int, lam: int, signed_split: bool = True) -> Result:
    """products_f64.cpp:123-143."""
    al = coeff_table("alpha", lam, N, b)
    be = coeff_table("beta", lam, N, b)
    a = split(u, n, b, N, signed_split)
    lib().orc_alpha_star_inplace(_pd(al), lam, N, _pd(a))
    c = split(v, n, b, N, signed_split)
    lib().orc_alpha_star_inplace(_pd(al), lam, N, _pd(c))
    w = np.ascontiguousarray(cyclic_convolve(a, c))
    low = np.empty(N)
    lib().orc_beta_star(_pd(be), lam, N, b, _pd(w), _pd(low))
    nout = (N * b + b + 128) // 64 + 4
    t, me, ma = _accumulate(low, b, b, nout)
    if t & ((1 << b) - 1):
        raise ConvolutionPrecisionFailure("low product recombination is not divisible by the chunk base")
    return Result((t >> b) & ((1 << n) - 1), me, ma)


def _round_even_shift(t: int, s: int) -> int:
    q, r = t >> s, t & ((1 << s) - 1)  # floor semantics for negative t
    half = 1 << (s - 1)
    if r > half or (r == half and (q & 1)):
        q += 1
    return q


def high_product(u, v, n: int, b: int, N: int, lam: int, signed_split: bool = True) -> Result:
    """products_f64.cpp:145-171."""
    ga = coeff_table("gamma", lam, N, b)
    de = coeff_table("delta", lam, N, b)
    sigma = (N + 1) * b - n
    a = np.zeros(N + 1)
    a[:] = split(u, n, b, N + 1, signed_split, sigma)
    au = ctypes.c_double(0.0)
    lib().orc_gamma_dagger_inplace(_pd(ga), lam, N, b, _pd(a), ctypes.byref(au))
    c = np.zeros(N + 1)
    c[:] = split(v, n, b, N + 1, signed_split, sigma)
    av = ctypes.c_double(0.0)
    lib().orc_gamma_dagger_inplace(_pd(ga), lam, N, b, _pd(c), ctypes.byref(av))
    w = np.ascontiguousarray(cyclic_convolve(a[:N].copy(), c[:N].copy()))
    h = np.empty(N + 1)
    lib().orc_delta_dagger(_pd(de), lam, N, b, _pd(w), au.value * av.value, _pd(h))
    nout = ((N + 1) * b + b + 128) // 64 + 4
    t, me, ma = _accumulate(h, b, b, nout)
    wv = _round_even_shift(t, 2 * b + sigma)
    if wv < 0 or wv > (1 << n):
        raise ConvolutionPrecisionFailure("high product left its admissible range")
    return Result(wv, me, ma)


def product(mode: str, u, v, n: int, b: int, N: int, lam: int = 0, signed_split: bool = True) -> Result:
    if mode == "full":
        return full_product(u, v, n, b, N, signed_split)
    if mode == "low":
        return low_product(u, v, n, b, N, lam, signed_split)
    return high_product(u, v, n, b, N, lam, signed_split)
