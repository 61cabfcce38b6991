"""Host-side mirror of the reference's product API (products.hpp).

Reference interface (arxiv 1703.00640 artifact, /root/reference/proj/core):

    enum class Mode { kFull, kLow, kHigh, kOracleFallback }   products.hpp:14
    struct Params { n, b, N, lambda, p, mode, backend, signed_split }
                                                              products.hpp:25-34
    required_precision / default_lambda / validate_params / select_params
                                                              products.hpp:39-62
    full_product / low_product / high_product               products.hpp:91-93
    exceptions                                                errors.hpp

Operands may be Python ints or little-endian uint64 limb arrays; products
return Python ints (the reference returns BigInt).  ``*_limbs`` variants
return limb arrays.  Everything below ``Context`` runs on the GPU through
the C ABI; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from ._native import tmg_params, tmg_stats

# ---------------------------------------------------------------------------
# errors (errors.hpp:9-67)


class Error(RuntimeError):
    """Base class of all library errors."""


class InputOutOfRange(Error):
    pass


class NoValidParams(Error):
    pass


class UnsupportedLength(Error):
    pass


class ConvolutionPrecisionFailure(Error):
    pass


class PlanMismatch(Error):
    pass


class Unsupported(Error):
    """Parameter set the GPU path refuses (e.g. the EXACT backend)."""


class CudaError(Error):
    pass


_ERRORS = {
    _native.TMG_ERR_INPUT_OUT_OF_RANGE: InputOutOfRange,
    _native.TMG_ERR_NO_VALID_PARAMS: NoValidParams,
    _native.TMG_ERR_UNSUPPORTED_LENGTH: UnsupportedLength,
    _native.TMG_ERR_PRECISION_FAILURE: ConvolutionPrecisionFailure,
    _native.TMG_ERR_PLAN_MISMATCH: PlanMismatch,
    _native.TMG_ERR_UNSUPPORTED: Unsupported,
    _native.TMG_ERR_CUDA: CudaError,
    _native.TMG_ERR_INTERNAL: Error,
}


def _check(code: int) -> None:
    if code != _native.TMG_OK:
        raise _ERRORS.get(code, Error)(_native.last_error())


# ---------------------------------------------------------------------------
# parameters


class Mode(enum.IntEnum):
    FULL = 0
    LOW = 1
    HIGH = 2
    ORACLE_FALLBACK = 3


class Backend(enum.IntEnum):
    EXACT = 0
    FFT = 1


class Policy(enum.IntEnum):
    REFERENCE = 0  # params.cpp exactly (the default, as products.hpp:60-61)
    ACCURATE = 1   # opt-in: + FP64 error model and GPU cost ranking


DEFAULT_FALLBACK_CUTOFF = 4096  # products.hpp:37


@dataclass(frozen=True)
class Params:
    n: int = 0
    b: int = 0
    N: int = 0
    lam: int = 0
    p: int = 0
    mode: Mode = Mode.FULL
    backend: Backend = Backend.EXACT
    signed_split: bool = False

    def to_c(self) -> tmg_params:
        return tmg_params(self.n, self.b, self.N, self.lam, self.p, int(self.mode),
                          int(self.backend), 1 if self.signed_split else 0)

    @staticmethod
    def from_c(c: tmg_params) -> "Params":
        return Params(c.n, c.b, c.N, c.lam, c.p, Mode(c.mode), Backend(c.backend),
                      bool(c.signed_split))

    @property
    def transform_length(self) -> int:
        return 2 * self.N if self.mode == Mode.FULL else self.N


def required_precision(mode: Mode, b: int, N: int) -> int:
    out = ctypes.c_int32()
    _check(_native.load().tmg_required_precision(int(mode), b, N, ctypes.byref(out)))
    return out.value


def default_lambda(mode: Mode, backend: Backend, b: int, p: int) -> int:
    out = ctypes.c_int64()
    _check(_native.load().tmg_default_lambda(int(mode), int(backend), b, p, ctypes.byref(out)))
    return out.value


def validate_params(params: Params) -> None:
    c = params.to_c()
    _check(_native.load().tmg_validate_params(ctypes.byref(c)))


def select_params(n: int, mode: Mode, backend: Backend = Backend.FFT,
                  fallback_cutoff: int = DEFAULT_FALLBACK_CUTOFF,
                  policy: Policy = Policy.REFERENCE) -> Params:
    out = tmg_params()
    _check(_native.load().tmg_select_params(n, int(mode), int(backend), fallback_cutoff,
                                            int(policy), ctypes.byref(out)))
    return Params.from_c(out)


def predicted_sigma(params: Params) -> float:
    c = params.to_c()
    return float(_native.load().tmg_predicted_sigma(ctypes.byref(c)))


def output_limbs(mode: Mode, n: int) -> int:
    return int(_native.load().tmg_output_limbs(int(mode), n))


def manual_params(n: int, b: int, N: int, mode: Mode, backend: Backend = Backend.FFT,
                  signed_split: bool = True, lam: int | None = None) -> Params:
    """Explicit parameter set (the reference CLI's --b/--N/--lambda overrides,
    truncmul_cli.cpp:82-97)."""
    p = required_precision(mode, b, N)
    if lam is None:
        lam = default_lambda(mode, backend, b, p) if mode != Mode.FULL else 0
    return Params(n, b, N, lam, p, mode, backend, signed_split)


# ---------------------------------------------------------------------------
# operands


def to_limbs(x, n: int) -> np.ndarray:
    """Little-endian uint64 limbs of x, exactly ceil(n/64) of them.  Raises
    InputOutOfRange outside [0, 2^n) (split.cpp:13-20)."""
    nl = (n + 63) // 64
    if isinstance(x, np.ndarray):
        a = np.ascontiguousarray(x, dtype=np.uint64)
        if len(a) > nl:
            if np.any(a[nl:]):
                raise InputOutOfRange("split: operand outside [0, 2^n)")
            a = a[:nl]
        elif len(a) < nl:
            a = np.concatenate([a, np.zeros(nl - len(a), dtype=np.uint64)])
        if n % 64 and nl and (int(a[-1]) >> (n % 64)):
            raise InputOutOfRange("split: operand outside [0, 2^n)")
        return np.ascontiguousarray(a)
    x = int(x)
    if x < 0 or x.bit_length() > n:
        raise InputOutOfRange("split: operand outside [0, 2^n)")
    return np.frombuffer(x.to_bytes(nl * 8, "little"), dtype=np.uint64).copy()


def from_limbs(a: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(a, dtype=np.uint64).tobytes(), "little")


# ---------------------------------------------------------------------------
# context


@dataclass
class Stats:
    max_round_err: float = 0.0
    max_abs: float = 0.0
    flags: int = 0
    transform_length: int = 0
    passes: int = 0
    kernels: int = 0
    attempts: int = 0
    b: int = 0
    N: int = 0
    first_round_err: float = 0.0

    @property
    def escalated(self) -> bool:
        return bool(self.flags & _native.TMG_STAT_ESCALATED)


class Context:
    """One CUDA device, one stream, cached plans and workspaces."""

    def __init__(self, device: int = 0, escalation: int = 0):
        self._lib = _native.load()
        h = ctypes.c_void_p()
        _check(self._lib.tmg_context_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device
        self.last_stats = Stats()
        if escalation:
            self.set_escalation(escalation)

    def set_escalation(self, max_escalations: int) -> None:
        """Recompute a refused single product at b - 1 (up to n times);
        0 keeps the reference behaviour (raise ConvolutionPrecisionFailure)."""
        _check(self._lib.tmg_context_set_escalation(self._h, int(max_escalations)))

    def set_option(self, option: int, value: int = 1) -> None:
        """Testing and diagnostics: select an alternative code path
        (_native.TMG_OPT_*; include/truncmul_b200.h lists them)."""
        _check(self._lib.tmg_context_set_option(self._h, int(option), int(value)))

    def close(self) -> None:
        if self._h:
            self._lib.tmg_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int) -> None:
        _check(self._lib.tmg_context_set_stream(self._h, ctypes.c_void_p(stream_ptr)))

    def synchronize(self) -> None:
        _check(self._lib.tmg_synchronize(self._h))

    def _stats(self, s: tmg_stats) -> Stats:
        self.last_stats = Stats(s.max_round_err, s.max_abs, s.flags, s.transform_length,
                                s.passes, s.kernels, s.attempts, s.b, s.N, s.first_round_err)
        return self.last_stats

    def product_limbs(self, mode: Mode, u, v, params: Params) -> np.ndarray:
        fn = {Mode.FULL: self._lib.tmg_full_product, Mode.LOW: self._lib.tmg_low_product,
              Mode.HIGH: self._lib.tmg_high_product}[Mode(mode)]
        ul = to_limbs(u, params.n)
        vl = to_limbs(v, params.n)
        out = np.zeros(max(1, output_limbs(mode, params.n)), dtype=np.uint64)
        c = params.to_c()
        st = tmg_stats()
        P64 = ctypes.POINTER(ctypes.c_uint64)
        rc = fn(self._h, ctypes.byref(c), ul.ctypes.data_as(P64), vl.ctypes.data_as(P64),
                out.ctypes.data_as(P64), ctypes.byref(st))
        self._stats(st)  # filled before a precision failure is reported too
        _check(rc)
        return out

    def product_batched(self, params: Params, u: np.ndarray, v: np.ndarray,
                        return_flags: bool = False):
        """count x ceil(n/64) operand arrays -> count x output_limbs results."""
        nl = (params.n + 63) // 64
        u = np.ascontiguousarray(u, dtype=np.uint64).reshape(-1, nl)
        v = np.ascontiguousarray(v, dtype=np.uint64).reshape(-1, nl)
        count = u.shape[0]
        mode = Mode.FULL if params.mode == Mode.ORACLE_FALLBACK else params.mode
        ol = output_limbs(mode, params.n)
        out = np.zeros((count, ol), dtype=np.uint64)
        flags = np.zeros(count, dtype=np.uint32)
        c = params.to_c()
        st = tmg_stats()
        P64 = ctypes.POINTER(ctypes.c_uint64)
        _check(self._lib.tmg_product_batched(
            self._h, ctypes.byref(c), u.ctypes.data_as(P64), v.ctypes.data_as(P64), count,
            out.ctypes.data_as(P64), flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
            ctypes.byref(st)))
        self._stats(st)
        return (out, flags) if return_flags else out

    def cyclic_convolve_f64(self, f, g) -> np.ndarray:
        """out[k] = sum_j f[j] g[(k - j) mod n] in FP64 (cyclic_convolve_f64 on an
        FFT plan, convolution.hpp:64-67).  n must be {2,3,5,7}-smooth
        (UnsupportedLength otherwise, like make_plan)."""
        fa = np.ascontiguousarray(f, dtype=np.float64)
        ga = np.ascontiguousarray(g, dtype=np.float64)
        if fa.ndim != 1 or fa.shape != ga.shape:
            raise PlanMismatch("cyclic_convolve_f64: operands must be two sequences of one length")
        out = np.empty(len(fa), dtype=np.float64)
        PD = ctypes.POINTER(ctypes.c_double)
        _check(self._lib.tmg_cyclic_convolve_f64(self._h, len(fa), fa.ctypes.data_as(PD),
                                                 ga.ctypes.data_as(PD), out.ctypes.data_as(PD)))
        return out

    def _map(self, name: str, N: int, b: int, lam: int, x, nin: int, nout: int, aux=None):
        xa = np.ascontiguousarray(x, dtype=np.float64)
        if xa.ndim != 1 or len(xa) != nin:
            raise PlanMismatch(f"{name}: the input must hold {nin} doubles")
        out = np.empty(nout, dtype=np.float64)
        PD = ctypes.POINTER(ctypes.c_double)
        fn = getattr(self._lib, "tmg_" + name)
        if name == "gamma_dagger_f64":
            au = ctypes.c_double(0.0)
            _check(fn(self._h, N, b, lam, xa.ctypes.data_as(PD), out.ctypes.data_as(PD), ctypes.byref(au)))
            return out, float(au.value)
        if name == "delta_dagger_f64":
            _check(fn(self._h, N, b, lam, xa.ctypes.data_as(PD), float(aux), out.ctypes.data_as(PD)))
            return out
        _check(fn(self._h, N, b, lam, xa.ctypes.data_as(PD), out.ctypes.data_as(PD)))
        return out

    def alpha_star_f64(self, N: int, b: int, lam: int, x) -> np.ndarray:
        """alpha* of the low product's pre-map (maps_f64.hpp alpha_star_f64): N -> N."""
        return self._map("alpha_star_f64", N, b, lam, x, N, N)

    def beta_star_f64(self, N: int, b: int, lam: int, w) -> np.ndarray:
        """beta* of the low product's post-map (beta_star_f64): N -> N."""
        return self._map("beta_star_f64", N, b, lam, w, N, N)

    def gamma_dagger_f64(self, N: int, b: int, lam: int, x):
        """gamma-dagger of the high product's pre-map (gamma_dagger_f64): N + 1
        chunks -> (N values, the root channel aux)."""
        return self._map("gamma_dagger_f64", N, b, lam, x, N + 1, N)

    def delta_dagger_f64(self, N: int, b: int, lam: int, w, aux: float) -> np.ndarray:
        """delta-dagger of the high product's post-map (delta_dagger_f64): N
        convolution values and aux = theta_u theta_v -> N + 1 values."""
        return self._map("delta_dagger_f64", N, b, lam, w, N, N + 1, aux)

    def split_i64(self, u, params: Params, high: bool = False) -> np.ndarray:
        """The chunks of one operand as int64 words (split_low_i64 /
        split_high_i64, products.hpp:77-79): N of them, or the N + 1 chunks
        of the top-aligned u 2^sigma.  u: exactly ceil(n/64) limbs; the range
        check u < 2^n runs on the device."""
        ul = np.ascontiguousarray(u, dtype=np.uint64)
        if params.n >= 1 and len(ul) != (params.n + 63) // 64:
            raise InputOutOfRange("operands must hold ceil(n/64) limbs")
        count = params.N + 1 if high else params.N
        out = np.zeros(max(count, 0), dtype=np.int64)
        c = params.to_c()
        fn = self._lib.tmg_split_high_i64 if high else self._lib.tmg_split_low_i64
        _check(fn(self._h, ctypes.byref(c), ul.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return out

    def product_device(self, params: Params, d_u: int, d_v: int, d_out: int, count: int = 1):
        """Enqueue on device pointers (ints); no synchronisation."""
        c = params.to_c()
        _check(self._lib.tmg_product_device(self._h, ctypes.byref(c), ctypes.c_void_p(d_u),
                                            ctypes.c_void_p(d_v), ctypes.c_void_p(d_out), count))

    def check(self) -> Stats:
        st = tmg_stats()
        _check(self._lib.tmg_check(self._h, ctypes.byref(st)))
        return self._stats(st)

    def last_kernel_count(self) -> int:
        return int(self._lib.tmg_last_kernel_count(self._h))

    def profile(self, on: bool = True) -> None:
        """Bracket every kernel launch with CUDA events on the context stream."""
        _check(self._lib.tmg_profile_enable(self._h, 1 if on else 0))

    def profile_read(self, max_records: int = 4096) -> list[tuple[str, float, float]]:
        """[(kernel name, milliseconds, algorithmic bytes)] since the last read."""
        stride = 32
        names = ctypes.create_string_buffer(stride * max_records)
        ms = (ctypes.c_double * max_records)()
        by = (ctypes.c_double * max_records)()
        cnt = ctypes.c_int(0)
        _check(self._lib.tmg_profile_read(self._h, names, stride, ms, by, max_records,
                                          ctypes.byref(cnt)))
        out = []
        for i in range(cnt.value):
            nm = names.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode()
            out.append((nm, ms[i], by[i]))
        return out


_default: dict[int, Context] = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


# ---------------------------------------------------------------------------
# products (products.hpp:81-93)


def _run(mode: Mode, u, v, params: Params, ctx: Context | None) -> np.ndarray:
    if params.mode != Mode.ORACLE_FALLBACK and params.mode != mode:
        raise InputOutOfRange(f"{mode.name.lower()}_product: params were built for a different mode")
    return (ctx or default_context()).product_limbs(mode, u, v, params)


def full_product_limbs(u, v, params: Params, ctx: Context | None = None) -> np.ndarray:
    return _run(Mode.FULL, u, v, params, ctx)


def low_product_limbs(u, v, params: Params, ctx: Context | None = None) -> np.ndarray:
    return _run(Mode.LOW, u, v, params, ctx)


def high_product_limbs(u, v, params: Params, ctx: Context | None = None) -> np.ndarray:
    return _run(Mode.HIGH, u, v, params, ctx)


def full_product(u, v, params: Params, ctx: Context | None = None) -> int:
    """u v exactly (Alg. 1, products.hpp:91)."""
    return from_limbs(full_product_limbs(u, v, params, ctx))


def low_product(u, v, params: Params, ctx: Context | None = None) -> int:
    """u v mod 2^n (Alg. 2, products.hpp:92)."""
    return from_limbs(low_product_limbs(u, v, params, ctx))


def high_product(u, v, params: Params, ctx: Context | None = None) -> int:
    """w with |u v - 2^n w| < 2^n, 0 <= w <= 2^n (Alg. 3, products.hpp:93)."""
    return from_limbs(high_product_limbs(u, v, params, ctx))


def cyclic_convolve_f64(f, g, ctx: Context | None = None) -> np.ndarray:
    """FP64 cyclic convolution of two equally long sequences
    (convolution.hpp:64-67)."""
    return (ctx or default_context()).cyclic_convolve_f64(f, g)


def split_low_i64(u, params: Params, ctx: Context | None = None) -> np.ndarray:
    """u = sum_i chunk_i 2^{i b}, N chunks (products.hpp:77; balanced below the
    top chunk when params.signed_split)."""
    if params.n < 1:
        raise InputOutOfRange("split: bit length must be positive")
    return (ctx or default_context()).split_i64(to_limbs(u, params.n), params, high=False)


def split_high_i64(u, params: Params, ctx: Context | None = None) -> np.ndarray:
    """The N + 1 chunks of u 2^sigma, sigma = (N + 1) b - n (products.hpp:78-79)."""
    if params.n < 1:
        raise InputOutOfRange("split: bit length must be positive")
    return (ctx or default_context()).split_i64(to_limbs(u, params.n), params, high=True)


def multiply(mode: Mode, u, v, n: int | None = None, backend: Backend = Backend.FFT,
             policy: Policy = Policy.REFERENCE, ctx: Context | None = None) -> int:
    """Convenience: select parameters like the reference CLI (truncmul_cli.cpp:
    99-150: n defaults to the longer operand, the oracle fallback below the
    cutoff) and run the product."""
    if n is None:
        n = max(1, int(u).bit_length(), int(v).bit_length())
    params = select_params(n, mode, backend, DEFAULT_FALLBACK_CUTOFF, policy)
    return from_limbs(_run(mode, u, v, params, ctx))
