"""Where does the pipeline's rounding error come from?  Runs one product on
the GPU, reads back its pre-mapped input z and convolution output w
(tmg_debug_read), computes the exact cyclic convolution of the same z with
GMP (Kronecker substitution), and splits the final error into the FFT part
and the post-map part, next to numpy's FFT on the same z.

    python tools/conv_err.py low 22 alternating
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from paper_1703_00640_b200 import _native  # noqa: E402
from oracle import port  # noqa: E402

F = 60          # input grid 2^-F
S = 192         # Kronecker slot bits


def exact_cyclic(a, c):
    """Exact cyclic convolution of two float64 vectors rounded to 2^-F,
    returned as Python ints scaled by 2^(2F)."""
    N = len(a)
    M = 1 << 84
    ai = [int(x * 2.0**F) + M for x in a.tolist()]
    ci = [int(x * 2.0**F) + M for x in c.tolist()]
    sb = S // 8

    def pack(v):
        buf = b"".join(x.to_bytes(sb, "little") for x in v)
        buf += b"\0" * (-len(buf) % 8)
        return np.frombuffer(buf, dtype=np.uint64).copy()

    P = port.gmp_mul(pack(ai), pack(ci)).tobytes()
    slots = [int.from_bytes(P[i * sb:(i + 1) * sb], "little") for i in range(2 * N)]
    const = M * sum(ci) + M * sum(ai) - N * M * M  # cross terms of the offsets
    # sum_j (a_j+M)(c_j+M) = conv + M*sum(c) + M*sum(a) + N M^2; sum(ai) includes N*M
    out = [slots[k] + slots[k + N] - const for k in range(N)]
    return out


def main():
    mode = tm.Mode[sys.argv[1].upper()]
    lg = int(sys.argv[2])
    pattern = sys.argv[3] if len(sys.argv) > 3 else "alternating"
    n = 1 << lg
    nl = n // 64
    if pattern == "ones":
        u = np.full(nl, np.uint64(0xFFFFFFFFFFFFFFFF))
        v = u
    elif pattern == "alternating":
        u = np.zeros(nl, dtype=np.uint64)
        u[0::2] = np.uint64(0xFFFFFFFFFFFFFFFF)
        v = u
    else:
        u, v = port.config_operands(int(pattern), nl)
    p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
    if len(sys.argv) > 4:  # manual N (and lambda from the reference rule)
        Nm = int(sys.argv[4])
        p = tm.manual_params(n, p.b, Nm, mode, tm.Backend.FFT, True)
    ctx = tm.Context(0)
    ctx.set_option(_native.TMG_OPT_Z_NATURAL, 1)  # z read back in natural order
    try:
        ctx.product_limbs(mode, u, v, p)
        st = "ok"
    except tm.ConvolutionPrecisionFailure:
        st = "TRIP"
    s = ctx.last_stats
    print(f"{mode.name} 2^{lg} {pattern}: b={p.b} N={p.N} lam={p.lam} L={s.transform_length} "
          f"gpu max_err={s.max_round_err:.4f} {st}")
    N = p.N
    lib = _native.load()
    z = np.zeros(2 * N, dtype=np.float64)
    nb = ctypes.c_size_t(z.nbytes)
    lib.tmg_debug_read(ctx.handle, 0, z.ctypes.data, ctypes.byref(nb))
    L = s.transform_length
    w = np.zeros(L, dtype=np.float64)
    nb = ctypes.c_size_t(w.nbytes)
    lib.tmg_debug_read(ctx.handle, 1, w.ctypes.data, ctypes.byref(nb))
    a, c = z[0::2].copy(), z[1::2].copy()
    if mode == tm.Mode.FULL:
        a, c = np.concatenate([a, np.zeros(L - N)]), np.concatenate([c, np.zeros(L - N)])
    ex = exact_cyclic(a, c)
    exf = np.array([float(x) for x in ex]) / 2.0 ** (2 * F)
    scale = 2.0 ** p.b if mode == tm.Mode.LOW else 1.0
    eg = (w - exf)
    en = (port.cyclic_convolve(a, c) - exf)
    mx = np.abs(exf).max()
    ulp = np.spacing(mx)
    print(f"  max|w| = 2^{np.log2(mx):.2f} ulp={ulp:.3g}")
    for name, e in (("gpu fft", eg), ("numpy fft", en)):
        print(f"  {name:10s} max|err| = {np.abs(e).max():.4g} ({np.abs(e).max() / ulp:.2f} ulp of max, "
              f"x2^b {np.abs(e).max() * scale:.4f})  rms {np.sqrt((e ** 2).mean()) / ulp:.3f} ulp  "
              f"mean {e.mean() / ulp:+.4f} ulp")
    # a global scale bias shows up as e ~ slope * w
    for name, e in (("gpu fft", eg), ("numpy fft", en)):
        slope = float((e * exf).sum() / (exf * exf).sum())
        res = e - slope * exf
        print(f"  {name:10s} scale bias {slope / 2.0**-53:+.3f} x 2^-53; after removing it max "
              f"{np.abs(res).max() / ulp:.2f} ulp rms {np.sqrt((res ** 2).mean()) / ulp:.3f} ulp")
    # where are the worst errors
    idx = np.argsort(-np.abs(eg))[:8]
    print("  worst gpu k:", idx.tolist(), (eg[idx] / ulp).round(2).tolist())
    # does the error correlate with k (bias)?
    if mode == tm.Mode.LOW:
        be = port.coeff_table("beta", p.lam, N, p.b)
        for name, ww in (("exact conv", exf), ("gpu conv", w), ("numpy conv", exf + en)):
            low = np.empty(N)
            port.lib().orc_beta_star(port._pd(be), p.lam, N, p.b, port._pd(np.ascontiguousarray(ww)),
                                     port._pd(low))
            x = low * 2.0 ** p.b
            r = np.abs(x - np.round(x)).max()
            print(f"  oracle post-map of {name:10s}: max rounding residual {r:.4f}")


if __name__ == "__main__":
    main()
