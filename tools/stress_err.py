"""Max pre-rounding error of the GPU pipeline on the BASELINE config-5
stress operands (all ones / alternating limbs), next to the oracle port's.

    python tools/stress_err.py [log2n ...] [--port]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def operands(pattern, nl):
    if pattern == "ones":
        return np.full(nl, np.uint64(0xFFFFFFFFFFFFFFFF))
    u = np.zeros(nl, dtype=np.uint64)
    u[0::2] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return u


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    do_port = "--port" in sys.argv
    ctx = tm.Context(0)
    for lg in map(int, args or ["28"]):
        n = 1 << lg
        for pattern in ("ones", "alternating"):
            u = operands(pattern, n // 64)
            for mode in (tm.Mode.LOW, tm.Mode.HIGH, tm.Mode.FULL):
                p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
                t = time.time()
                try:
                    ctx.product_limbs(mode, u, u, p)
                    ok = "ok"
                except tm.ConvolutionPrecisionFailure:
                    ok = "TRIP"
                s = ctx.last_stats
                line = (f"n=2^{lg} {pattern:11s} {mode.name:4s} b={p.b} N={p.N} lam={p.lam} "
                        f"L={s.transform_length} passes={s.passes} gpu_err={s.max_round_err:.4f} "
                        f"maxabs=2^{np.log2(max(s.max_abs, 1)):.2f} {ok} ({time.time() - t:.1f}s)")
                if do_port:
                    # the reference's scaling order (1/n on the spectrum) and
                    # pocketfft's normalised irfft (1/n on the outputs)
                    for sa in ("spectrum", "end"):
                        port.SCALE_AT = sa
                        try:
                            r = port.product(mode.name.lower(), u, u, n, p.b, p.N, p.lam)
                            line += f" port[{sa}]={r.max_err:.4f}"
                        except port.ConvolutionPrecisionFailure:
                            line += f" port[{sa}]=TRIP"
                print(line, flush=True)


if __name__ == "__main__":
    main()
