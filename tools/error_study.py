"""FP64 error of the reference pipeline (oracle port: pocketfft standing in
for FFTW, the reference's maps in C) at the reference's and the accurate
policy's chunk widths, on uniform random operands.

    python tools/error_study.py [log2n ...]

Prints, per (n, mode, policy): b, N, lambda, the predicted sigma of the
accurate policy's model (params.cpp) and the measured max pre-rounding
residual over a few seeds.  A residual above 0.25 is the reference's own
tripwire (products_f64.cpp:16-27).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def main():
    lgs = [int(a) for a in sys.argv[1:]] or [20, 22, 24]
    seeds = 2
    print("| n | mode | policy | b | N | lambda | predicted sigma | max residual (seeds) |")
    print("|---|---|---|---|---|---|---|---|")
    for lg in lgs:
        n = 1 << lg
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            for pol in (tm.Policy.REFERENCE, tm.Policy.ACCURATE):
                p = tm.select_params(n, mode, policy=pol)
                errs = []
                for s in range(seeds):
                    u, v = port.config_operands(100 + s, n // 64)
                    try:
                        errs.append(f"{port.product(mode.name.lower(), u, v, n, p.b, p.N, p.lam).max_err:.3f}")
                    except port.ConvolutionPrecisionFailure:
                        errs.append("TRIP")
                print(f"| 2^{lg} | {mode.name.lower()} | {pol.name.lower()} | {p.b} | {p.N} | {p.lam} | "
                      f"{tm.predicted_sigma(p):.4f} | {', '.join(errs)} |", flush=True)


if __name__ == "__main__":
    main()
