"""Exactness sweep over multi-pass plan shapes: for smooth lengths N with
distinct (C, A, B) factorisations, run a low (and full) product of random
operands on the GPU and compare with GMP.

    python tools/shape_sweep.py [max_cases]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def shape(L):
    C = next(c for c in range(4096, 15, -1) if c % 2 == 0 and L % c == 0)
    AB = L // C
    return C, AB


def smooth(lo, hi):
    out = []
    for a in range(2, 24):
        for b3 in range(0, 6):
            for c5 in range(0, 4):
                for d7 in range(0, 3):
                    N = 2**a * 3**b3 * 5**c5 * 7**d7
                    if lo <= N <= hi:
                        out.append(N)
    return sorted(out)


def main():
    maxc = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seen = set()
    cases = []
    for N in smooth(8193, 1 << 21):
        C, AB = shape(N)
        key = (C, AB if AB <= 2048 else -1, N % 9 == 0, N % 25 == 0, N % 49 == 0)
        if key in seen:
            continue
        seen.add(key)
        cases.append(N)
    cases = cases[:maxc]
    ctx = tm.Context(0)
    rng = np.random.default_rng(7)
    bad = 0
    for N in cases:
        for mode in (tm.Mode.LOW, tm.Mode.FULL):
            b = 12 if mode == tm.Mode.LOW else 16
            Nn = N if mode == tm.Mode.LOW else N // 2
            if mode == tm.Mode.FULL and N % 8:
                continue
            n = Nn * b - 5 if mode == tm.Mode.LOW else Nn * b - 3
            p = tm.manual_params(n, b, Nn, mode, tm.Backend.FFT, True)
            nl = (n + 63) // 64
            u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
            v = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
            try:
                r = ctx.product_limbs(mode, u, v, p)
                exp = port.oracle_low(u, v, n) if mode == tm.Mode.LOW else port.oracle_full(u, v)[:len(r)]
                ok = np.array_equal(r, exp)
                st = "ok" if ok else "WRONG"
            except tm.Error as e:
                ok = False
                st = f"{type(e).__name__}: {e}"
            s = ctx.last_stats
            C, AB = shape(s.transform_length) if s.transform_length else (0, 0)
            if not ok:
                bad += 1
            print(f"{mode.name:4s} N={Nn:8d} L={s.transform_length:8d} C={C:5d} AB={AB:6d} passes={s.passes} "
                  f"err={s.max_round_err:.4f} {st}", flush=True)
    print("bad", bad, "of", 2 * len(cases))


if __name__ == "__main__":
    main()
