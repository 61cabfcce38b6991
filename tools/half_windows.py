"""Worst case of the split's carry walk: operands whose every b-bit window
equals 2^{b-1} (each carry-in is decided only at chunk 0).  Times one low
product per size and checks it against GMP.
    python tools/half_windows.py [log2n ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402

ctx = tm.default_context(0)
for lg in [int(a) for a in sys.argv[1:]] or [20, 22, 24]:
    n = 1 << lg
    for mode in (tm.Mode.LOW, tm.Mode.FULL):
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
        b = p.b
        x = 0
        N = n // b
        x = ((1 << (b * N)) - 1) // ((1 << b) - 1) << (b - 1)  # sum_i 2^{i b + b - 1}
        u = tm.to_limbs(x & ((1 << n) - 1), n)
        rng = np.random.default_rng(lg)
        v = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
        for rep in range(2):
            t0 = time.time()
            try:
                r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
                tag = "ok"
            except tm.ConvolutionPrecisionFailure:
                r, tag = None, "refused"
            dt = time.time() - t0
        if r is not None:
            P = port.limbs_to_int(port.oracle_full(u, v))
            good = r == (P if mode == tm.Mode.FULL else P & ((1 << n) - 1))
            tag = "exact" if good else "WRONG"
        t0 = time.time()
        w = ctx.split_i64(u, p)
        ds = time.time() - t0
        print(f"2^{lg} {mode.name} b={b}: product {dt * 1e3:.1f} ms (host call) {tag}; "
              f"split_i64 {ds * 1e3:.1f} ms, chunks all 2^(b-1): {bool(np.all(w[:N - 1] == (1 << (b - 1))))}",
              flush=True)
