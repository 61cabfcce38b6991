"""Exactness at random large sizes (n in [2^24.5, 2^27.2], where the split
and carry by runs are the default): full and low products bit-exact against
GMP, high products within the bound, both parameter policies (a refusal by
the tripwire is reported, not an error: the reference's b trips at 2^26).

    python tools/large_sizes.py [count] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 10
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 9)
ctx = tm.default_context(0)
bad = refused = 0
for i in range(count):
    n = int(2 ** rng.uniform(24.5, 27.2))
    if i % 3 == 0:
        n |= 1  # odd sizes
    nl = (n + 63) // 64
    kind = int(rng.integers(0, 3))
    if kind == 0:
        u = int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1)
        v = int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1)
    elif kind == 1:
        u = (1 << n) - 1
        v = int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1)
    else:
        u = (1 << n) - 1 - (1 << (n // 3))
        v = (1 << (n - 1)) + 12345
    ul, vl = port.int_to_limbs(u, nl), port.int_to_limbs(v, nl)
    P = u * v
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        for pol in (tm.Policy.ACCURATE, tm.Policy.REFERENCE):
            p = tm.select_params(n, mode, policy=pol)
            try:
                r = tm.from_limbs(ctx.product_limbs(mode, ul, vl, p))
            except tm.ConvolutionPrecisionFailure:
                refused += 1
                continue
            if mode == tm.Mode.FULL:
                ok = r == P
            elif mode == tm.Mode.LOW:
                ok = r == P & ((1 << n) - 1)
            else:
                ok = abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)
            if not ok:
                bad += 1
                print("BAD", n, kind, mode.name, pol.name, p, flush=True)
    print(f"{i}: n={n} kind={kind} bad {bad} refused {refused}", flush=True)
print(f"bad {bad} refused {refused}")
sys.exit(1 if bad else 0)
