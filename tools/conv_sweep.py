"""Exactness sweep of tmg_cyclic_convolve_f64 over {2,3,5,7}-smooth lengths:
every smooth multiple of 4 in (4096, LIMIT] (or a random sample of COUNT of
them) plus smooth lengths below, integer operands, rounded result against the
oracle's convolution, residual < 0.25.  Lengths the GPU plans refuse must be
refused with UnsupportedLength.

    python tools/conv_sweep.py [limit] [count] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402

limit = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 400
rng = np.random.default_rng(int(sys.argv[3]) if len(sys.argv) > 3 else 11)
smooth = []
p2 = 1
while p2 <= limit:
    p3 = p2
    while p3 <= limit:
        p5 = p3
        while p5 <= limit:
            p7 = p5
            while p7 <= limit:
                smooth.append(p7)
                p7 *= 7
            p5 *= 5
        p3 *= 3
    p2 *= 2
smooth = sorted(smooth)
big = [n for n in smooth if n > 4096 and n % 4 == 0]
small = [n for n in smooth if n <= 4096 or (n % 4 and n <= 32768)]
pick = sorted(set(rng.choice(big, min(count, len(big)), replace=False).tolist() +
                  rng.choice(small, min(count // 4, len(small)), replace=False).tolist()))
ctx = tm.default_context(0)
bad = refused = 0
for i, n in enumerate(pick):
    f = rng.integers(-2048, 2049, n).astype(np.float64)
    g = rng.integers(-2048, 2049, n).astype(np.float64)
    try:
        out = ctx.cyclic_convolve_f64(f, g)
    except tm.UnsupportedLength as e:
        refused += 1
        print("refused", n, e, flush=True)
        continue
    r = np.rint(out)
    ok = np.array_equal(r, np.rint(port.cyclic_convolve(f, g))) and np.max(np.abs(out - r)) < 0.25
    if not ok:
        bad += 1
        print("BAD", n, flush=True)
    if i % 50 == 0:
        print(f"{i}: n={n} ok={ok} kernels={ctx.last_kernel_count()}", flush=True)
print(f"lengths {len(pick)} bad {bad} refused {refused}")
sys.exit(1 if bad else 0)
