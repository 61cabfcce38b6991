"""k_split_i64 at product sizes: kernel time (CUDA events on the context
stream, the library's profiler) against its algorithmic bytes (n / 8 read,
8 per chunk written).   python tools/split_bench.py [log2n ...]"""
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402

PEAK = 6553.3  # GB/s, MEASURED_PEAKS.json
ctx = tm.default_context(0)
rng = np.random.default_rng(1)
for lg in [int(a) for a in sys.argv[1:]] or [20, 24, 26, 28]:
    n = 1 << lg
    u = rng.integers(0, 2**64, n // 64, dtype=np.uint64)
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
        high = mode == tm.Mode.HIGH
        for _ in range(2):
            ctx.split_i64(u, p, high=high)
        ctx.profile(True)
        for _ in range(10):
            ctx.split_i64(u, p, high=high)
        recs = [r for r in ctx.profile_read() if r[0].endswith("k_split_i64")]
        ctx.profile(False)
        ms = float(np.median([r[1] for r in recs]))
        gbs = recs[0][2] / ms / 1e6
        print(f"2^{lg} {mode.name:4s} b={p.b} chunks={p.N + (1 if high else 0)}: {ms * 1e3:.1f} us, "
              f"{gbs:.0f} GB/s, {gbs / PEAK:.2f} of the HBM copy peak")
