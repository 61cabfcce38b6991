"""Stand-alone cyclic convolution at the products' transform lengths: kernel
times (the library's CUDA-event profiler on the context stream) against the
algorithmic bytes of each pass.   python tools/conv_bench.py [L ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402

PEAK = 6553.3  # GB/s, MEASURED_PEAKS.json
ctx = tm.default_context(0)
rng = np.random.default_rng(1)
for L in [int(a) for a in sys.argv[1:]] or [81920, 1310720, 5898240, 7077888, 22937600]:
    f = rng.integers(-2048, 2049, L).astype(np.float64)
    g = rng.integers(-2048, 2049, L).astype(np.float64)
    for _ in range(2):
        ctx.cyclic_convolve_f64(f, g)
    ctx.profile(True)
    reps = 5
    for _ in range(reps):
        ctx.cyclic_convolve_f64(f, g)
    recs = ctx.profile_read()
    ctx.profile(False)
    names = []
    for r in recs:
        if r[0] not in names:
            names.append(r[0])
    tot_ms, tot_b = 0.0, 0.0
    parts = []
    for nm in names:
        ms = float(np.median([r[1] for r in recs if r[0] == nm]))
        by = [r[2] for r in recs if r[0] == nm][0]
        tot_ms += ms
        tot_b += by
        parts.append(f"{nm.split(':')[-1]} {ms * 1e3:.1f} us ({by / ms / 1e6:.0f} GB/s)")
    print(f"L={L}: {tot_ms * 1e3:.1f} us, {tot_b / tot_ms / 1e6:.0f} GB/s algorithmic "
          f"({tot_b / tot_ms / 1e6 / PEAK:.2f} of the copy peak): " + ", ".join(parts), flush=True)
