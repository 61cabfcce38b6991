import sys; sys.path.insert(0,'.')
import numpy as np, paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import _native
ctx = tm.Context(0); ctx.set_option(_native.TMG_OPT_DEBUG_SYNC, 1)
rng = np.random.default_rng(1)
for n in (8192, 1 << 17):
    u = rng.integers(0, 2**64, n//64, dtype=np.uint64); v = rng.integers(0, 2**64, n//64, dtype=np.uint64)
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        try:
            ctx.product_limbs(mode, u, v, tm.select_params(n, mode)); print("ok", n, mode, flush=True)
        except Exception as e:
            print("FAIL", n, mode, e, flush=True); sys.exit(0)
p = tm.manual_params(3840, 30, 128, tm.Mode.LOW, tm.Backend.FFT, signed_split=False, lam=4)
top = (1 << 3840) - 1
try:
    tm.low_product(top, top, p, ctx); print("b30 no trip?")
except Exception as e:
    print("b30:", type(e).__name__, e, flush=True)
