import sys; sys.path.insert(0,'.')
import numpy as np, paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import _native
from oracle import port
ns = [int(x) for x in sys.argv[1:]] or [4748529]
for n in ns:
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        ctx = tm.Context(0); ctx.set_option(_native.TMG_OPT_DEBUG_SYNC, 1)
        rng = np.random.default_rng(1); nl = (n + 63)//64
        u = rng.integers(0, 2**64, nl, dtype=np.uint64); v = rng.integers(0, 2**64, nl, dtype=np.uint64)
        if n % 64: u[-1] &= np.uint64((1 << (n % 64)) - 1); v[-1] &= np.uint64((1 << (n % 64)) - 1)
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
        try:
            r = ctx.product_limbs(mode, u, v, p); print("ok", n, mode, ctx.last_stats.transform_length, flush=True)
        except Exception as e:
            print("FAIL", n, mode, e, flush=True); sys.exit(0)
