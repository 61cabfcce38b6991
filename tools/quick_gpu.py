import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import __graft_entry__ as g
g.build()
import paper_1703_00640_b200 as tm
from oracle import port
ctx = tm.default_context(0)
rng = np.random.default_rng(1)
for n in [int(x) for x in (sys.argv[1:] or ["8192", "5001", "65536", "262144", "1000000", "4194304"])]:
    nl = (n + 63)//64
    u = rng.integers(0, 2**64, nl, dtype=np.uint64); v = rng.integers(0, 2**64, nl, dtype=np.uint64)
    if n % 64:
        u[-1] &= np.uint64((1 << (n % 64)) - 1); v[-1] &= np.uint64((1 << (n % 64)) - 1)
    P = port.limbs_to_int(port.oracle_full(u, v))
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
        try:
            t0 = time.time()
            r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
            dt = time.time() - t0
            if mode == tm.Mode.FULL: ok = r == P
            elif mode == tm.Mode.LOW: ok = r == (P & ((1 << n) - 1))
            else: ok = port.is_valid_high(u, v, n, r)
            s = ctx.last_stats
            print(f"n={n} {mode.name} b={p.b} N={p.N} L={s.transform_length} passes={s.passes} ok={ok} err={s.max_round_err:.4f} t={dt*1e3:.2f}ms", flush=True)
        except Exception as e:
            print(f"n={n} {mode.name} EXC {type(e).__name__}: {e}", flush=True)
