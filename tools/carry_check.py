"""Runs kernel (TMG_OPT_CARRY_KERNELS = 3) against GMP and against the lanes
kernel (= 2): products and residuals, random and structured operands.
python tools/carry_check.py [count] [seed]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from paper_1703_00640_b200 import _native  # noqa: E402
from oracle import port  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
c3 = tm.Context(0); c3.set_option(_native.TMG_OPT_CARRY_KERNELS, 3)
c2 = tm.Context(0); c2.set_option(_native.TMG_OPT_CARRY_KERNELS, 2)
cg = tm.Context(0); cg.set_option(_native.TMG_OPT_CARRY_KERNELS, 4); cg.set_option(_native.TMG_OPT_GENERIC_RUNS, 1)
c4 = tm.Context(0); c4.set_option(_native.TMG_OPT_CARRY_KERNELS, 4)
bad = 0
def operands(n, kind):
    nl = (n + 63) // 64
    if kind == 0:
        u = int.from_bytes(rng.bytes(nl * 8), "little"); v = int.from_bytes(rng.bytes(nl * 8), "little")
    elif kind == 1:
        u = (1 << n) - 1; v = (1 << n) - 1
    elif kind == 2:
        u = (1 << n) - 1; v = 1
    elif kind == 3:
        u = 1 << (n - 1); v = (1 << n) - 1
    else:
        u = int.from_bytes(rng.bytes(nl * 8), "little"); v = 0
    m = (1 << n) - 1
    return port.int_to_limbs(u & m, nl), port.int_to_limbs(v & m, nl)
sizes = [1 << 19, (1 << 20) + 77, 3_000_001, 1 << 22, 4748529, (1 << 23) + 12345]
for i in range(count):
    n = sizes[i] if i < len(sizes) else int(np.exp(rng.uniform(np.log(1 << 17), np.log(1 << 24))))
    kind = 0 if i < len(sizes) else int(rng.integers(0, 5))
    u, v = operands(n, kind)
    P = port.limbs_to_int(port.oracle_full(u, v))
    for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        for pol in (tm.Policy.ACCURATE, tm.Policy.REFERENCE):
            p = tm.select_params(n, mode, policy=pol)
            res = []
            for c in (c3, c2, cg, c4):
                try:
                    r = tm.from_limbs(c.product_limbs(mode, u, v, p)); err = c.last_stats.max_round_err
                except Exception as e:  # noqa: BLE001
                    r = None; err = str(e)[:60]
                res.append((r, err))
            (r3, e3), (r2, e2), (rg, eg), (r4, e4) = res
            if r3 != r2 or e3 != e2 or rg != r2 or eg != e2 or r4 != r2 or e4 != e2:
                bad += 1; print("DIFF", n, kind, mode.name, pol.name, p, e3, e2, flush=True); continue
            if r3 is None: continue
            if mode == tm.Mode.FULL: ok = r3 == P
            elif mode == tm.Mode.LOW: ok = r3 == P & ((1 << n) - 1)
            else: ok = abs(P - (r3 << n)) < (1 << n) and 0 <= r3 <= (1 << n)
            if not ok:
                bad += 1; print("BAD", n, kind, mode.name, pol.name, p, flush=True)
    print(f"{i}: n={n} kind={kind} bad so far {bad}", flush=True)
print(f"bad {bad}")
sys.exit(1 if bad else 0)
