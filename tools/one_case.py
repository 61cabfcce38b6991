"""Run one product on the GPU and check it against the oracle:
python tools/one_case.py MODE LOG2N [seed]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1703_00640_b200 as tm
from oracle import port
mode = tm.Mode[sys.argv[1].upper()]
n = 1 << int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 3
nl = (n + 63) // 64
u, v = port.config_operands(seed, nl)
p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
print("params", p, flush=True)
ctx = tm.default_context(0)
t0 = time.time()
r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
print("gpu done", time.time() - t0, ctx.last_stats, flush=True)
P = port.limbs_to_int(port.oracle_full(u, v))
if mode == tm.Mode.FULL: ok = r == P
elif mode == tm.Mode.LOW: ok = r == (P & ((1 << n) - 1))
else: ok = port.is_valid_high(u, v, n, r)
print("ok", ok, flush=True)
