"""One warm-up and one measured product of each mode at n = 2^LOG2N, for ncu:
python tools/prof_case.py [log2n]  (kernels per product at 2^26: full 5, low 5, high 6)"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1703_00640_b200 as tm
from oracle import port
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << lg
u, v = port.config_operands(3, n // 64)
ctx = tm.default_context(0)
for rep in range(2):
    for m in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
        ctx.product_limbs(m, u, v, tm.select_params(n, m, policy=tm.Policy.ACCURATE))
print("done")
