"""Exactness over random operand sizes: full and low products bit-exact
against GMP, high products within the bound, for random n in [4096, 2^24]
(every plan family: fused single-CTA, two-pass generic and compiled column
shapes, fallback schoolbook below 4096).

    python tools/random_sizes.py [count] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    ctx = tm.default_context(0)
    bad = 0
    for i in range(count):
        n = int(np.exp(rng.uniform(np.log(1000), np.log(1 << 24))))
        nl = (n + 63) // 64
        u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        v = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        P = port.limbs_to_int(port.oracle_full(u, v))
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
            try:
                r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
                if mode == tm.Mode.FULL:
                    ok = r == P
                elif mode == tm.Mode.LOW:
                    ok = r == P & ((1 << n) - 1)
                else:
                    ok = abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)
            except Exception as e:  # noqa: BLE001
                ok = False
                print("EXC", n, mode.name, e)
            if not ok:
                bad += 1
                print("BAD", n, mode.name, p)
        if i % 20 == 0:
            print(f"{i}: n={n} ok", flush=True)
    print(f"bad {bad} of {3 * count}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
