"""Products of every plan family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_case.py [max_log2n]
    compute-sanitizer --tool racecheck python tools/sanitize_case.py [max_log2n]

Sizes: the schoolbook fallback (n < 4096), the fused single-CTA kernels
(compiled 5120 / 6144 and generic lengths), the two-pass plans with generic
and compiled column shapes, mid-size row passes (1024 / 2048 rows), the
runs split and runs carry (2^24 and above) and, with max_log2n >= 28, the
three-pass plans.  Both parameter policies, a small batch through the fused
kernel and through graph-replayed multi-pass products, and ragged sizes.
Every result is checked against the exact product (oracle), so a run under
the sanitizer is also a parity run; where the sanitizer is unavailable (it
is closed on the round's GPU pool) the script alone is a parity run over
every plan family.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def check(mode, n, u, v, r, P):
    if mode == tm.Mode.FULL:
        return r == P
    if mode == tm.Mode.LOW:
        return r == P & ((1 << n) - 1)
    return abs(P - (r << n)) < (1 << n) and 0 <= r <= (1 << n)


def main():
    maxlg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    rng = np.random.default_rng(17)
    ctx = tm.default_context(0)
    sizes = [1000, 4096, 5001, 8192, 40000, 1 << 16, 100003, 1 << 18, 700001, 1 << 20, 3000017,
             1 << 22, 1 << 24, (1 << 24) + 12345, 1 << 26, 1 << 28]
    bad = 0
    for n in sizes:
        if n > (1 << maxlg) + (1 << 20):
            continue
        nl = (n + 63) // 64
        u = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        v = port.int_to_limbs(int.from_bytes(rng.bytes(nl * 8), "little") & ((1 << n) - 1), nl)
        P = port.limbs_to_int(port.oracle_full(u, v))
        for policy in (tm.Policy.ACCURATE, tm.Policy.REFERENCE):
            for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
                p = tm.select_params(n, mode, policy=policy)
                try:
                    r = tm.from_limbs(ctx.product_limbs(mode, u, v, p))
                    ok = check(mode, n, u, v, r, P)
                    tag = "ok" if ok else "BAD"
                except tm.ConvolutionPrecisionFailure:
                    # the reference's own parameters may trip its tripwire (2^26 low / high)
                    ok, tag = policy == tm.Policy.REFERENCE, "refused"
                bad += 0 if ok else 1
                print(f"n={n} {policy.name} {mode.name} b={p.b} N={p.N}: {tag}", flush=True)
    # batches: fused kernel (2^16) and multi-pass graph replay (2^18)
    for n, count in ((1 << 16, 8), (1 << 18, 4), (6000, 5)):
        nl = (n + 63) // 64
        w = rng.integers(0, 2**64, (count, 2, nl), dtype=np.uint64)
        if n & 63:
            w[:, :, -1] &= np.uint64((1 << (n & 63)) - 1)
        u = np.ascontiguousarray(w[:, 0, :])
        v = np.ascontiguousarray(w[:, 1, :])
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
            out, flags = ctx.product_batched(p, u, v, return_flags=True)
            ok = not flags.any()
            for i in range(count):
                P = port.limbs_to_int(port.oracle_full(u[i], v[i]))
                ok = ok and check(mode, n, u[i], v[i], tm.from_limbs(out[i]), P)
            bad += 0 if ok else 1
            print(f"batch n={n} x{count} {mode.name}: {'ok' if ok else 'BAD'}", flush=True)
    print(f"bad {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
