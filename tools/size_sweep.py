"""Device-resident throughput of single products across sizes (input Gbit/s
= 2n bits per product / time), back-to-back products on one stream timed
with CUDA events, next to the sum of the per-kernel times (the gap is launch
overhead).

    python tools/size_sweep.py [log2n ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def main():
    lgs = [int(x) for x in sys.argv[1:]] or [16, 18, 20, 22, 24, 26, 28]
    ctx = tm.Context(0)
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream(dev)
    ctx.set_stream(st.cuda_stream)
    print("| n | mode | b | L | us / product | Gbit/s | sum of kernels us | kernels |")
    print("|---|---|---|---|---|---|---|---|")
    for lg in lgs:
        n = 1 << lg
        u, v = port.config_operands(7, n // 64)
        du = torch.from_numpy(u.view(np.int64)).to(dev)
        dv = torch.from_numpy(v.view(np.int64)).to(dev)
        for mode in (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH):
            p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
            out = torch.zeros(tm.output_limbs(mode, n), dtype=torch.int64, device=dev)
            reps = max(3, min(200, (1 << 26) // n))
            for _ in range(3):
                ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
            s = ctx.check()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(reps):
                ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
            b.record(st)
            b.synchronize()
            ms = a.elapsed_time(b) / reps
            ctx.check()
            ctx.profile(True)
            ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
            recs = ctx.profile_read()
            ctx.profile(False)
            ctx.check()
            ksum = sum(r[1] for r in recs)
            print(f"| 2^{lg} | {mode.name.lower()} | {p.b} | {s.transform_length} | {ms * 1e3:.1f} | "
                  f"{2 * n / (ms * 1e-3) / 1e9:.1f} | {ksum * 1e3:.1f} | {len(recs)} |", flush=True)


if __name__ == "__main__":
    main()
