"""BASELINE config 4: 4096 independent low products of n = 2^16 bits in one
batched launch (k_small_product, one CTA per product).  Device-resident
operands, CUDA-event timing, input Gbit/s.

    python tools/batch_bench.py [count] [log2n] [mode]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00640_b200 as tm  # noqa: E402
from oracle import port  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    lg = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    mode = tm.Mode[(sys.argv[3] if len(sys.argv) > 3 else "low").upper()]
    n = 1 << lg
    nl = n // 64
    w = port.mt19937_64(4, 2 * count * nl).reshape(count, 2, nl)
    u = np.ascontiguousarray(w[:, 0, :])
    v = np.ascontiguousarray(w[:, 1, :])
    p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE)
    ctx = tm.Context(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    du = torch.from_numpy(u.view(np.int64)).to(dev)
    dv = torch.from_numpy(v.view(np.int64)).to(dev)
    ol = tm.output_limbs(mode, n)
    dout = torch.zeros(count * ol, dtype=torch.int64, device=dev)
    for _ in range(3):
        ctx.product_device(p, du.data_ptr(), dv.data_ptr(), dout.data_ptr(), count)
    ctx.check()
    times = []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.product_device(p, du.data_ptr(), dv.data_ptr(), dout.data_ptr(), count)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    st = ctx.check()
    ms = float(np.median(times))
    out = dout.cpu().numpy().view(np.uint64).reshape(count, ol)
    ok = all(np.array_equal(out[i], port.oracle_low(u[i], v[i], n)) for i in range(0, count, 97)) \
        if mode == tm.Mode.LOW else None
    bits = count * 2 * n
    print(f"{count} x {mode.name} n=2^{lg} (b={p.b}, N={p.N}, L={st.transform_length}): "
          f"{ms:.3f} ms, {bits / (ms * 1e-3) / 1e9:.1f} Gbit/s, "
          f"{count / (ms * 1e-3) / 1e6:.2f} M products/s, max err {st.max_round_err:.4f}, sample exact {ok}")


if __name__ == "__main__":
    main()
