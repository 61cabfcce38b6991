"""Step throughput with the three products of a step on three contexts
(streams, workspaces) vs one context: python tools/concurrent_step.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from oracle import port
n = 1 << 26
u, v = port.config_operands(3, n // 64)
dev = torch.device('cuda:0')
du = torch.from_numpy(u.view(np.int64)).to(dev)
dv = torch.from_numpy(v.view(np.int64)).to(dev)
modes = (tm.Mode.FULL, tm.Mode.LOW, tm.Mode.HIGH)
params = {m: tm.select_params(n, m, policy=tm.Policy.ACCURATE) for m in modes}
outs = {m: torch.zeros(tm.output_limbs(m, n), dtype=torch.int64, device=dev) for m in modes}
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ctxs = {m: tm.Context(0) for m in modes}
streams = {m: torch.cuda.Stream(device=dev) for m in modes}
for m in modes:
    ctxs[m].set_stream(streams[m].cuda_stream)
one = tm.Context(0)
s1 = torch.cuda.Stream(device=dev)
one.set_stream(s1.cuda_stream)


def run(concurrent, steps):
    ms = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream(dev)
        a.record(main)
        if concurrent:
            for m in modes:
                streams[m].wait_event(a)
                ctxs[m].product_device(params[m], du.data_ptr(), dv.data_ptr(), outs[m].data_ptr(), 1)
            for m in modes:
                e = torch.cuda.Event()
                e.record(streams[m])
                main.wait_event(e)
        else:
            s1.wait_event(a)
            for m in modes:
                one.product_device(params[m], du.data_ptr(), dv.data_ptr(), outs[m].data_ptr(), 1)
            e = torch.cuda.Event()
            e.record(s1)
            main.wait_event(e)
        b.record(main)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    for c in list(ctxs.values()) + [one]:
        c.check()
    return float(np.mean(ms))


for conc in (False, True, False, True):
    run(conc, 5)
    t = run(conc, 50)
    print(f"concurrent={conc}: {t:.4f} ms/step, {3 * 2 * n / (t * 1e-3) / 1e9:.1f} Gbit/s", flush=True)
