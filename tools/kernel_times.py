"""Median per-kernel times (us) of the multi-pass products at 2^LG bits,
plus the whole product (events around 5 back-to-back products):
python tools/kernel_times.py [LG ...] [--opt NAME=VALUE ...]
(NAME: a TMG_OPT_* constant of _native without the prefix)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import _native
from oracle import port
args = sys.argv[1:]
opts = [a.split('=') for a in args[args.index('--opt') + 1:]] if '--opt' in args else []
lgs = [int(x) for x in (args[:args.index('--opt')] if '--opt' in args else args)] or [20, 22]
ctx = tm.Context(0); dev = torch.device('cuda:0'); st = torch.cuda.current_stream(dev); ctx.set_stream(st.cuda_stream)
for k, v in opts:
    ctx.set_option(getattr(_native, 'TMG_OPT_' + k), int(v))
for lg in lgs:
    n = 1 << lg; u, v = port.config_operands(7, n // 64)
    du = torch.from_numpy(u.view(np.int64)).to(dev); dv = torch.from_numpy(v.view(np.int64)).to(dev)
    for mode in (tm.Mode.LOW, tm.Mode.FULL, tm.Mode.HIGH):
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE); out = torch.zeros(tm.output_limbs(mode, n), dtype=torch.int64, device=dev)
        for _ in range(3): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
        ctx.check()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
        e1.record(st); torch.cuda.synchronize(); tot = e0.elapsed_time(e1) / 5 * 1e3
        ctx.check(); ctx.profile(True)
        for _ in range(5): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
        recs = ctx.profile_read(); ctx.profile(False); ctx.check()
        agg = {}
        for nm, ms, by in recs: agg.setdefault(nm, []).append(ms)
        print(f"2^{lg} {mode.name} N={p.N} product {tot:.1f}:", ", ".join(f"{k.split(':')[1]} {1e3*np.median(v):.1f}" for k, v in agg.items()), flush=True)
