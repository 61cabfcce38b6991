import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from oracle import port
ctx = tm.Context(0); dev = torch.device('cuda:0'); st = torch.cuda.current_stream(dev); ctx.set_stream(st.cuda_stream)
for lg in [int(x) for x in (sys.argv[1:] or ["20", "22"])]:
    n = 1 << lg; u, v = port.config_operands(7, n // 64)
    du = torch.from_numpy(u.view(np.int64)).to(dev); dv = torch.from_numpy(v.view(np.int64)).to(dev)
    for mode in (tm.Mode.LOW, tm.Mode.FULL, tm.Mode.HIGH):
        p = tm.select_params(n, mode, policy=tm.Policy.ACCURATE); out = torch.zeros(tm.output_limbs(mode, n), dtype=torch.int64, device=dev)
        for _ in range(3): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
        ctx.check(); ctx.profile(True)
        for _ in range(5): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
        recs = ctx.profile_read(); ctx.profile(False); ctx.check()
        agg = {}
        for nm, ms, by in recs: agg.setdefault(nm, []).append(ms)
        print(f"2^{lg} {mode.name}:", ", ".join(f"{k.split(':')[1]} {1e3*np.median(v):.1f}" for k, v in agg.items()))
