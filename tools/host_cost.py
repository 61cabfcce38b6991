import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from oracle import port
ctx = tm.Context(0); dev = torch.device('cuda:0'); st = torch.cuda.current_stream(dev); ctx.set_stream(st.cuda_stream)
for lg in (18, 20):
    n = 1 << lg; u, v = port.config_operands(7, n // 64)
    du = torch.from_numpy(u.view(np.int64)).to(dev); dv = torch.from_numpy(v.view(np.int64)).to(dev)
    p = tm.select_params(n, tm.Mode.LOW, policy=tm.Policy.ACCURATE); out = torch.zeros(tm.output_limbs(tm.Mode.LOW, n), dtype=torch.int64, device=dev)
    for _ in range(5): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); R = 200
    for _ in range(R): ctx.product_device(p, du.data_ptr(), dv.data_ptr(), out.data_ptr(), 1)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"2^{lg}: host enqueue {1e6*(t1-t0)/R:.1f} us/product, wall {1e6*(t2-t0)/R:.1f} us/product")
