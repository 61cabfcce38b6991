"""Phase clocks of one row pair of k_mid_4096w (library built with -DTMG_MID_DEBUG)."""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import _native
from oracle import port
lib = _native.load()
n = 1 << 26
u, v = port.config_operands(3, n // 64)
ctx = tm.default_context(0)
old = len(sys.argv) > 1 and sys.argv[1] == 'old'
if old: ctx.set_option(_native.TMG_OPT_ROW_PASS_BARRIERS, 1)
for m in (tm.Mode.FULL,):
    for _ in range(3):
        ctx.product_limbs(m, u, v, tm.select_params(n, m, policy=tm.Policy.ACCURATE))
buf = (ctypes.c_longlong * 256)()
lib.tmg_debug_mid_clocks.argtypes = [ctypes.c_void_p]
print("rc", lib.tmg_debug_mid_clocks(buf))
a = np.array(buf).reshape(16, 16)
t0 = a[:, 0].min()
if old: names = ["start", "mbar", "loads", "s0 stored", "s1 loaded", "s1 stored", "s2 dft", "spec+i0", "i0 stored", "done", "", ""]
else: names = ["start", "loads issued", "dft0", "barA", "stored+barB1", "S1 done", "S2 done", "spectral", "I0 stored", "I1 done", "barB2", "I2 done"]
print("warp " + " ".join(f"{x[:9]:>9}" for x in names))
for w in range(16):
    print(f"{w:4d} " + " ".join(f"{a[w, i] - t0:9d}" for i in range(12)))
