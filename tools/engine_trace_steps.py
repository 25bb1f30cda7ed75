"""Debug: per-step cycles of the CPQR engine along the factorisation (RQLP_ENGINE_TRACE=1, CTA 0):
  python tools/engine_trace_steps.py l n"""
import ctypes, os, sys
os.environ["RQLP_ENGINE_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_09334_b200 as rq
l, n = int(sys.argv[1]), int(sys.argv[2])
B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda"))
for _ in range(2):
    rq.cpqr(B)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
steps = min(l, n)
buf = (ctypes.c_ulonglong * (4 * steps))()
assert lib.rqlp_debug_trace(buf, 4 * steps) == 0
t = np.array(buf, dtype=np.float64).reshape(steps, 4)
d = np.diff(t[:, 0])
for a in range(0, steps - 1, max(1, (steps - 1) // 16)):
    seg = d[a:a + 16]
    print(f"steps {a:5d}+: {np.median(seg):8.0f} cycles/step  update {np.median(t[a+1:a+17,3]-t[a+1:a+17,2]):8.0f}  poll {np.median(t[a+1:a+17,1]-t[a+1:a+17,0]):7.0f}")
print("total cycles", t[-1, 0] - t[0, 0], "=", (t[-1, 0] - t[0, 0]) / 1.965e3, "us")
