import ctypes, os, sys
os.environ["RQLP_ENGINE_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_09334_b200 as rq
l, n = int(sys.argv[1]), int(sys.argv[2])
B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda"))
for _ in range(3):
    rq.cpqr(B)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * (16 * 4096))()
assert lib.rqlp_debug_trace(buf, 16 * 4096) == 0
a = np.array(buf, dtype=np.float64)
steps = min(l, n)
t = a[:4 * steps].reshape(steps, 4)
x = a[4 * 4096:4 * 4096 + 8 * steps].reshape(steps, 8)
m = lambda v: np.median(v[2:-2])
print("refl->colstart", m(x[:, 0] - t[:, 2]), "dot+gsum", m(x[:, 1] - x[:, 0]), "w/store", m(x[:, 2] - x[:, 1]),
      "downdate", m(x[:, 3] - x[:, 2]), "warpbest", m(x[:, 4] - x[:, 3]), "sync", m(t[:, 3] - x[:, 4]))
