"""Debug: per-phase timing of the CPQR engine (RQLP_ENGINE_TRACE=1), phases per step:
poll/exchange -> reflector -> update -> publish."""
import ctypes
import os
import sys

os.environ["RQLP_ENGINE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 110
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
B = torch.randn(n, l, dtype=torch.float64, device="cuda").t().contiguous().t()
B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda"))
for _ in range(3):
    rq.cpqr(B)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
steps = min(l, n)
buf = (ctypes.c_ulonglong * (4 * steps))()
assert lib.rqlp_debug_trace(buf, 4 * steps) == 0
t = np.array(buf, dtype=np.float64).reshape(steps, 4)
d_poll = t[1:, 1] - t[1:, 0]
d_refl = t[1:, 2] - t[1:, 1]
d_upd = t[1:, 3] - t[1:, 2]
d_pub = t[1:, 0] - t[:-1, 3]
print(f"l={l} n={n}: per-step SM cycles  poll/exchange {np.median(d_poll):.0f}  reflector {np.median(d_refl):.0f}  "
      f"update {np.median(d_upd):.0f}  publish {np.median(d_pub):.0f}  total/step {np.median(np.diff(t[:, 0])):.0f}")
d = np.diff(t[:, 0])
print(f"   first steps (cycles): {d[:4].astype(int).tolist()}  last: {d[-3:].astype(int).tolist()}")
