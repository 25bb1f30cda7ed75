"""Debug: phase timing of the blocked Cholesky kernel (RQLP_ENGINE_TRACE=1)."""
import ctypes
import os
import sys

os.environ["RQLP_ENGINE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 110
Y = rq.cm_empty(4 * n, n, torch.device("cuda"))
Y.normal_()
for _ in range(3):
    rq.orth(Y)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
nt = (n + 7) // 8
cnt = 4 + 4 * nt
buf = (ctypes.c_ulonglong * cnt)()
assert lib.rqlp_debug_trace(buf, cnt) == 0
t = np.array(buf, dtype=np.int64)
print(f"n={n}: first phase1 {t[1] - t[0]} ns")
st = t[4:].reshape(nt, 4)[:-1]
p2 = st[:, 1] - st[:, 0]
p1 = st[:, 3] - st[:, 2]
tile0 = st[:, 2] - st[:, 1]
blk = np.diff(t[4:].reshape(nt, 4)[:, 0])
print(f"per block (median ns): phase2+barrier {np.median(p2):.0f}  tile0 {np.median(tile0):.0f}  phase1 {np.median(p1):.0f}  block total {np.median(blk):.0f}")
