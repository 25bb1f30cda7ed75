"""Per-block phase times (SM cycles) of chol_blk_kernel (RQLP_ENGINE_TRACE=1 debug stamps):
orth of a random m x c matrix; the LAST full (non-near-identity) Cholesky of the call is traced.

  python tools/chol_trace.py [m] [c]
"""
import ctypes
import os
import sys

os.environ["RQLP_ENGINE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
c = int(sys.argv[2]) if len(sys.argv) > 2 else 110
Y = rq.col_major(torch.randn(m, c, dtype=torch.float64, device="cuda"))
for _ in range(3):
    rq.orth(Y)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
n = 16 * 4096
buf = (ctypes.c_ulonglong * n)()
assert lib.rqlp_debug_trace(buf, n) == 0
raw = np.array(buf[8 * 4096:8 * 4096 + 160], dtype=np.int64)
t = raw[:128].reshape(32, 4)
pv = raw[128:137]
print("phase1(block 0) per pivot:", np.diff(pv).tolist(), " start offset", int(pv[0] - t[31, 0]), " end->stamp", int(t[31, 1] - pv[8]))
nt = (c + 7) // 8
print(f"chol_blk n={c}: phase1(block 0) {t[31, 1] - t[31, 0]} cycles")
print(" kb   phase2  phase3  (warp0: tile0+phase1(kb+1))  block total")
tot = 0
for kb in range(nt):
    p2 = t[kb, 1] - t[kb, 0]
    p3 = t[kb, 2] - t[kb, 1]
    w0 = t[kb, 3] - t[kb, 1] if kb + 1 < nt else 0
    blk = (t[kb + 1, 0] - t[kb, 0]) if kb + 1 < nt else (t[kb, 2] - t[kb, 0])
    tot += blk
    print(f"{kb:3d} {p2:8d} {p3:7d} {w0:12d} {blk:18d}")
print(f"blocked loop: {tot} cycles = {tot / 1.965e3:.1f} us at 1965 MHz")
