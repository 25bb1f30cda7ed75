"""Debug: per-CTA timing of the grid CPQR engine (RQLP_ENGINE_TRACE=1), steps 20..59, SM cycles
(clock64 is per SM: only differences within one CTA are compared).
  work  = record out (step j+1)  - fetch done (step j)   : this CTA's own step work
  tail  = poll start (j+1)       - record out (j+1)      : warp 0's deferred updates after its publish
  wait  = poll done (j+1)        - poll start (j+1)      : waiting for the other CTAs' records
  fetch = fetch done (j+1)       - poll done (j+1)       : candidate-column round trip + barriers"""
import ctypes
import os
import sys

os.environ.setdefault("RQLP_ENGINE_TRACE", "1")   # "2": %globaltimer ns (comparable across SMs)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 110
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda"))
for _ in range(3):
    rq.cpqr(B)
torch.cuda.synchronize()
lib = rq.lib()
lib.rqlp_debug_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
N = 8192 + 40 * 148 * 4
buf = (ctypes.c_ulonglong * N)()
assert lib.rqlp_debug_trace(buf, N) == 0
t = np.array(buf[8192:], dtype=np.float64).reshape(40, 148, 4)
G = min(148, (n + 7) // 8)


def q(x):
    return f"min {np.min(x):6.0f} med {np.median(x):6.0f} p90 {np.percentile(x, 90):6.0f} max {np.max(x):6.0f}"


t = t[:, :G]
work = t[1:, :, 3] - t[:-1, :, 2]
tail = t[1:, :, 0] - t[1:, :, 3]
wait = t[1:, :, 1] - t[1:, :, 0]
fetch = t[1:, :, 2] - t[1:, :, 1]
step = t[1:, :, 2] - t[:-1, :, 2]
print(f"l={l} n={n} G={G} (env W0FREE={os.environ.get('RQLP_ENGINE_W0FREE', '1')}, trace={os.environ['RQLP_ENGINE_TRACE']})")
if os.environ["RQLP_ENGINE_TRACE"] == "2":
    # globaltimer (ns, 32 ns ticks): cross-CTA comparisons of step j+1 (rows 1..)
    rec = t[1:, :, 3]            # record out for step j
    pd = t[1:, :, 1]             # poll done, step j
    fd = t[1:, :, 2]             # fetch done, step j
    last = rec.max(axis=1, keepdims=True)
    first = rec.min(axis=1, keepdims=True)
    print(f"  record spread (last-first) ns: {q(last - first)}")
    print(f"  poll done - last record ns:   {q(pd - last)}")
    print(f"  fetch done spread ns:          {q(fd.max(axis=1) - fd.min(axis=1))}")
    print(f"  last-record CTA per step: {np.argmax(rec, axis=1)[:20].tolist()}")
    stp = np.diff(fd.mean(axis=1))
    print(f"  mean step ns: {np.median(stp):.0f}")
for nm, x in (("work", work), ("tail", tail), ("wait", wait), ("fetch", fetch), ("step", step)):
    print(f"  {nm:5s} {q(x)}")
# which CTAs are late: per step, the CTA with the largest work
wmax = np.argmax(work, axis=1)
print("  slowest-work CTA per step:", wmax[:20].tolist())
print("  per-CTA median work (first 16 CTAs):", np.median(work, axis=0)[:16].astype(int).tolist())
print("  per-CTA median work (last 8 CTAs):", np.median(work, axis=0)[-8:].astype(int).tolist())
