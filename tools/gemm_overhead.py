"""Fixed per-launch cost of the A-pass GEMM kernel: Y = A X with one 128-row tile per SM
(m = 128 x #SMs) and k = 24 s (s k-tiles), for s = 1 .. 64; the intercept of time vs s is the
launch + ramp + cold-instruction-fetch cost, the slope the per-k-tile time.

  python tools/gemm_overhead.py [c]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 112
sms = torch.cuda.get_device_properties(0).multi_processor_count
m = 128 * sms
res = []
for s in (1, 2, 4, 8, 16, 32, 64):
    k = 24 * s
    A = rq.cm_empty(m, k, torch.device("cuda"))
    A.normal_()
    X = rq.cm_empty(k, c, torch.device("cuda"))
    X.normal_()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ts = []
    for rep in range(12):
        flush.add_(1.0)   # evict L2 (and, with it, the kernel's instructions)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rq.gemm_nn(A, X)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    res.append((s, ts[len(ts) // 2]))
    print(f"c={c} k-tiles={s:3d}: {ts[len(ts) // 2]:8.2f} us", flush=True)
# least squares t = a + b s
n = len(res)
sx = sum(s for s, _ in res)
sy = sum(t for _, t in res)
sxx = sum(s * s for s, _ in res)
sxy = sum(s * t for s, t in res)
b = (n * sxy - sx * sy) / (n * sxx - sx * sx)
a = (sy - b * sx) / n
print(f"fit: {a:.2f} us fixed + {b:.3f} us per k-tile (ideal per k-tile at 37.07 TF: "
      f"{128 * c * 24 * 2 * sms / 37.07e12 * 1e6:.3f} us)")
