"""Host-side cost of one rq.factorize call (graph replay path) and the GPU step time, C2."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from synthetic import CONFIGS, make_A_config  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
A = make_A_config(c, device="cuda")
h = rq.Handle.default()
for _ in range(3):
    rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
    ts.append(time.perf_counter() - t0)
ts.sort()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(20):
    rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
e.record()
torch.cuda.synchronize()
print(f"{c.name}: host time per call {ts[len(ts) // 2] * 1e6:.1f} us; back-to-back GPU {s.elapsed_time(e) / 20 * 1e3:.1f} us/call")
