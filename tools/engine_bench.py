"""Timing of the CPQR stage (rq.cpqr: engine + compaction + R extraction + explicit Q) on
B-shaped inputs, CUDA events over many repetitions.  python tools/engine_bench.py [l n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

shapes = [(110, 4096), (272, 8192), (64, 16384), (25, 800), (110, 110)]
if len(sys.argv) > 2:
    a = list(map(int, sys.argv[1:]))
    shapes = list(zip(a[0::2], a[1::2]))
tag = os.environ.get("TAG", "")
for l, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda", generator=g))
    for _ in range(3):
        rq.cpqr(B)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        rq.cpqr(B)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    s = min(l, n)
    print(f"{tag} cpqr {l}x{n}: median {ts[reps // 2]:.1f} us  min {ts[0]:.1f} us  ({ts[reps // 2] / s:.2f} us/step)",
          flush=True)
