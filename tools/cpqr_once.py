"""Run rq.cpqr on a random rows x cols matrix `reps` times (for ncu captures of the engine)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402

l, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 2
B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda"))
for _ in range(reps):
    rq.cpqr(B)
torch.cuda.synchronize()
