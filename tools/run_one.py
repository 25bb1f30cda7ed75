"""Run `reps` factorisations of a workload (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from synthetic import CONFIGS, make_A_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
c = CONFIGS[a.workload]
A = make_A_config(c, device="cuda")
torch.cuda.synchronize()
for _ in range(a.reps):
    rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed)
torch.cuda.synchronize()
print("done", a.workload, rq.Handle.default().launches(), "launches/factorisation")
