#!/usr/bin/env python
"""Time rq.orth (CholeskyQR2 incl. the c x c Cholesky kernel) at given shapes.
  python tools/orth_bench.py [--reps 50] [--shapes m,c ...]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--shapes", nargs="*", default=["110,110", "125,125", "4096,110", "2000,125", "64,64", "128,128"])
a = ap.parse_args()
for sh in a.shapes:
    m, c = map(int, sh.split(","))
    Y = rq.cm_empty(m, c, torch.device("cuda"))
    Y.normal_()
    rq.orth(Y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        rq.orth(Y)
    e.record()
    torch.cuda.synchronize()
    print(f"orth m={m} c={c}: {s.elapsed_time(e) / a.reps * 1e3:9.1f} us", flush=True)
