#!/usr/bin/env python
"""Per-stage device times (handle timing marks) of one factorisation, graph-replayed.

  python tools/stage_times.py --m 2000 --n 2000 --k 120 --p 5 --q 0 --d 0 [--tqlp] [--reps 5]
"""
import argparse
import collections
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from synthetic import make_A, sigma  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--k", type=int, default=120)
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--q", type=int, default=0)
ap.add_argument("--d", type=int, default=0)
ap.add_argument("--b", type=int, default=None)
ap.add_argument("--tqlp", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
A = make_A(a.m, a.n, sigma("exp50", min(a.m, a.n)), seed=1, device="cuda")
h = rq.Handle.default()
h.set_timing(True)
acc = collections.OrderedDict()


def run():
    if a.tqlp:
        return rq.tqlp(A, a.k + a.p)
    return rq.factorize(A, a.k, a.p, q=a.q, d=a.d, b=a.b, seed=3)


for _ in range(2):
    run()
torch.cuda.synchronize()
tot = []
for _ in range(a.reps):
    run()
    t = h.timing()
    tot.append(sum(ms for _, ms in t))
    per = collections.OrderedDict()
    for name, ms in t:
        per[name] = per.get(name, 0.0) + ms
    for name, ms in per.items():
        acc.setdefault(name, []).append(ms)
for name, v in acc.items():
    v = sorted(v)
    print(f"{name:24s} {v[len(v) // 2] * 1e3:10.1f} us")
tot.sort()
print(f"{'total':24s} {tot[len(tot) // 2] * 1e3:10.1f} us   launches={h.launches()}")
