"""Run `reps` factorisations of a workload (for ncu / compute-sanitizer captures).

  python tools/run_one.py --workload c2 [--reps 2] [--loopback P] [--host]
--loopback P runs the workload row-sharded over P loopback ranks (rqlp_create_loopback, one host
thread per rank); --host runs the end-to-end entry point rqlp_factorize with pinned host A.
"""
import argparse
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from paper_1811_09334_b200.dist import row_block  # noqa: E402
from synthetic import CONFIGS, make_A_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--loopback", type=int, default=0)
ap.add_argument("--host", action="store_true")
a = ap.parse_args()
c = CONFIGS[a.workload]
A = make_A_config(c, device="cuda")
torch.cuda.synchronize()
if a.loopback:
    hs = rq.Handle.loopback(a.loopback)

    def job(r):
        r0, r1 = row_block(c.m, r, a.loopback)
        for _ in range(a.reps):
            rq.factorize(A[r0:r1], c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=hs[r])

    ths = [threading.Thread(target=job, args=(r,)) for r in range(a.loopback)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    print("done", a.workload, f"loopback p={a.loopback}", [h.sync() for h in hs])
elif a.host:
    Ah = torch.empty(c.n, c.m, dtype=torch.float64, pin_memory=True).t()
    Ah.copy_(A)
    h = rq.Handle()
    for _ in range(a.reps):
        rq.factorize_host(Ah, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
    print("done", a.workload, "host feed", h.sync())
else:
    for _ in range(a.reps):
        rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed)
    torch.cuda.synchronize()
    print("done", a.workload, rq.Handle.default().launches(), "launches/factorisation")
