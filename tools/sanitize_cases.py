"""The cases compute-sanitizer runs in ONE process (one tool per gpurun call, B200_PROFILING.md):
C1 RQLP and C1e ERQLP (eager, then graph capture and replays: 3 calls each), C2 ERQLP (3 calls),
a BRQLP block case with the deflated power step (C4's shape reduced to m = 4096, n = 2048), the
rare orth branch (an ill-conditioned and a rank-deficient sketch: the cooperative rescue kernel
and its grid barrier), the row-sharded path on 3 loopback ranks, and the host-fed end-to-end entry
point.  Each case's output is checked for finiteness only: parity is the tests' job.

  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from paper_1811_09334_b200.dist import row_block  # noqa: E402
from synthetic import CONFIGS, make_A, make_A_config, sigma  # noqa: E402


def finite(out):
    for k in ("Q", "T", "P"):
        assert torch.isfinite(out[k]).all(), k


def run(name, fn):
    fn()
    torch.cuda.synchronize()
    print(f"[sanitize] {name}: ok", flush=True)


def main():
    for w in ("c1", "c1e", "c2"):
        c = CONFIGS[w]
        A = make_A_config(c, device="cuda")
        h = rq.Handle()

        def f():
            for _ in range(3):
                finite(rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h))
        run(w, f)
    # BRQLP block loop with a ragged block and a deflated power step (C4's n, k, p, b, q; m reduced)
    A = make_A(4096, 2048, sigma("exp100", 1024), rank=1024, noise=1e-8, seed=4, device="cuda")
    run("brqlp", lambda: [finite(rq.factorize(A, 120, 16, q=1, b=64, seed=4)) for _ in range(2)])
    # the rare orth branch: shifted passes (ill-conditioned) and random completion (rank deficient)
    rng = np.random.default_rng(3)
    for kind, sig in (("illcond", np.logspace(0, -13, 16)), ("deficient", np.array([3.0, 2.0, 1.0, 0.5]))):
        U, _ = np.linalg.qr(rng.standard_normal((600, len(sig))))
        V, _ = np.linalg.qr(rng.standard_normal((400, len(sig))))
        Ad = torch.from_numpy(np.ascontiguousarray(((U * sig) @ V.T).T)).cuda().t()
        run(f"rescue-{kind}", lambda Ad=Ad: [finite(rq.factorize(Ad, 12, 4, q=1, d=2, seed=5)) for _ in range(2)])
    # three loopback ranks (row-sharded path)
    c = CONFIGS["c1e"]
    A = make_A_config(c, device="cuda")
    hs = rq.Handle.loopback(3)
    errs = []

    def rank(r):
        try:
            r0, r1 = row_block(c.m, r, 3)
            for _ in range(2):
                rq.factorize(A[r0:r1], c.k, c.p, q=c.q, d=c.d, seed=c.seed, handle=hs[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    def lb():
        ths = [threading.Thread(target=rank, args=(r,)) for r in range(3)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        assert not errs, errs
    run("loopback-3", lb)
    # host-fed end-to-end entry point (rqlp_factorize with pinned host A: row panels on a copy stream)
    # (40000 x 2048: two row panels of 32768 and 7232 rows)
    A = make_A(40000, 2048, sigma("inv", 512), rank=512, noise=1e-6, seed=3, device="cuda")
    Ah = torch.empty(2048, 40000, dtype=torch.float64, pin_memory=True).t()
    Ah.copy_(A)
    h = rq.Handle()
    run("host-feed", lambda: [rq.factorize_host(Ah, 100, 10, q=1, d=2, seed=3, handle=h) for _ in range(3)])
    print("[sanitize] all cases done", flush=True)


if __name__ == "__main__":
    main()
