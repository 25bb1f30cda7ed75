#!/usr/bin/env python
"""Time the A-pass GEMMs (stage entry points rqlp_gemm_nn / rqlp_gemm_tn) at given shapes.

  python tools/gemm_bench.py [--reps 20] [--shapes m,k,c ...]
Prints TFLOP/s per shape and mode (CUDA events around `reps` back-to-back calls).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--shapes", nargs="*", default=["4096,4096,110", "65536,8192,272", "131072,16384,1056",
                                                 "2000,2000,125", "262144,16384,64"])
a = ap.parse_args()
for sh in a.shapes:
    m, k, c = map(int, sh.split(","))
    A = rq.cm_empty(m, k, torch.device("cuda"))
    A.normal_()
    X = rq.cm_empty(k, c, torch.device("cuda"))
    X.normal_()
    V = rq.cm_empty(m, c, torch.device("cuda"))
    V.normal_()
    for mode in ("nn", "tn"):
        f = (lambda: rq.gemm_nn(A, X)) if mode == "nn" else (lambda: rq.gemm_tn(A, V, trans_out=True))
        f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.reps):
            f()
        e.record()
        torch.cuda.synchronize()
        t = s.elapsed_time(e) / a.reps / 1e3
        print(f"{mode} m={m} k={k} c={c}: {t * 1e6:9.1f} us  {2 * m * k * c / t / 1e12:6.2f} TFLOP/s", flush=True)
    del A, X, V
    torch.cuda.empty_cache()
