"""Break down the host time of one rq.erqlp call (graph replay) into its Python/C pieces."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_09334_b200 as rq  # noqa: E402
from paper_1811_09334_b200 import _ld, _mat, _outputs, _ptr, lib  # noqa: E402
from synthetic import CONFIGS, make_A_config  # noqa: E402

c = CONFIGS["c2"]
A = make_A_config(c, device="cuda")
h = rq.Handle.default()
for _ in range(3):
    rq.factorize(A, c.k, c.p, q=c.q, d=c.d, seed=c.seed, handle=h)
torch.cuda.synchronize()
m, n, l = c.m, c.n, c.k + c.p
acc = {}
for it in range(30):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    A2 = _mat(A, "A"); t.append(time.perf_counter())
    h.workspace(1, m, n, c.k, c.p, c.q, c.d, 0); t.append(time.perf_counter())
    Q, T, P, piv0 = _outputs(m, n, l, 1, A.device); t.append(time.perf_counter())
    args = (h.h, m, n, c.k, c.p, c.q, c.d, _ptr(A2), _ld(A2), c.seed, _ptr(Q), _ld(Q), _ptr(T), _ld(T))
    t.append(time.perf_counter())
    tu = ctypes.c_int(0)
    rc = lib().erqlp_ex(*args, ctypes.byref(tu), _ptr(P), _ld(P), _ptr(piv0)); t.append(time.perf_counter())
    for i, name in enumerate(["mat", "workspace", "outputs", "args", "C call"]):
        acc.setdefault(name, []).append(t[i + 1] - t[i])
for k, v in acc.items():
    v.sort()
    print(f"{k:10s} {v[len(v) // 2] * 1e6:7.1f} us")
