"""One CPQR per shape after a warm-up, for ncu (-k regex:hh_engine): python tools/ncu_engine.py l n [l n ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1811_09334_b200 as rq  # noqa: E402

a = list(map(int, sys.argv[1:])) or [110, 4096]
for l, n in zip(a[0::2], a[1::2]):
    g = torch.Generator(device="cuda").manual_seed(1)
    B = rq.col_major(torch.randn(l, n, dtype=torch.float64, device="cuda", generator=g))
    rq.cpqr(B)
    torch.cuda.synchronize()
    rq.cpqr(B)
    torch.cuda.synchronize()
print("ok")
