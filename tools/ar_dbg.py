import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import _rand_svd, _cm
import paper_1811_09334_b200 as rq, oracle as orc
m, n, b, lm, eps, q = [float(x) if "." in x or "e" in x else int(x) for x in sys.argv[1:7]]
sig = np.exp(-np.arange(1, min(m, n) + 1.0) / 40)
A = _rand_svd(m, n, sig, m + 3 * n)
g = rq.autorank(_cm(A), b=b, l_max=lm, eps=eps, q=q, seed=6)
torch.cuda.synchronize()
o = orc.autorank(A, b=b, l_max=lm, eps=eps, q=q, seed=6)
print("gpu", g["l"], g["err"], "orc", o["l"], o["err"])
