"""The optional Stream-K GEMM schedule (RQLP_STREAMK=1, gemm_tma.cu) against the oracle GEMMs.
Runs in a subprocess because the schedule switch is read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch, sys
sys.path.insert(0, %(root)r)
import paper_1811_09334_b200 as rq, oracle
U = 2.0 ** -53
def cm(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()
for m, k, c in [(4096, 4096, 110), (2000, 2000, 125), (3000, 700, 300), (70000, 300, 40)]:
    rng = np.random.default_rng(m + k + c)
    A = rng.standard_normal((m, k)); X = rng.standard_normal((k, c)); V = rng.standard_normal((m, c))
    Y = rq.gemm_nn(cm(A), cm(X)).cpu().numpy()
    assert np.all(np.abs(Y - oracle.gemm_nn(A, X)) <= 64 * U * k * (np.abs(A) @ np.abs(X))), ("nn", m, k, c)
    for trans in (False, True):
        Z = rq.gemm_tn(cm(A), cm(V), trans_out=trans).cpu().numpy()
        ref = oracle.gemm_tn(A, V)
        bound = 64 * U * m * (np.abs(A).T @ np.abs(V))
        if trans:
            ref, bound = ref.T, bound.T
        assert np.all(np.abs(Z - ref) <= bound), ("tn", m, k, c, trans)
print("ok")
"""


def test_streamk_gemm_parity():
    if not __import__("torch").cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, RQLP_STREAMK="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
