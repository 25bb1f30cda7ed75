"""Full-size end-to-end parity of one BASELINE.json config against the CPU oracle.

The GPU factorises the full synthetic A through the C ABI (the bench's launch configuration); the
oracle (oracle/, plain C + OpenMP, explicit eq. (19) deflation for BRQLP) factorises the same bytes
on the host cores.  Graded at BASELINE.json north_star's tolerances: identical pivot sequences,
L-values relative 1e-10 where sigma_j/sigma_1 >= 1e-8, |Δ residual| <= 1e-12 (relative to ||A||_F),
||Q^T Q - I||_max <= 1e-13 l; element-wise Q, P, T differences and the oracle's wall time are
reported.  The residuals ||A - Q T P^T||_F of both factorisations are evaluated with plain torch
matmuls (cuBLAS) on the GPU in row chunks -- test infrastructure, not the product path.

  python tools/full_parity.py --workload c4 [--out gpurun_out/c4_full_parity.json]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def residual_torch(A, Q, T, P, chunk=16384) -> float:
    """||A - Q T P^T||_F with plain torch matmuls, row chunks (never forms m x n)."""
    M = T @ P.t()
    s = torch.zeros((), dtype=torch.float64, device=A.device)
    for r0 in range(0, A.shape[0], chunk):
        r1 = min(A.shape[0], r0 + chunk)
        R = A[r0:r1] - Q[r0:r1] @ M
        s += (R * R).sum()
    return float(s.sqrt())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import oracle
    import paper_1811_09334_b200 as rq
    from paper_1811_09334_b200 import build as rqbuild
    from synthetic import CONFIGS, make_A_config, sigma

    rqbuild.build()
    oracle.build()
    c = CONFIGS[args.workload]
    out_path = args.out or os.path.join(ROOT, "gpurun_out", f"{c.name}_full_parity.json")
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    rep = {"workload": c.name, "m": c.m, "n": c.n, "k": c.k, "p": c.p, "l": c.l, "q": c.q, "d": c.d, "b": c.b,
           "cpu_model": cpu_model(), "oracle_threads": oracle.num_threads()}

    def dump():
        with open(out_path, "w") as f:
            json.dump(rep, f, indent=1)

    t0 = time.time()
    A = make_A_config(c, device="cuda")
    torch.cuda.synchronize()
    rep["gen_s"] = time.time() - t0
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed)
    torch.cuda.synchronize()
    t0 = time.time()
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed)
    torch.cuda.synchronize()
    rep["gpu_s"] = time.time() - t0
    print(f"[full_parity] GPU {c.name} done in {rep['gpu_s']:.3f}s", flush=True)
    An = A.cpu().numpy()          # column-major (Fortran) host copy of the same bytes
    assert An.flags.f_contiguous
    dump()
    t0 = time.time()
    if c.b is not None:
        o = oracle.brqlp(An, c.k, c.p, b=c.b, q=c.q, seed=c.seed)
    else:
        o = oracle.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed)
    rep["oracle_s"] = time.time() - t0
    print(f"[full_parity] oracle {c.name} done in {rep['oracle_s']:.1f}s", flush=True)
    del An
    l = c.l
    dev = A.device
    Qo, To, Po = (torch.from_numpy(np.ascontiguousarray(o[k].T)).to(dev).t() for k in ("Q", "T", "P"))
    Qg, Tg, Pg = g["Q"], g["T"], g["P"]
    rep["piv0_identical"] = bool(np.array_equal(g["piv0"].cpu().numpy(), o["piv0"]))
    if g.get("piv1") is not None and c.d == 0:
        rep["piv1_identical"] = bool(np.array_equal(g["piv1"].cpu().numpy(), o["piv1"]))
    if not rep["piv0_identical"]:
        pg = g["piv0"].cpu().numpy()
        rep["first_piv_diff"] = int(np.argmax(pg != o["piv0"]))
    r = c.rank if c.rank is not None else min(c.m, c.n)
    sig = sigma(c.spectrum, r).numpy()
    mask = sig[:l] / sig[0] >= 1e-8
    Lg, Lo = np.diag(Tg.cpu().numpy()), np.diag(o["T"])
    rel = np.abs(Lg - Lo)[mask] / np.abs(Lo)[mask]
    rep["lvalue_rel_max"] = float(rel.max())
    nA = float(torch.linalg.norm(A))
    rg = residual_torch(A, Qg, Tg, Pg) / nA
    ro = residual_torch(A, Qo, To, Po) / nA
    rep.update(residual_gpu=rg, residual_oracle=ro, residual_absdiff=abs(rg - ro))
    I = torch.eye(l, dtype=torch.float64, device=dev)
    rep["QtQ_minus_I_max"] = float((Qg.t() @ Qg - I).abs().max())
    rep["dQ_max"] = float((Qg - Qo).abs().max())
    rep["dP_max"] = float((Pg - Po).abs().max())
    rep["dT_max_rel"] = float((Tg - To).abs().max() / To.abs().max())
    if c.b is not None:   # BRQLP: P orthonormal within each block (reading R17)
        dev_b = 0.0
        for c0 in range(0, l, c.b):
            Pb = Pg[:, c0:c0 + c.b]
            dev_b = max(dev_b, float((Pb.t() @ Pb - torch.eye(Pb.shape[1], dtype=torch.float64, device=dev)).abs().max()))
        rep["PtP_minus_I_max_per_block"] = dev_b
    else:
        rep["PtP_minus_I_max"] = float((Pg.t() @ Pg - I).abs().max())
    rep["pass"] = bool(rep["piv0_identical"] and rep.get("piv1_identical", True) and rep["lvalue_rel_max"] <= 1e-10
                       and rep["residual_absdiff"] <= 1e-12 and rep["QtQ_minus_I_max"] <= 1e-13 * l)
    dump()
    print(json.dumps(rep, indent=1), flush=True)
    return 0 if rep["pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
