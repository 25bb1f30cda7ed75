"""C5 at its OWN size (ERQLP, 1048576 x 16384 = 137 GB, l = 1056, q = 2, d = 2) on ONE B200.

BASELINE.json describes C5 as row-sharded over 8 GPUs; A plus the workspace (~175 GB) also fits the
192 GB of a single B200, so the single-GPU library path can run it whole.  The oracle cannot (its
full run would take hours), so the check is staged like tests/test_gpu_fullsize.py, using only
the outputs and the l x n stage output B (the m x l stage outputs Y, V do not fit beside A):

  * Omega bit-exact against the oracle's generator;
  * the oracle's own QLP tail on the GPU's B: pivots identical, L-values to relative 1e-10 on the
    sigma_j/sigma_1 >= 1e-8 mask, T / P element-wise;
  * Q = V Q_B with Q_B orthogonal gives V^T = Q_B Q^T, so sampled columns of the projection pass
    are recomputed as B[:, c] = Q_B^o (Q^T A[:, c]) with the oracle's Q_B and GEMM and compared
    with the GPU's B within the gamma_m bound;
  * properties at full size: ||Q^T Q - I||_max <= 1e-13 l, ||P^T P - I||_max, the eq. (3)
    identity ||A - Q T P^T||_F^2 = ||A||_F^2 - ||B||_F^2 (the library's residual kernel), and the
    library's own indicator (rqlp_get_indicator);
  * interlacing sigma_j(T) <= sigma_j(A) (+ noise bound).

  python tools/c5_full_check.py [--out gpurun_out/c5_full_1gpu_check.json]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
U = 2.0 ** -53


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5_full_1gpu_check.json"))
    args = ap.parse_args()
    import oracle
    import paper_1811_09334_b200 as rq
    from paper_1811_09334_b200 import build as rqbuild
    from synthetic import CONFIGS, make_A_config, sigma

    rqbuild.build()
    oracle.build()
    c = CONFIGS[args.workload]
    l, m, n = c.l, c.m, c.n
    rep = {"workload": c.name, "m": m, "n": n, "l": l, "q": c.q, "d": c.d, "gpu": torch.cuda.get_device_name(0),
           "gpu_mem_total_bytes": torch.cuda.get_device_properties(0).total_memory}

    def dump():
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(rep, f, indent=1)

    t0 = time.time()
    A = make_A_config(c, device="cuda")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    rep["gen_s"] = round(time.time() - t0, 2)
    h = rq.Handle()
    B = rq.cm_empty(l, n, A.device)
    h.set_stage_outputs(None, None, B)
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, seed=c.seed, handle=h)   # eager first call
    torch.cuda.synchronize()
    g = None
    t0 = time.time()
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, seed=c.seed, handle=h)
    torch.cuda.synchronize()
    rep["gpu_s"] = round(time.time() - t0, 3)
    rep["device_flags"] = h.sync()
    ind = h.indicator() if hasattr(h, "indicator") else None
    h.set_stage_outputs()
    rep["peak_mem_bytes"] = torch.cuda.max_memory_allocated()
    print(f"[c5_full] GPU factorisation {rep['gpu_s']} s, peak {rep['peak_mem_bytes'] / 1e9:.1f} GB", flush=True)
    dump()

    # 1. Omega bit-exact
    Om_o = oracle.omega(c.seed, n, l)
    Om_g = rq.omega(n, l, c.seed).cpu().numpy()
    rep["omega_bit_exact"] = bool(np.array_equal(Om_g.view(np.uint64), np.asarray(Om_o).view(np.uint64)))
    del Om_g, Om_o

    # 2. the oracle's tail on the GPU's B
    Bh = np.asfortranarray(B.cpu().numpy())
    t0 = time.time()
    o = oracle.qlp_tail(Bh, d=c.d)
    rep["oracle_tail_s"] = round(time.time() - t0, 1)
    T = np.asfortranarray(g["T"].cpu().numpy())
    P = np.asfortranarray(g["P"].cpu().numpy())
    rep["piv0_identical"] = bool(np.array_equal(g["piv0"].cpu().numpy(), o["piv0"]))
    rep["t_is_upper_same"] = bool(g["t_is_upper"] == o["t_is_upper"])
    r = c.rank if c.rank is not None else min(m, n)
    sig = sigma(c.spectrum, r).numpy()
    mask = sig[:l] / sig[0] >= 1e-8
    Lg, Lo = np.diag(T), np.diag(o["T"])
    rep["lvalue_rel_max"] = float((np.abs(Lg - Lo)[mask] / np.abs(Lo)[mask]).max())
    rep["dT_max_rel"] = float(np.abs(T - o["T"]).max() / np.abs(o["T"]).max())
    rep["dP_max"] = float(np.abs(P - o["PB"]).max())

    # 3. sampled columns of the projection pass: B[:, c] = Q_B (Q^T A[:, c])
    rng = np.random.default_rng(5)
    cols = np.sort(rng.choice(n, size=16, replace=False))
    cidx = torch.from_numpy(cols).to(A.device)
    A_c = np.asfortranarray(A[:, cidx].cpu().numpy())
    Qh = np.asfortranarray(g["Q"].cpu().numpy())
    QtA = oracle.gemm_tn(Qh, A_c)                       # l x 16
    B_o = oracle.gemm_nn(np.asfortranarray(o["QB"]), QtA)
    bound = 64 * U * (m + l) * (np.abs(o["QB"]) @ (np.abs(Qh).T @ np.abs(A_c)))
    ratio = np.abs(Bh[:, cols] - B_o) / bound
    rep["B_sampled_cols_max_ratio_to_bound"] = float(ratio.max())
    del Qh, A_c

    # 4. properties at full size
    Qg, Pg = g["Q"], g["P"]
    eye = torch.eye(l, dtype=torch.float64, device=A.device)
    rep["QtQ_minus_I_max"] = float((Qg.t() @ Qg - eye).abs().max())
    rep["PtP_minus_I_max"] = float((Pg.t() @ Pg - eye).abs().max())
    nA2 = 0.0
    for c0 in range(0, n, 1024):                        # column chunks: no m x n temporary
        blk = A[:, c0:c0 + 1024]
        nA2 += float((blk * blk).sum())
    nB2 = float((B * B).sum())
    res = rq.residual(A, g["Q"], g["T"], g["P"], handle=h)
    rep.update(normA2=nA2, normB2=nB2, residual_rel=res / math.sqrt(nA2),
               eq3_identity_relerr=abs(res ** 2 - (nA2 - nB2)) / nA2)
    if ind is not None:
        rep["library_indicator"] = ind
    noise2 = c.noise * (1.0 + math.sqrt(m / n)) * 1.5
    sL = np.linalg.svd(T, compute_uv=False)
    rep["interlacing_ok"] = bool(np.all(sL <= sig[:l] + noise2))
    rep["pass"] = bool(rep["omega_bit_exact"] and rep["piv0_identical"] and rep["t_is_upper_same"]
                       and rep["lvalue_rel_max"] <= 1e-10 and rep["dT_max_rel"] <= 1e-11 and rep["dP_max"] <= 1e-10
                       and rep["B_sampled_cols_max_ratio_to_bound"] <= 1.0
                       and rep["QtQ_minus_I_max"] <= 1e-13 * l and rep["PtP_minus_I_max"] <= 1e-13 * l
                       and rep["eq3_identity_relerr"] <= 1e-10 and rep["interlacing_ok"])
    dump()
    print(json.dumps(rep, indent=1), flush=True)
    return 0 if rep["pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
