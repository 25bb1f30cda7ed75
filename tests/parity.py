"""GPU-vs-oracle comparison of whole factorisations at BASELINE.json north_star's tolerances
(DESIGN.md §6 states every bound used here and the readings R29/R30 behind the two that are not
north_star's literal numbers).

  * pivot sequences identical -- or, at the first differing step s, the two chosen columns'
    residual norms ‖(I - P_s) b_i‖ (P_s = projector on the first s pivot columns of the oracle's
    B) agree to TIE_REL relative: a numerical near-tie, where both choices are correct to working
    precision (reading R30); the pivot-dependent comparisons (L-values, element-wise factors) are
    then skipped (RQLP/ERQLP) or stop before the tied block (BRQLP), the basis-invariant ones stay;
  * L-values: |ΔL_j| <= max(1e-10 |L_j|, C_L u |L_1|) for every j with σ_j/σ_1 >= 1e-8 -- the
    north_star's relative 1e-10 wherever FP64 can deliver it; below |L_j| ~ C_L u |L_1| / 1e-10
    the achievable agreement of two FP64 computations is absolute (reading R29);
  * |‖A−QTPᵀ‖_F − ‖A−Q_oT_oP_oᵀ‖_F| / ‖A‖_F <= 1e-12;  ‖QᵀQ − I‖_max <= 1e-13 l;
    ‖PᵀP − I‖_max <= 1e-13 l (per block for BRQLP, reading R17);
  * element-wise (Q, T, P are unique given the pivots, reading R3): column j of Q within
    C_Q u |L_1|/|L_j|, of P within C_P u |L_1|/|L_j|, T within C_T u |L_1| (perturbation of the
    j-th pivoted-QR direction ~ u ‖B‖ / |R_jj|).

RQLP_PARITY_LOG=<file> appends one JSON record per comparison with the normalised errors (the
calibration data of DESIGN.md §6).
"""
from __future__ import annotations

import json
import os

import numpy as np

U = 2.0 ** -53
# Constants calibrated on the whole -m gpu suite (RQLP_PARITY_LOG): largest measured
# normalised errors 41 (L), 1830 (Q), 14 (P), 41 (T); each bound leaves a margin of >= 1.5x.
TIE_REL = 1e-8       # R30: downdated-norm agreement of two FP64 CPQRs (LAPACK recompute at sqrt(u))
C_L = 64.0           # R29: |ΔL_j| floor in units of u |L_1|
C_Q = 4096.0         # column j of Q: C_Q u |L_1| / |L_j|
C_P = 256.0          # column j of P: C_P u |L_1| / |L_j|
C_T = 128.0          # T entries: C_T u |L_1|


def _np(t):
    return np.asfortranarray(t.detach().cpu().numpy()) if hasattr(t, "detach") else np.asarray(t)


def residual_norms_at_step(B: np.ndarray, piv: np.ndarray, s: int) -> np.ndarray:
    """‖(I − P_s) b_i‖ for every column i of B after s pivot steps (exact-arithmetic downdated
    norms; P_s projects on span(B[:, piv[:s]]))."""
    if s == 0:
        return np.linalg.norm(B, axis=0)
    Qs, _ = np.linalg.qr(B[:, piv[:s]])
    Rm = B - Qs @ (Qs.T @ B)
    return np.linalg.norm(Rm, axis=0)


def first_pivot_diff(pg, po, B=None, tag=""):
    """Index of the first differing pivot (None if identical).  Raises AssertionError unless the
    flip is a near-tie of the oracle's B (reading R30)."""
    pg, po = np.asarray(pg), np.asarray(po)
    if np.array_equal(pg, po):
        return None
    s = int(np.argmax(pg != po))
    assert B is not None, f"{tag}: pivot sequences differ from step {s} (no B to judge a near-tie)"
    r = residual_norms_at_step(np.asarray(B), po, s)
    rg, ro = r[pg[s]], r[po[s]]
    gap = abs(rg - ro) / max(ro, 1e-300)
    assert gap <= TIE_REL, f"{tag}: pivot {s} differs ({pg[s]} vs {po[s]}): norms {rg!r} vs {ro!r} rel {gap:.2e}"
    return s


def _log(rec):
    path = os.environ.get("RQLP_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def check_factorization(orc, A, g, o, l, sig_ratio=None, block=None, B_oracle=None, tag="", elementwise=True,
                        residual_slack=False):
    """Compare the GPU factorisation g (dict of tensors) with the oracle's o (dict of numpy arrays)
    on the same A.  block = BRQLP block size (P orthonormal per block; per-block pivots).
    B_oracle = the oracle's projected B (l x n) for the near-tie rule.  residual_slack: a
    numerically rank-deficient sketch (reading R4) -- the completion directions differ, so the
    GPU residual may exceed the oracle's by up to 2x.  Returns the records logged."""
    An = np.linalg.norm(A)
    Q, T, P = _np(g["Q"]), _np(g["T"]), _np(g["P"])
    pg = _np(g["piv0"])
    # ---- pivots (piv0: CPQR of B; piv1: CPQR of R0^T) -----------------------------------------
    s_tie = None
    if block is None:
        s_tie = first_pivot_diff(pg, o["piv0"], B_oracle, tag)
        if s_tie is None and g.get("piv1") is not None and o.get("piv1") is not None:
            assert np.array_equal(_np(g["piv1"]), o["piv1"]), f"{tag}: piv1 differ"
    else:
        for c0 in range(0, l, block):
            c1 = min(l, c0 + block)
            Bj = None if B_oracle is None else B_oracle[c0:c1]
            s = first_pivot_diff(pg[c0:c1], o["piv0"][c0:c1], Bj, f"{tag} block {c0 // block}")
            if s is not None:
                s_tie = c0      # the tied block's L_j, Q_j, P_j are not comparable (earlier blocks are)
                break
            if g.get("piv1") is not None and o.get("piv1") is not None:
                assert np.array_equal(_np(g["piv1"])[c0:c1], o["piv1"][c0:c1]), f"{tag}: piv1 block {c0 // block}"
    # pivot-dependent comparisons: everything when the pivots agree; after a near-tie in CPQR(B)
    # the second factorisation mixes every row of R0, so nothing (RQLP/ERQLP) or only the blocks
    # before the tied one (BRQLP: V_j does not depend on earlier blocks' pivots)
    jmax = l if s_tie is None else (s_tie if block is not None else 0)
    # ---- L-values -----------------------------------------------------------------------------
    Lg, Lo = np.abs(np.diag(T)), np.abs(np.diag(o["T"]))
    mask = np.ones(l, bool) if sig_ratio is None else np.asarray(sig_ratio)[:l] >= 1e-8
    mask[jmax:] = False
    L1 = max(Lo.max(), 1e-300)
    dL = np.abs(Lg - Lo)
    rec = {"tag": tag, "l": l, "tie_step": s_tie}
    if mask.any():
        tolL = np.maximum(1e-10 * Lo, C_L * U * L1)
        rec["L_rel_max"] = float((dL[mask] / np.maximum(Lo[mask], 1e-300)).max())
        rec["L_abs_over_uL1"] = float((dL[mask] / (U * L1)).max())
        if not os.environ.get("RQLP_PARITY_CALIBRATE"):
            assert np.all(dL[mask] <= tolL[mask]), (tag, "L-values", rec)
    # ---- basis-invariant quantities ------------------------------------------------------------
    rg = orc.residual(A, Q, T, P) / An if An > 0 else 0.0
    ro = orc.residual(A, o["Q"], o["T"], o["P"]) / An if An > 0 else 0.0
    rec.update(res_gpu=rg, res_orc=ro)
    if residual_slack:
        assert abs(rg - ro) <= 1e-12 or rg <= 2 * ro + 1e-14, (tag, rg, ro)
    else:
        assert abs(rg - ro) <= 1e-12, (tag, rg, ro)
    lq = Q.shape[1]
    qd = np.abs(Q.T @ Q - np.eye(lq)).max()
    rec["QtQ"] = float(qd)
    assert qd <= 1e-13 * lq, (tag, "QtQ", qd)
    if block is None:
        pd = np.abs(P.T @ P - np.eye(lq)).max()
    else:
        pd = max(np.abs(P[:, c0:c0 + block].T @ P[:, c0:c0 + block] - np.eye(min(block, lq - c0))).max()
                 for c0 in range(0, lq, block))
    rec["PtP"] = float(pd)
    assert pd <= 1e-13 * lq, (tag, "PtP", pd)
    # ---- element-wise Q, P, T (unique given the pivots, R3) -----------------------------------
    if elementwise and jmax > 0:
        scale = U * L1 / np.maximum(Lo[:jmax], U * L1)          # u |L_1| / |L_j|, capped at 1
        dQ = np.abs(Q[:, :jmax] - o["Q"][:, :jmax]).max(axis=0)
        dP = np.abs(P[:, :jmax] - o["P"][:, :jmax]).max(axis=0)
        rec["Q_over"] = float((dQ / scale).max())
        rec["P_over"] = float((dP / scale).max())
        rec["dQ_max"], rec["dP_max"] = float(dQ.max()), float(dP.max())
        dT = np.abs(T[:jmax, :jmax] - o["T"][:jmax, :jmax]).max()
        rec["T_over"] = float(dT / (U * L1))
        if not os.environ.get("RQLP_PARITY_CALIBRATE"):
            assert rec["Q_over"] <= C_Q, (tag, "Q elementwise", rec)
            assert rec["P_over"] <= C_P, (tag, "P elementwise", rec)
            assert rec["T_over"] <= C_T, (tag, "T elementwise", rec)
    _log(rec)
    return rec
