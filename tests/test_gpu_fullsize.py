"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu).

C1, C2, C3: full GPU-vs-oracle parity (the oracle runs the whole factorisation).
C4 (BRQLP) and C5w (C5's per-GPU shape): the oracle cannot run the whole factorisation in a
test's time budget (the one full C4 run is tools/full_parity.py, committed under profiles/), so
parity is staged: Ω bit-exact; sampled rows / columns of EVERY A-pass recomputed by the oracle
from the GPU's own inputs -- the sketch Y = AΩ, each power step's Z = A^T V and Y = A W (BRQLP:
per block, with the implicit deflation terms), B = V^T A / each deflated B_j; the oracle's own
QLP tail run on the GPU's B (pivots identical,
L-values relative 1e-10, Q_B/P_B/T elementwise); properties that hold at any size (QᵀQ = I,
eq. (3)/(21) residual identity, interlacing); plus full oracle parity on a reduced-m shape of
the same config.  Tolerances: BASELINE.json north_star (see tests/test_gpu_parity.py).
"""
import dataclasses
import math
import time

import numpy as np
import pytest
import torch
from parity import check_factorization

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def rq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1811_09334_b200 as rq
    return rq


def _np(t):
    return np.asfortranarray(t.detach().cpu().numpy())


def _gpu_run(rq, c, A, stages=True, power_stages=False):
    h = rq.Handle()
    Y = V = B = None
    if stages:
        Y, V = rq.cm_empty(c.m, c.l, A.device), rq.cm_empty(c.m, c.l, A.device)
        B = rq.cm_empty(c.l, c.n, A.device)
        h.set_stage_outputs(Y, V, B)
    ps = {}
    if power_stages and c.q > 0:
        ql = c.q * c.l
        ps = dict(Vpre=rq.cm_empty(c.m, ql, A.device), Z=rq.cm_empty(c.n, ql, A.device),
                  W=rq.cm_empty(c.n, ql, A.device), Ypow=rq.cm_empty(c.m, ql, A.device))
        h.set_power_stage_outputs(**ps)
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
    torch.cuda.synchronize()
    g.update(Y=Y, V=V, B=B, flags=h.sync(), **ps)
    h.set_stage_outputs()
    h.set_power_stage_outputs()
    return g


def _check_full(orc, An, g, o, c, sig, B_oracle=None):
    if c.d:
        o = dict(o, piv1=None)
    rec = check_factorization(orc, An, g, o, c.l, sig_ratio=sig[:c.l] / sig[0], block=c.b, B_oracle=B_oracle,
                              tag=f"full {c.name} m={c.m}")
    return rec["res_gpu"]


def _within(x, ref, bound, what):
    bad = np.abs(x - ref) > bound
    assert not bad.any(), f"{what}: {bad.sum()} entries off, max ratio {(np.abs(x - ref) / bound).max():.3g}"


def _staged_power_rqlp(orc, c, A, g, rows, cols):
    """Every power-step A-pass of RQLP/ERQLP at sampled rows / columns, recomputed by the oracle from
    the GPU's own inputs: Z = A^T V (sampled columns of A) and Y = A W (sampled rows)."""
    l, m, n = c.l, c.m, c.n
    ridx, cidx = torch.from_numpy(rows).to(A.device), torch.from_numpy(cols).to(A.device)
    A_r, A_c = _np(A[ridx, :]), _np(A[:, cidx])
    for it in range(c.q):
        s = slice(it * l, (it + 1) * l)
        Vp = _np(g["Vpre"][:, s])
        Z_g = _np(g["Z"][cidx, s])                       # rows of Z = columns of A
        Z_o = orc.gemm_tn(A_c, Vp)
        _within(Z_g, Z_o, 64 * U * m * (np.abs(A_c).T @ np.abs(Vp)), f"power {it} Z = A^T V")
        W = _np(g["W"][:, s])
        Y_g = _np(g["Ypow"][ridx, s])
        Y_o = orc.gemm_nn(A_r, W)
        _within(Y_g, Y_o, 64 * U * n * (np.abs(A_r) @ np.abs(W)), f"power {it} Y = A W")


def _staged_blocks_brqlp(orc, c, A, g, rows, cols):
    """Every per-block A-pass of BRQLP at sampled rows / columns, recomputed by the oracle from the
    GPU's own inputs with the implicit deflation written out (exact-arithmetic eq. (19)):
      Z_j = A^T V_j - B_<j^T (V_<j^T V_j),   Y_j = A W_j - V_<j (B_<j W_j),
      B_j = V_j^T A - (V_j^T V_<j) B_<j."""
    l, b, m, n = c.l, c.b, c.m, c.n
    ridx, cidx = torch.from_numpy(rows).to(A.device), torch.from_numpy(cols).to(A.device)
    A_r, A_c = _np(A[ridx, :]), _np(A[:, cidx])
    Vf = _np(g["V"])
    Bf = _np(g["B"])
    Vf_r = Vf[rows]
    for c0 in range(0, l, b):
        bj = min(b, l - c0)
        s = slice(c0, c0 + bj)
        Vl, Bl = Vf[:, :c0], Bf[:c0]
        Bl_c = Bl[:, cols]
        for it in range(c.q):
            si = slice(it * l + c0, it * l + c0 + bj)
            Vp = _np(g["Vpre"][:, si])
            Z_g = _np(g["Z"][cidx, si])
            Z_o = orc.gemm_tn(A_c, Vp)
            bound = m * (np.abs(A_c).T @ np.abs(Vp))
            if c0:
                C = orc.gemm_tn(Vl, Vp)
                Z_o = Z_o - orc.gemm_tn(Bl_c, C)
                bound = bound + c0 * (np.abs(Bl_c).T @ np.abs(C)) + m * (np.abs(Bl_c).T @ (np.abs(Vl).T @ np.abs(Vp)))
            _within(Z_g, Z_o, 64 * U * bound, f"block {c0 // b} power {it} Z")
            W = _np(g["W"][:, si])
            Y_g = _np(g["Ypow"][ridx, si])
            Y_o = orc.gemm_nn(A_r, W)
            bound = n * (np.abs(A_r) @ np.abs(W))
            if c0:
                D = orc.gemm_nn(Bl, W)
                Y_o = Y_o - orc.gemm_nn(Vf_r[:, :c0], D)
                bound = bound + c0 * (np.abs(Vf_r[:, :c0]) @ np.abs(D)) + n * (np.abs(Vf_r[:, :c0]) @ (np.abs(Bl) @ np.abs(W)))
            _within(Y_g, Y_o, 64 * U * bound, f"block {c0 // b} power {it} Y")
        Vj = Vf[:, s]
        Bj_g = Bf[s][:, cols]
        Bj_o = orc.gemm_tn(Vj, A_c)
        bound = m * (np.abs(Vj).T @ np.abs(A_c))
        if c0:
            E = orc.gemm_tn(Vj, Vl)
            Bj_o = Bj_o - orc.gemm_nn(E, Bl_c)
            bound = bound + c0 * (np.abs(E) @ np.abs(Bl_c)) + m * ((np.abs(Vj).T @ np.abs(Vl)) @ np.abs(Bl_c))
        _within(Bj_g, Bj_o, 64 * U * bound, f"block {c0 // b} B_j")


def _sigma(c):
    from synthetic import sigma
    r = c.rank if c.rank is not None else min(c.m, c.n)
    return sigma(c.spectrum, r).numpy()


@pytest.mark.parametrize("name", ["c1", "c1e", "c2"])
def test_full_parity_small_configs(rq, orc, name):
    from synthetic import CONFIGS, make_A_config
    c = CONFIGS[name]
    A = make_A_config(c, device="cuda")
    g = _gpu_run(rq, c, A, stages=False)
    An = _np(A)
    o = orc.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed, stages=True)
    _check_full(orc, An, g, o, c, _sigma(c), B_oracle=o["B"])


def test_full_parity_c3(rq, orc):
    """C3 full size (65536 x 8192, l = 272, q = 2, d = 2): the oracle runs the whole thing."""
    from synthetic import CONFIGS, make_A_config
    c = CONFIGS["c3"]
    A = make_A_config(c, device="cuda")
    g = _gpu_run(rq, c, A)
    An = _np(A)
    t0 = time.time()
    o = orc.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed, stages=True)
    print(f"oracle C3 {time.time() - t0:.1f}s")
    _check_full(orc, An, g, o, c, _sigma(c), B_oracle=o["B"])
    # stage parity: V spans the same space with the same unique basis (R_ii > 0)
    assert np.abs(_np(g["V"]) - o["V"]).max() <= 1e-11
    assert np.abs(_np(g["B"]) - o["B"]).max() <= 1e-11 * np.abs(o["B"]).max()


def _staged(rq, orc, c, A, g, n_rows=256, tail_d=None):
    """Staged parity at full size (shared by C4 and C5w)."""
    l, m, n = c.l, c.m, c.n
    # 1. Ω bit-exact
    Om_g = _np(rq.omega(n, l, c.seed))
    Om_o = orc.omega(c.seed, n, l)
    assert np.array_equal(Om_g.view(np.uint64), Om_o.view(np.uint64))
    # 2. sampled rows of the sketch Y = AΩ (the production A-pass)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(m, size=n_rows, replace=False))
    idx = torch.from_numpy(rows).to(A.device)
    A_s = _np(A[idx, :])
    Y_o = orc.gemm_nn(A_s, Om_o)
    Y_g = _np(g["Y"][idx, :])
    bound = 64 * U * n * (np.abs(A_s) @ np.abs(Om_o))
    assert np.all(np.abs(Y_g - Y_o) <= bound)
    # 3. sampled columns of the projection pass B = V^T A (RQLP/ERQLP: B is exactly V^T A;
    #    BRQLP's B_j carries the deflation terms, checked through eq. (21) by the callers)
    B = _np(g["B"])
    if c.b is None:
        cols = np.sort(rng.choice(n, size=32, replace=False))
        cidx = torch.from_numpy(cols).to(A.device)
        V_h, A_c = _np(g["V"]), _np(A[:, cidx])
        B_o = orc.gemm_tn(V_h, A_c)
        bound = 64 * U * m * (np.abs(V_h).T @ np.abs(A_c))
        assert np.all(np.abs(B[:, cols] - B_o) <= bound)
    # 4. (callers) the oracle's tail on the GPU's B: pivots, L-values, T, Q_B, P_B
    return B


def test_staged_parity_c5w(rq, orc):
    """C5's per-GPU shape (131072 x 16384, l = 1056, q = 2, d = 2) in bench.py's configuration."""
    from synthetic import CONFIGS, make_A_config
    c = CONFIGS["c5w"]
    A = make_A_config(c, device="cuda")
    g = _gpu_run(rq, c, A, power_stages=True)
    B = _staged(rq, orc, c, A, g)
    rng = np.random.default_rng(2)
    _staged_power_rqlp(orc, c, A, g, np.sort(rng.choice(c.m, 256, replace=False)),
                       np.sort(rng.choice(c.n, 32, replace=False)))
    t0 = time.time()
    o = orc.qlp_tail(B, d=c.d)
    print(f"oracle C5w tail {time.time() - t0:.1f}s")
    l = c.l
    assert np.array_equal(g["piv0"].cpu().numpy(), o["piv0"])
    assert g["t_is_upper"] == o["t_is_upper"]
    T = _np(g["T"])
    sig = _sigma(c)
    mask = sig[:l] / sig[0] >= 1e-8
    rel = np.abs(np.diag(T) - np.diag(o["T"]))[mask] / np.abs(np.diag(o["T"]))[mask]
    assert rel.max() <= 1e-10, rel.max()
    assert np.abs(T - o["T"]).max() <= 1e-11 * np.abs(o["T"]).max()
    assert np.abs(_np(g["P"]) - o["PB"]).max() <= 1e-10
    # Q = V Q_B with the oracle's Q_B on sampled rows
    rng = np.random.default_rng(1)
    rows = torch.from_numpy(np.sort(rng.choice(c.m, size=512, replace=False))).to(A.device)
    Qs = _np(g["Q"][rows, :])
    assert np.abs(Qs - _np(g["V"][rows, :]) @ o["QB"]).max() <= 1e-11
    # properties at full size: orthonormality, eq. (3) residual identity (GPU residual kernel)
    Qg, Vg = g["Q"], g["V"]
    eye = torch.eye(l, dtype=torch.float64, device=A.device)
    assert (Qg.t() @ Qg - eye).abs().max().item() <= 1e-13 * l
    assert (Vg.t() @ Vg - eye).abs().max().item() <= 1e-13 * l
    res = rq.residual(A, g["Q"], g["T"], g["P"])
    nA2 = float((A * A).sum().item())
    nB2 = float((g["B"] * g["B"]).sum().item())
    assert abs(res ** 2 - (nA2 - nB2)) <= 1e-10 * nA2
    # interlacing (Lemma): sigma_j(L) <= sigma_j(A) <= sigma_j + ||noise||_2 (Weyl);
    # ||c G||_2 <= c (1 + sqrt(m/n)) (1 + slack) for G_ij ~ N(0, 1/n)
    noise2 = c.noise * (1.0 + math.sqrt(c.m / c.n)) * 1.5
    sL = np.linalg.svd(T, compute_uv=False)
    assert np.all(sL <= sig[:l] + noise2)


def test_staged_parity_c4_brqlp(rq, orc):
    """C4 (BRQLP, 262144 x 16384, l = 528, b = 64 -> 8 blocks of 64 + a ragged 16, q = 1)."""
    from synthetic import CONFIGS, make_A_config
    c = CONFIGS["c4"]
    A = make_A_config(c, device="cuda")
    g = _gpu_run(rq, c, A, power_stages=True)
    B = _staged(rq, orc, c, A, g)
    rng = np.random.default_rng(3)
    _staged_blocks_brqlp(orc, c, A, g, np.sort(rng.choice(c.m, 256, replace=False)),
                         np.sort(rng.choice(c.n, 32, replace=False)))
    l, b = c.l, c.b
    T = _np(g["T"])
    P = _np(g["P"])
    piv0, piv1 = g["piv0"].cpu().numpy(), g["piv1"].cpu().numpy()
    nblk = -(-l // b)
    for j in range(nblk):
        c0, c1 = j * b, min(l, (j + 1) * b)
        o = orc.qlp_tail(B[c0:c1], d=0)            # Alg.3 l.8 on the GPU's B_j
        assert np.array_equal(piv0[c0:c1], o["piv0"]), f"block {j} piv0"
        assert np.array_equal(piv1[c0:c1], o["piv1"]), f"block {j} piv1"
        Lo = o["T"]
        np.testing.assert_allclose(np.diag(T)[c0:c1], np.diag(Lo), rtol=1e-10)
        assert np.abs(T[c0:c1, c0:c1] - Lo).max() <= 1e-11 * np.abs(Lo).max()
        assert np.abs(P[:, c0:c1] - o["PB"]).max() <= 1e-10
        off = T[c0:c1].copy()
        off[:, c0:c1] = 0
        assert not off.any()
    Qg, Vg = g["Q"], g["V"]
    eye = torch.eye(l, dtype=torch.float64, device=A.device)
    assert (Qg.t() @ Qg - eye).abs().max().item() <= 1e-13 * l   # cross-block orthogonality (eq. (18))
    res = rq.residual(A, g["Q"], g["T"], g["P"])
    nA2 = float((A * A).sum().item())
    nB2 = float((g["B"] * g["B"]).sum().item())
    assert abs(res ** 2 - (nA2 - nB2)) <= 1e-10 * nA2               # eq. (21): A - QLP^T = A - VV^T A


@pytest.mark.parametrize("name,m", [("c4", 8192), ("c5w", 4096)])
def test_full_parity_reduced_m(rq, orc, name, m):
    """The C4 / C5 configuration (n, k, p, q, d, b, spectrum) at a reduced row count the oracle
    finishes in seconds: full parity including BRQLP's explicit-vs-implicit deflation."""
    from synthetic import CONFIGS, make_A_config
    c = dataclasses.replace(CONFIGS[name], m=m)
    A = make_A_config(c, device="cuda")
    g = _gpu_run(rq, c, A, stages=False)
    An = _np(A)
    if c.b is not None:
        o = orc.brqlp(An, c.k, c.p, b=c.b, q=c.q, seed=c.seed, stages=True)
        B_o = o["V"].T @ An
    else:
        o = orc.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed, stages=True)
        B_o = o["B"]
    _check_full(orc, An, g, o, c, _sigma(c), B_oracle=B_o)
