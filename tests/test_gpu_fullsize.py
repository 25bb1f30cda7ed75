"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu).

C1, C2, C3: full GPU-vs-oracle parity (the oracle runs the whole factorisation).
C4 (BRQLP) and C5w (C5's per-GPU shape): the oracle cannot run the whole factorisation in a
test's time budget, so parity is staged: Ω bit-exact; sampled rows of the sketch Y = AΩ
recomputed by the oracle; the oracle's own QLP tail run on the GPU's B (pivots identical,
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


def _gpu_run(rq, c, A, stages=True):
    h = rq.Handle()
    Y = V = B = None
    if stages:
        Y, V = rq.cm_empty(c.m, c.l, A.device), rq.cm_empty(c.m, c.l, A.device)
        B = rq.cm_empty(c.l, c.n, A.device)
        h.set_stage_outputs(Y, V, B)
    g = rq.factorize(A, c.k, c.p, q=c.q, d=c.d, b=c.b, seed=c.seed, handle=h)
    torch.cuda.synchronize()
    g.update(Y=Y, V=V, B=B, flags=h.sync())
    h.set_stage_outputs()
    return g


def _check_full(orc, An, g, o, c, sig):
    l = c.l
    assert np.array_equal(g["piv0"].cpu().numpy(), o["piv0"]), "piv0 differ"
    if g["piv1"] is not None and c.d == 0:
        assert np.array_equal(g["piv1"].cpu().numpy(), o["piv1"]), "piv1 differ"
    Lg, Lo = np.diag(_np(g["T"])), np.diag(o["T"])
    mask = sig[:l] / sig[0] >= 1e-8
    rel = np.abs(Lg - Lo)[mask] / np.abs(Lo)[mask]
    assert rel.max() <= 1e-10, rel.max()
    Q, T, P = _np(g["Q"]), _np(g["T"]), _np(g["P"])
    nA = np.linalg.norm(An)
    rg = orc.residual(An, Q, T, P) / nA
    ro = orc.residual(An, o["Q"], o["T"], o["P"]) / nA
    assert abs(rg - ro) <= 1e-12, (rg, ro)
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 1e-13 * l
    return rg


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
    o = orc.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed)
    _check_full(orc, An, g, o, c, _sigma(c))


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
    _check_full(orc, An, g, o, c, _sigma(c))
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
    g = _gpu_run(rq, c, A)
    B = _staged(rq, orc, c, A, g)
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
    g = _gpu_run(rq, c, A)
    B = _staged(rq, orc, c, A, g)
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
        o = orc.brqlp(An, c.k, c.p, b=c.b, q=c.q, seed=c.seed)
    else:
        o = orc.rqlp(An, c.k, c.p, q=c.q, d=c.d, seed=c.seed)
    _check_full(orc, An, g, o, c, _sigma(c))
