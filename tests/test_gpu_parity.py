"""GPU-vs-oracle parity through the C ABI (librqlp.so).  All tests need a B200 (-m gpu).

Tolerances are BASELINE.json north_star's: identical pivots; L-values relative 1e-10 for
σ_j/σ_1 >= 1e-8; residual ‖A−QLPᵀ‖_F/‖A‖_F within 1e-12 absolute; ‖QᵀQ−I‖_max <= 1e-13·l.
Per-stage GEMM tolerances: |ΔY_ij| <= 64 u k (|A||X|)_ij.
"""
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
    rq.lib()
    return rq


def _cm(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda().t()


def _np(t: torch.Tensor) -> np.ndarray:
    return np.asfortranarray(t.detach().cpu().numpy())


def _rand_svd(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    U_, _ = np.linalg.qr(rng.standard_normal((m, len(sig))))
    V_, _ = np.linalg.qr(rng.standard_normal((n, len(sig))))
    return np.asfortranarray((U_ * sig) @ V_.T)


# ------------------------------------------------------------------ stages
@pytest.mark.parametrize("n,l,seed", [(800, 25, 1), (4097, 110, 2), (1, 1, 0), (33, 7, 2**64 - 1), (1029, 138, 77)])
def test_omega_bit_exact(rq, orc, n, l, seed):
    Om = _np(rq.omega(n, l, seed))
    ref = orc.omega(seed, n, l)
    assert np.array_equal(Om.view(np.uint64), ref.view(np.uint64))


# (2000, 3000, 40), (4100, 4100, 110), (2500, 2600, 200): fewer output tiles than SMs and many
# k-tiles -> the balanced split (equal runs of (tile, k-tile) units per CTA, ragged at both ends)
# (40000, 300, 64), (38001, 1000, 48), (37900, 70, 33): >= 296 output tiles of width 32..64 -> two
# CTAs per SM (3-stage rings), ragged rows / columns; (6000, 21000, 64): few tiles, many k-tiles ->
# the two-CTA split-K / balanced split
@pytest.mark.parametrize("m,k,c", [(1000, 800, 25), (1031, 1030, 110), (4133, 1029, 138), (517, 93, 17), (64, 64, 64),
                                   (3, 5, 2), (2000, 3000, 40), (4100, 4100, 110), (2500, 2600, 200),
                                   (40000, 300, 64), (38001, 1000, 48), (37900, 70, 33), (6000, 21000, 64)])
def test_gemm_nn_parity(rq, orc, m, k, c):
    rng = np.random.default_rng(m + k + c)
    A, X = rng.standard_normal((m, k)), rng.standard_normal((k, c))
    Y = _np(rq.gemm_nn(_cm(A), _cm(X)))
    ref = orc.gemm_nn(A, X)
    bound = 64 * U * k * (np.abs(A) @ np.abs(X))
    assert np.all(np.abs(Y - ref) <= bound)


@pytest.mark.parametrize("m,k,c,trans", [(1000, 800, 25, True), (1031, 1030, 110, False), (4133, 1029, 138, True),
                                         (517, 93, 17, False), (5, 3, 2, True), (3000, 2000, 40, True),
                                         (4100, 4100, 110, False), (4100, 4100, 110, True), (2600, 2500, 200, False),
                                         (70001, 4000, 48, True), (64000, 2000, 64, False), (50000, 300, 64, True)])
def test_gemm_tn_parity(rq, orc, m, k, c, trans):
    rng = np.random.default_rng(m * 3 + k + c)
    A, V = rng.standard_normal((m, k)), rng.standard_normal((m, c))
    Z = _np(rq.gemm_tn(_cm(A), _cm(V), trans_out=trans))
    ref = orc.gemm_tn(A, V)
    if trans:
        ref = ref.T
    bound = 64 * U * m * (np.abs(A).T @ np.abs(V))
    if trans:
        bound = bound.T
    assert np.all(np.abs(Z - ref) <= bound)


@pytest.mark.parametrize("m,c,cond", [(1000, 25, 1e2), (4133, 138, 1e4), (2000, 300, 1e5), (777, 129, 1e9)])
def test_orth_matches_householder(rq, orc, m, c, cond):
    """CholeskyQR2 (+ shifted pass when cond(Y) is large) reproduces the unique thin Q, R of
    Householder QR with R_ii >= 0 (reading R3)."""
    Y = _rand_svd(m, c, np.logspace(0, -np.log10(cond), c), m + c)
    V, R = rq.orth(_cm(Y), return_r=True)
    V, R = _np(V), _np(R)
    Qo, Ro = orc.hqr(Y)
    assert np.abs(V.T @ V - np.eye(c)).max() <= 1e-13 * c
    tol = 1e-15 * cond * c
    assert np.abs(V - Qo).max() <= max(tol, 1e-13)
    assert np.abs(R - Ro).max() <= max(tol, 1e-13) * np.abs(Ro).max()


_RESCUE_SPECTRA = {
    "graded1e-20": lambda c: np.logspace(0, -20, c),
    "graded1e-39": lambda c: np.logspace(0, -39, c),
    "rank_half": lambda c: np.r_[np.ones(c - c // 2), np.zeros(c // 2)],
    "gap1e-9": lambda c: np.r_[np.ones(c - c // 3), 1e-9 * np.ones(c // 3)],
    "one_big": lambda c: np.r_[np.ones(1), 1e-12 * np.ones(c - 1)],
    "zero": lambda c: np.zeros(c),
}


@pytest.mark.parametrize("spec", sorted(_RESCUE_SPECTRA))
@pytest.mark.parametrize("m,c", [(400, 16), (5000, 110), (3000, 200)])
def test_orth_rescue(rq, orc, spec, m, c):
    """cond(Y) far beyond CholeskyQR2's reach (or rank(Y) < c): CholeskyQR2 breaks down and the
    rescue kernel's shifted passes must still return V with orthonormal columns and Y = V R to
    O(u ||Y||), R upper triangular -- what Householder QR guarantees for any Y (the oracle's hqr:
    the same bounds hold for it, checked alongside).  c = 200 runs the blocked Cholesky path."""
    Y = _rand_svd(m, c, _RESCUE_SPECTRA[spec](c), m + 3 * c)
    h = rq.Handle()
    V, R = rq.orth(_cm(Y), return_r=True, handle=h)
    flags = h.sync()
    V, R = _np(V), _np(R)
    nY = max(np.linalg.norm(Y, 2), 1e-300)
    Qo, Ro = orc.hqr(Y)
    for Qx, Rx in ((V, R), (Qo, Ro)):
        assert np.abs(Qx.T @ Qx - np.eye(c)).max() <= 1e-14 * np.sqrt(c) * 10
        assert np.abs(Qx @ Rx - Y).max() <= 1e-14 * max(nY, 1e-300) * 10 or spec == "zero"
    assert not np.tril(R, -1).any()
    if spec == "zero":
        assert not R.any()
    assert flags & 1  # the shifted passes ran
    # the factor R agrees with Householder's on the leading, well-separated directions
    if spec in ("gap1e-9", "rank_half"):
        k = c - c // 2 if spec == "rank_half" else c - c // 3
        np.testing.assert_allclose(np.abs(np.diag(R)[:k]), np.abs(np.diag(Ro)[:k]), rtol=1e-8)


# (30, 17), (25, 25), (32, 32), (32, 7), (5, 32), (1, 1), (31, 29): the one-warp kernel (<= 32 x 32);
# (600, 8000), (460, 9001): columns in global memory (too many rows x columns per CTA for shared
# memory) with the lazy panel updates: full panels, and a partial last panel (460 = 57 x 8 + 4)
@pytest.mark.parametrize("rows,cols", [(25, 800), (110, 4096), (64, 5000), (40, 40), (30, 17), (25, 25), (32, 32),
                                       (32, 7), (5, 32), (1, 1), (31, 29), (600, 8000), (460, 9001)])
def test_cpqr_parity(rq, orc, rows, cols):
    rng = np.random.default_rng(rows * cols)
    M = rng.standard_normal((rows, cols)) * np.logspace(0, -4, cols)[rng.permutation(cols)]
    Q, R, perm = rq.cpqr(_cm(M))
    Qo, Ro, permo = orc.cpqr(M)
    s = min(rows, cols)
    perm = perm.cpu().numpy()
    assert np.array_equal(perm[:s], permo[:s])
    R = _np(R)
    # columns past s: compare as a set-permuted R (non-pivot order may differ, reading R5/§8(c.1))
    np.testing.assert_allclose(R[:, :s], Ro[:, :s], atol=1e-13 * np.abs(Ro).max())
    np.testing.assert_allclose(_np(Q), Qo, atol=1e-12)


@pytest.mark.parametrize("d", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("l,n", [(25, 800), (110, 1030)])
def test_qlp_tail_parity(rq, orc, d, l, n):
    rng = np.random.default_rng(l + n + d)
    B = _rand_svd(l, n, np.logspace(0, -4, l), l * n)
    g = rq.qlp_tail(_cm(B), d=d)
    o = orc.qlp_tail(B, d=d)
    assert np.array_equal(g["piv0"].cpu().numpy(), o["piv0"])
    assert np.array_equal(g["piv1"].cpu().numpy(), o["piv1"])
    assert g["t_is_upper"] == o["t_is_upper"]
    T, To = _np(g["T"]), o["T"]
    np.testing.assert_allclose(np.diag(T), np.diag(To), rtol=1e-10)
    np.testing.assert_allclose(T, To, atol=1e-12 * np.abs(To).max())
    np.testing.assert_allclose(_np(g["QB"]), o["QB"], atol=1e-11)
    np.testing.assert_allclose(_np(g["PB"]), o["PB"], atol=1e-11)


# ------------------------------------------------------------------ end to end
def _check_factorization(rq, orc, A, g, o, l, sig_ratio=None, block=None, B_oracle=None, tag=""):
    """north_star tolerances plus element-wise Q, T, P and P^T P (tests/parity.py)."""
    rec = check_factorization(orc, A, g, o, l, sig_ratio=sig_ratio, block=block, B_oracle=B_oracle, tag=tag)
    return rec["res_gpu"], rec["res_orc"]


CASES = [  # (name, m, n, k, p, q, d, sigma)
    ("c1_rqlp", 1000, 800, 20, 5, 0, 0, lambda j: j**-2.0),
    ("c1_erqlp", 1000, 800, 20, 5, 1, 2, lambda j: j**-2.0),
    ("c2_small", 1031, 1030, 100, 10, 1, 2, lambda j: np.exp(-j / 50.0)),
    ("c3_small", 2053, 1029, 122, 16, 2, 2, lambda j: 1.0 / j),
    ("odd_d", 700, 500, 40, 8, 1, 3, lambda j: j**-1.5),
    ("d1", 700, 500, 40, 8, 0, 1, lambda j: j**-1.5),
    ("d4", 700, 500, 40, 8, 0, 4, lambda j: j**-1.5),
    ("wide", 300, 900, 40, 8, 1, 0, lambda j: j**-1.0),
    ("d5", 700, 500, 40, 8, 1, 5, lambda j: j**-1.5),      # NEXT-4: larger odd / even d
    ("d6", 700, 500, 40, 8, 0, 6, lambda j: np.exp(-j / 30.0)),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_end_to_end_parity(rq, orc, case):
    name, m, n, k, p, q, d, sf = case
    r = min(m, n)
    sig = sf(np.arange(1, r + 1.0))
    A = _rand_svd(m, n, sig, m + n)
    l = k + p
    g = rq.factorize(_cm(A), k, p, q=q, d=d, seed=7)
    o = orc.rqlp(A, k, p, q=q, d=d, seed=7, stages=True)
    if d >= 1:
        o["piv1"] = None
    _check_factorization(rq, orc, A, g, o, l, sig[:l] / sig[0], B_oracle=o["B"], tag=name)


@pytest.mark.parametrize("b,q", [(64, 1), (7, 0), (16, 1), (136, 0)])
def test_brqlp_parity(rq, orc, b, q):
    m, n, k, p = 1500, 700, 120, 16
    sig = np.exp(-np.arange(1, 701.0) / 100)
    A = _rand_svd(m, n, sig, 99)
    g = rq.factorize(_cm(A), k, p, q=q, b=b, seed=4)
    o = orc.brqlp(A, k, p, b=b, q=q, seed=4, stages=True)
    _check_factorization(rq, orc, A, g, o, k + p, block=b, B_oracle=o["V"].T @ A, tag=f"brqlp b={b} q={q}")


def test_residual_kernel(rq, orc):
    A = _rand_svd(900, 400, np.arange(1, 401.0) ** -1, 5)
    o = orc.rqlp(A, 30, 6, q=0, d=0, seed=1)
    r = rq.residual(_cm(A), _cm(o["Q"]), _cm(o["T"]), _cm(o["P"]))
    assert r == pytest.approx(orc.residual(A, o["Q"], o["T"], o["P"]), rel=1e-10)


# ------------------------------------------------------------------ edge cases
def test_zero_matrix(rq, orc):
    """Zero A (reading R21): tau = 0 reflectors, L = 0, identity pivots; the GPU completes the
    basis (rank deficiency) so Q and P stay orthonormal."""
    A = np.zeros((60, 40), order="F")
    g = rq.factorize(_cm(A), 3, 2, q=1, d=0, seed=1)
    h = rq.Handle.default()
    flags = h.sync()
    o = orc.rqlp(A, 3, 2, q=1, d=0, seed=1)
    assert not _np(g["T"]).any() and not o["T"].any()
    assert list(g["piv0"].cpu().numpy()) == list(o["piv0"]) == [0, 1, 2, 3, 4]
    Q, P = _np(g["Q"]), _np(g["P"])
    assert np.abs(Q.T @ Q - np.eye(5)).max() <= 1e-13 * 5
    assert np.abs(P.T @ P - np.eye(5)).max() <= 1e-13 * 5
    assert flags & 2  # RQLP_FLAG_RANK_DEFICIENT


@pytest.mark.parametrize("d", [0, 2])
def test_exact_rank_deficient(rq, orc, d):
    """rank(A) = 6 < l = 12: V's completion is not unique (reading R4), so compare the
    basis-invariant quantities: residual ~ 0, the leading 6 pivots and L-values, orthonormality."""
    sig = np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125])
    A = _rand_svd(300, 200, sig, 21)
    g = rq.factorize(_cm(A), 8, 4, q=1, d=d, seed=5)
    o = orc.rqlp(A, 8, 4, q=1, d=d, seed=5)
    nA = np.linalg.norm(A)
    Q, T, P = _np(g["Q"]), _np(g["T"]), _np(g["P"])
    assert orc.residual(A, Q, T, P) <= 1e-13 * nA
    assert np.array_equal(g["piv0"].cpu().numpy()[:6], o["piv0"][:6])
    np.testing.assert_allclose(np.diag(T)[:6], np.diag(o["T"])[:6], rtol=1e-10)
    assert np.abs(np.diag(T)[6:]).max() <= 1e-12 * sig[0]
    assert np.abs(Q.T @ Q - np.eye(12)).max() <= 1e-13 * 12
    assert np.abs(P.T @ P - np.eye(12)).max() <= 1e-13 * 12


def test_l_equals_n_stewart(rq, orc):
    """l = n: RQLP reduces to Stewart's pivoted QLP; GPU == oracle."""
    A = _rand_svd(70, 30, np.logspace(0, -4, 30), 6)
    g = rq.factorize(_cm(A), 25, 5, q=0, d=0, seed=11)
    o = orc.rqlp(A, 25, 5, q=0, d=0, seed=11)
    _check_factorization(rq, orc, A, g, o, 30)


@pytest.mark.parametrize("m,n,k,p,q,d", [(40, 30, 2, 2, 0, 0), (9, 300, 3, 2, 1, 1), (500, 400, 30, 10, 3, 5),
                                         (12, 12, 8, 4, 2, 2)])
def test_small_and_degenerate_shapes(rq, orc, m, n, k, p, q, d):
    """Minimal k = p = 2, m = l (square sketch), wide, many power steps / inner QRs."""
    r = min(m, n)
    sig = np.logspace(0, -3, r)
    A = _rand_svd(m, n, sig, m * n + q)
    g = rq.factorize(_cm(A), k, p, q=q, d=d, seed=3)
    o = orc.rqlp(A, k, p, q=q, d=d, seed=3)
    if d >= 1:
        o["piv1"] = None
    _check_factorization(rq, orc, A, g, o, k + p, sig[:k + p] / sig[0])


def test_brqlp_unit_blocks(rq, orc):
    """b = 1: every block is a single column (Alg. 3 with h = l)."""
    A = _rand_svd(200, 120, np.exp(-np.arange(1, 121.0) / 10), 31)
    g = rq.factorize(_cm(A), 6, 3, q=1, b=1, seed=2)
    o = orc.brqlp(A, 6, 3, b=1, q=1, seed=2)
    _check_factorization(rq, orc, A, g, o, 9, block=1)


def test_argument_errors_gpu(rq):
    A = torch.zeros(10, 8, dtype=torch.float64, device="cuda").t().contiguous().t()
    with pytest.raises(rq.RQLPError):
        rq.rqlp(A, 1, 2)
    with pytest.raises(rq.RQLPError):
        rq.rqlp(A, 5, 4)          # l = 9 > n = 8
    with pytest.raises(rq.RQLPError):
        rq.erqlp(A, 3, 2, d=0)    # d >= 1
    with pytest.raises(rq.RQLPError):
        rq.brqlp(A, 3, 2, b=6)    # b <= l


def test_host_pointer_entry_points(rq, orc):
    """The north-star rqlp() and rqlp_factorize() with HOST buffers (e2e path) equal the device path."""
    A = _rand_svd(300, 200, np.arange(1, 201.0) ** -2, 41)
    Qh, Lh, Ph = rq.rqlp_host(A, 20, 5, q=1, seed=9)
    g = rq.factorize(_cm(A), 20, 5, q=1, seed=9)
    np.testing.assert_array_equal(Lh, _np(g["T"]))
    np.testing.assert_array_equal(Qh, _np(g["Q"]))
    At = torch.from_numpy(np.ascontiguousarray(A.T)).pin_memory().t()
    Q2, T2, P2, tu = rq.factorize_host(At, 20, 5, q=1, d=2, seed=9)
    g2 = rq.factorize(_cm(A), 20, 5, q=1, d=2, seed=9)
    np.testing.assert_array_equal(T2.numpy(), _np(g2["T"]))
    assert tu


@pytest.mark.parametrize("pin_a", [True, False])
def test_brqlp_host_outputs_streamed(rq, pin_a):
    """BRQLP through rqlp_factorize with pinned host Q/P: each block's Q_j, P_j is copied out on the
    copy stream while the later blocks run; the result equals the device path bit for bit (ragged
    last block; pinned A fed in row panels, or pageable A copied up front), also on a graph replay."""
    A = _rand_svd(1500, 700, np.exp(-np.arange(1, 701.0) / 40), 77)
    g = rq.factorize(_cm(A), 40, 10, q=1, b=16, seed=5)
    At = torch.from_numpy(np.ascontiguousarray(A.T))
    if pin_a:
        At = At.pin_memory()
    At = At.t()
    out = tuple(torch.empty(c, r, dtype=torch.float64, pin_memory=True).t() for r, c in ((1500, 50), (50, 50), (700, 50)))
    h = rq.Handle()
    for _ in range(2):   # the second call replays the captured graph
        for t in out:
            t.fill_(np.nan)
        Q, T, P, _ = rq.factorize_host(At, 40, 10, q=1, b=16, seed=5, handle=h, out=out)
        np.testing.assert_array_equal(Q.numpy(), _np(g["Q"]))
        np.testing.assert_array_equal(T.numpy(), _np(g["T"]))
        np.testing.assert_array_equal(P.numpy(), _np(g["P"]))


def test_deterministic_reruns(rq):
    """Bitwise-identical results across reruns (fixed-order reductions, no atomics in sums)."""
    A = _cm(_rand_svd(1031, 1030, np.exp(-np.arange(1, 1031.0) / 50), 2))
    a = rq.factorize(A, 100, 10, q=1, d=2, seed=2)
    b = rq.factorize(A, 100, 10, q=1, d=2, seed=2)
    for key in ("Q", "T", "P", "piv0"):
        assert torch.equal(a[key], b[key])


# ------------------------------------------------------------------ NEXT-1: auto-rank RQLP
@pytest.mark.parametrize("m,n,b,l_max,eps,q", [(1500, 700, 16, 256, 1e-2, 1), (1200, 900, 24, 100, 0.0, 0),
                                               (900, 600, 32, 320, 1e-3, 2), (400, 300, 8, 64, 1.0, 0)])
def test_autorank_parity(rq, orc, m, n, b, l_max, eps, q):
    """Auto-rank RQLP (eq. (3) indicator): same stopping block, pivots and
    L-values as the oracle; the reported indicator equals the direct residual.  (1200, 900, 24, 100,
    eps=0) runs to l_max with a ragged last block; eps = 1 stops after the first block."""
    sig = np.exp(-np.arange(1, min(m, n) + 1.0) / 40)
    A = _rand_svd(m, n, sig, m + 3 * n)
    g = rq.autorank(_cm(A), b=b, l_max=l_max, eps=eps, q=q, seed=6)
    o = orc.autorank(A, b=b, l_max=l_max, eps=eps, q=q, seed=6)
    assert g["l"] == o["l"], (g["l"], o["l"])
    l = g["l"]
    _check_factorization(rq, orc, A, g, o, l, block=b)
    assert g["err"] == pytest.approx(o["err"], rel=1e-8, abs=1e-13)
    direct = orc.residual(A, _np(g["Q"]), _np(g["T"]), _np(g["P"])) / np.linalg.norm(A)
    assert g["err"] == pytest.approx(direct, rel=1e-6, abs=1e-13)
    if eps > 0 and l < l_max:
        assert g["err"] <= eps


def test_autorank_argument_errors(rq):
    A = torch.zeros(10, 8, dtype=torch.float64, device="cuda").t().contiguous().t()
    with pytest.raises(rq.RQLPError):
        rq.autorank(A, b=4, l_max=2, eps=0.1)     # l_max < b
    with pytest.raises(rq.RQLPError):
        rq.autorank(A, b=2, l_max=9, eps=0.1)     # l_max > n
    with pytest.raises(rq.RQLPError):
        rq.autorank(A, b=2, l_max=4, eps=-1.0)    # eps < 0


# ------------------------------------------------------------------ NEXT-3: truncated pivoted QLP
TQLP_CASES = [  # (name, m, n, l, sigma)
    ("tall", 500, 300, 40, lambda j: 2.0 ** (-j / 4)),
    ("c2_like", 1031, 1030, 110, lambda j: np.exp(-j / 50.0)),
    ("wide", 300, 900, 50, lambda j: j**-1.0),
    ("full", 64, 64, 64, lambda j: np.logspace(0, -6, 64)[(j - 1).astype(int)]),
    ("one", 200, 150, 1, lambda j: j**-2.0),
]


@pytest.mark.parametrize("case", TQLP_CASES, ids=[c[0] for c in TQLP_CASES])
def test_tqlp_parity(rq, orc, case):
    """Deterministic truncated pivoted QLP on the GPU engine == oracle."""
    name, m, n, l, sf = case
    sig = sf(np.arange(1, min(m, n) + 1.0))
    A = _rand_svd(m, n, sig, 5 * m + n)
    g = rq.tqlp(_cm(A), l)
    o = orc.tqlp(A, l)
    _check_factorization(rq, orc, A, g, o, l, sig[:l] / sig[0])
    Pg = _np(g["P"])
    assert np.abs(Pg.T @ Pg - np.eye(l)).max() <= 1e-13 * l
    assert not np.triu(_np(g["T"]), 1).any()



def test_brqlp_q0_two_passes(rq, orc):
    """NEXT-4: BRQLP with q = 0 reads A exactly twice (one batched sketch, one batched
    projection) instead of 1 + h times, with the same result as the oracle's explicit deflation."""
    m, n, k, p, b = 1200, 500, 60, 12, 16        # h = 5 blocks, ragged last block
    A = _rand_svd(m, n, np.exp(-np.arange(1, 501.0) / 60), 314)
    h = rq.Handle.default()
    h.set_timing(True)
    try:
        g = rq.factorize(_cm(A), k, p, q=0, b=b, seed=9)
        names = [nm for nm, _ in h.timing()]
    finally:
        h.set_timing(False)
    o = orc.brqlp(A, k, p, b=b, q=0, seed=9)
    _check_factorization(rq, orc, A, g, o, k + p, block=b)
    passes = [nm for nm in names if nm.startswith("pass_")]
    assert passes == ["pass_sketch", "pass_project"], passes


def test_pivot_ties_duplicate_columns(rq, orc):
    """Exact ties (duplicate columns, equal norms): CPQR breaks them toward the lowest original
    column index (reading R5) in both implementations, for RQLP and the truncated QLP."""
    rng = np.random.default_rng(77)
    A = rng.standard_normal((300, 120)) @ np.diag(np.logspace(0, -3, 120))
    A[:, 40] = A[:, 3]
    A[:, 90] = A[:, 3]
    A[:, 11] = -A[:, 7]          # equal norms, opposite signs
    A = np.asfortranarray(A)
    g = rq.factorize(_cm(A), 20, 6, q=1, d=0, seed=2)
    o = orc.rqlp(A, 20, 6, q=1, d=0, seed=2)
    assert np.array_equal(g["piv0"].cpu().numpy(), o["piv0"])
    gt, ot = rq.tqlp(_cm(A), 26), orc.tqlp(A, 26)
    assert np.array_equal(gt["piv0"].cpu().numpy(), ot["piv0"])
    assert np.array_equal(gt["piv1"].cpu().numpy(), ot["piv1"])


@pytest.mark.parametrize("b,l_max,q", [(10, 95, 2), (33, 99, 0)])
def test_autorank_ragged_and_power(rq, orc, b, l_max, q):
    """Auto-rank with a block size that does not divide l_max and with power steps."""
    sig = np.arange(1, 301.0) ** -1.2
    A = _rand_svd(700, 300, sig, 4242)
    g = rq.autorank(_cm(A), b=b, l_max=l_max, eps=5e-2, q=q, seed=8)
    o = orc.autorank(A, b=b, l_max=l_max, eps=5e-2, q=q, seed=8)
    assert g["l"] == o["l"]
    _check_factorization(rq, orc, A, g, o, g["l"], block=b)


# ------------------------------------------------------------------ graph replay of the rare branches
def _zero(m, n, seed):
    return np.zeros((m, n), order="F")


def _deficient(m, n, seed):
    return _rand_svd(m, n, np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125]), seed)


def _illcond(m, n, seed):
    # rank 16 = l, cond(Y) ~ 1e13 > u^-1/2: the unshifted Cholesky breaks down, the shifted
    # third pass runs
    return _rand_svd(m, n, np.logspace(0, -13, 16), seed)


def _wellcond(m, n, seed):
    return _rand_svd(m, n, np.exp(-np.arange(1, min(m, n) + 1.0) / 20), seed)


@pytest.mark.parametrize("make,flag,d", [(_zero, 2, 0), (_deficient, 2, 2), (_illcond, 1, 0), (_wellcond, 0, 2)])
def test_graph_replay_branches(rq, orc, make, flag, d):
    """Each call with the same arguments runs eagerly first, then as a captured CUDA graph in which
    the rare orth branch (the shifted CholeskyQR passes / random completion of orth_rescue.cu) is
    an early-exiting cooperative kernel that decides on the device whether to work.  Eager and
    replayed results must be bitwise identical and flag the branch."""
    A = make(400, 300, 5)
    h = rq.Handle()
    At = _cm(A)
    res, ptrs, flags = [], set(), []
    for _ in range(4):
        g = rq.factorize(At, 12, 4, q=1, d=d, seed=7, handle=h)
        flags.append(h.sync())
        ptrs.add(tuple(g[k].data_ptr() for k in ("Q", "T", "P")))
        res.append({k: _np(g[k]) for k in ("Q", "T", "P")})
        del g
    assert len(ptrs) == 1  # same buffers -> calls 2..4 are capture + replays of one graph
    for r in res[1:]:
        for k in ("Q", "T", "P"):
            np.testing.assert_array_equal(r[k], res[0][k])
    assert all((f & flag) == flag and (flag or not f & 3) for f in flags), flags
    Q, T, P = res[0]["Q"], res[0]["T"], res[0]["P"]
    assert np.abs(Q.T @ Q - np.eye(16)).max() <= 1e-12
    # the residual of the oracle on the same input bounds ours (rank(A) <= l: both ~ exact, up to
    # the directions the power step pushes below the rounding level of Y)
    o = orc.rqlp(A, 12, 4, q=1, d=d, seed=7)
    ro = orc.residual(A, o["Q"], o["T"], o["P"])
    assert orc.residual(A, Q, T, P) <= 10 * ro + 1e-13 * max(np.linalg.norm(A), 1.0)


@pytest.mark.parametrize("bad", [np.nan, np.inf])
@pytest.mark.parametrize("variant", [dict(q=1, d=0), dict(q=1, d=2), dict(q=0, b=4)])
def test_nonfinite_input_terminates(rq, bad, variant):
    """A non-finite entry in A must not hang any kernel (the Cholesky breakdown, the rescue's
    grid barriers, the CPQR engine's exchange): the call returns and the output is non-finite
    or flagged, never a deadlock."""
    A = _rand_svd(300, 200, np.logspace(0, -3, 200), 3)
    A[17, 23] = bad
    h = rq.Handle()
    g = rq.factorize(_cm(A), 10, 4, seed=1, handle=h, **variant)
    h.sync()
    assert g["Q"].shape == (300, 14)


@pytest.mark.parametrize("scale", [1e200, 1e-200])
def test_extreme_scale_terminates(rq, orc, scale):
    """|A| near the double range limits: CholeskyQR's Grams and the CPQR's squared column norms
    over/underflow (documented limit: max|A| sqrt(n) within ~1e+-150; scale A
    first otherwise).  The call must still return without a fault or a hang."""
    A = _rand_svd(300, 200, np.logspace(0, -3, 200), 4) * scale
    h = rq.Handle()
    g = rq.factorize(_cm(A), 10, 4, q=1, seed=1, handle=h)
    flags = h.sync()
    Q = _np(g["Q"])
    ok = np.isfinite(Q).all() and np.abs(Q.T @ Q - np.eye(14)).max() <= 1e-12
    print(f"scale {scale:g}: flags {flags}, Q finite and orthonormal: {ok}")


# ------------------------------------------------------------------ eq. (3) indicator (§8 a10)
IND_CASES = [  # (name, m, n, k, p, q, d, b, col-major padding of A)
    ("rqlp", 1000, 800, 20, 5, 0, 0, None, 0),
    ("erqlp", 1031, 1030, 100, 10, 1, 2, None, 0),
    ("brqlp", 1500, 700, 120, 16, 1, 0, 64, 0),
    ("brqlp_q0", 1200, 500, 60, 12, 0, 0, 16, 0),
    ("odd_lda_fallback", 700, 500, 40, 8, 1, 2, None, 1),   # lda odd: no TMA map, separate fro pass
]


@pytest.mark.parametrize("case", IND_CASES, ids=[c[0] for c in IND_CASES])
def test_indicator_eq3(rq, orc, case):
    """||A||_F^2 accumulated inside the first A-pass and ||B||_F^2 (BRQLP: the deflated B_j) give
    the eq. (3) identity ||A - V V^T A||_F^2 = ||A||^2 - ||B||^2: each term
    against the oracle, the difference against the oracle's and against the direct residual."""
    name, m, n, k, p, q, d, b, pad = case
    sig = np.exp(-np.arange(1, min(m, n) + 1.0) / 40)
    A = _rand_svd(m, n, sig, m + 7 * n)
    Ad = torch.zeros(n, m + pad, dtype=torch.float64, device="cuda")
    Ad[:, :m] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    Ad = Ad.t()[:m]                                  # column-major view, lda = m + pad
    h = rq.Handle()
    g = rq.factorize(Ad, k, p, q=q, d=d, b=b, seed=13, handle=h)
    ind = h.indicator()
    a2_o = orc.fro(A) ** 2
    if b is None:
        o = orc.rqlp(A, k, p, q=q, d=d, seed=13, stages=True)
        b2_o = orc.fro(o["B"]) ** 2
    else:
        o = orc.brqlp(A, k, p, b=b, q=q, seed=13, stages=True)
        b2_o = orc.fro(orc.gemm_tn(o["V"], A)) ** 2   # sum_j ||B_j||^2 = ||V^T A||^2 (V orthonormal)
    assert ind["a2"] == pytest.approx(a2_o, rel=1e-13)
    assert ind["b2"] == pytest.approx(b2_o, rel=1e-12)
    assert abs((ind["a2"] - ind["b2"]) - (a2_o - b2_o)) <= 1e-12 * a2_o
    res = orc.residual(A, _np(g["Q"]), _np(g["T"]), _np(g["P"]))
    assert abs((ind["a2"] - ind["b2"]) - res ** 2) <= 1e-12 * a2_o
