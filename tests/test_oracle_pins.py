"""Pins for the CPU oracle (oracle/), checked against things other than the oracle itself:
numpy's independent Philox4x64-10, mpmath, LAPACK (numpy/scipy), closed forms, invariants and
brute force.  Each test names the plausible oracle mistake it would catch.  CPU only."""
import math

import mpmath
import numpy as np
import pytest
import scipy.linalg as sla

from synthetic import sigma

mpmath.mp.dps = 40


def _rand_svd(m, n, sig, seed):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, len(sig))))
    V, _ = np.linalg.qr(rng.standard_normal((n, len(sig))))
    return np.asfortranarray((U * sig) @ V.T)


# ------------------------------------------------------------------ RNG
@pytest.mark.parametrize("seed,stream,ctr", [(0, 0, 0), (1, 0, 5), (12345, 3, 2**40 + 17),
                                             (2**64 - 1, 2, 2**64 - 1), (7, 2**63, 123456789)])
def test_philox_kat_vs_numpy(orc, seed, stream, ctr):
    """Raw Philox4x64-10 words == numpy's implementation (catches a wrong constant, round or
    key schedule).  numpy pre-increments its 256-bit counter, so start it at C-1."""
    val = (ctr + (stream << 64) - 1) % (1 << 256)
    words = [(val >> (64 * i)) & (2**64 - 1) for i in range(4)]
    g = np.random.Philox(key=np.array([seed, 0], dtype=np.uint64), counter=np.array(words, dtype=np.uint64))
    assert orc.philox([ctr, stream, 0, 0], [seed, 0]) == [int(x) for x in g.random_raw(4)]


def test_uniform_exact_open_interval(orc):
    assert orc.uniform(0) == 0.5 * 2.0**-52
    assert orc.uniform(2**64 - 1) == 1.0 - 0.5 * 2.0**-52
    assert orc.uniform(1 << 12) == 1.5 * 2.0**-52       # low 12 bits discarded


def _u_samples(count, seed=0):
    rng = np.random.default_rng(seed)
    xs = [int(x) for x in rng.integers(0, 2**63, size=count, dtype=np.int64).astype(np.uint64) * 2 + 1]
    return xs + [0, 2**64 - 1, 1 << 62, (1 << 63) + (1 << 12), (1 << 64) - (1 << 12)]


def test_pinned_ln_accuracy(orc):
    """Pinned ln within 2 ulp of the exact value (catches a wrong coefficient/reduction)."""
    worst = 0.0
    for x in _u_samples(1500):
        u = orc.uniform(x)
        ref = float(mpmath.log(mpmath.mpf(u)))
        worst = max(worst, abs(orc.ln(u) - ref) / math.ulp(ref))
    assert worst <= 2.0


def test_pinned_sincos_accuracy(orc):
    """Pinned sin/cos(2πu) within 2 ulp (or 2^-53 absolute near zeros): catches a wrong
    quadrant mapping or polynomial."""
    for x in _u_samples(1500, seed=1):
        u = mpmath.mpf(orc.uniform(x))
        s, c = orc.sincos_2pi(x)
        for got, ref in ((s, float(mpmath.sin(2 * mpmath.pi * u))), (c, float(mpmath.cos(2 * mpmath.pi * u)))):
            assert abs(got - ref) <= max(2 * math.ulp(ref), 2.0**-53)


def test_box_muller_structure(orc):
    """z0^2+z1^2 = -2 ln u(x0) and atan2(z1,z0) = 2π u(x1): ties the normals to the raw words
    (catches swapped pair roles, a dropped factor 2, sin/cos swapped)."""
    for blk in range(64):
        z = orc.normal4(99, 0, blk)
        x = orc.philox([blk, 0, 0, 0], [99, 0])
        for h in range(2):
            ua, ub = orc.uniform(x[2 * h]), orc.uniform(x[2 * h + 1])
            assert z[2 * h] ** 2 + z[2 * h + 1] ** 2 == pytest.approx(-2 * math.log(ua), rel=1e-13)
            ang = math.atan2(z[2 * h + 1], z[2 * h]) % (2 * math.pi)
            d = abs(ang - 2 * math.pi * ub)
            assert min(d, 2 * math.pi - d) < 1e-12


def test_gaussian_moments_and_layout(orc):
    """Mean/variance within 5σ of N(0,1); element t = i + rows*j uses block t//4,
    lane t%4 (so BRQLP's Ω_j are column slices of Ω)."""
    Z = orc.gaussian(5, 0, 1000, 100)
    N = Z.size
    assert abs(Z.mean()) < 5 / math.sqrt(N)
    assert abs(Z.var() - 1) < 5 * math.sqrt(2 / N)
    t = 1000 * 37 + 421
    assert Z[421, 37] == orc.normal4(5, 0, t // 4)[t % 4]
    Z2 = orc.gaussian(5, 0, 1000, 64)
    assert np.array_equal(Z2, Z[:, :64])


def test_golden_omega(orc):
    """Regression fixture written by tools/make_golden.py (oracle-only)."""
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "omega_seed1_800x25.txt")
    rows = np.loadtxt(path, comments="#")
    Om = orc.omega(1, 800, 25)
    for i, j, v in rows:
        assert Om[int(i), int(j)] == v


# ------------------------------------------------------------------ dense blocks
def test_gemm_vs_numpy(orc):
    rng = np.random.default_rng(3)
    A, B = rng.standard_normal((67, 45)), rng.standard_normal((45, 13))
    np.testing.assert_allclose(orc.gemm_nn(A, B), A @ B, rtol=0, atol=1e-13)
    np.testing.assert_allclose(orc.gemm_tn(A, rng.standard_normal((67, 9)))[:2].shape, (2, 9))
    C = rng.standard_normal((67, 9))
    np.testing.assert_allclose(orc.gemm_tn(A, C), A.T @ C, rtol=0, atol=1e-13)


def test_hqr_closed_forms(orc):
    Q, R = orc.hqr(np.array([[3.0], [4.0]]))
    assert R[0, 0] == pytest.approx(5.0, rel=1e-15)
    np.testing.assert_allclose(Q[:, 0], [0.6, 0.8], rtol=1e-15)
    Q, R = orc.hqr(np.eye(5))
    np.testing.assert_allclose(Q, np.eye(5), atol=1e-15)
    np.testing.assert_allclose(R, np.eye(5), atol=1e-15)
    Q, R = orc.hqr(-np.eye(3)[:, :2])                 # R_ii >= 0 normalisation flips signs
    np.testing.assert_allclose(R, np.eye(2), atol=1e-15)
    A = np.zeros((4, 2)); A[:, 1] = [1, 2, 2, 0]     # zero column -> tau = 0, Q column e_0
    Q, R = orc.hqr(A)
    np.testing.assert_allclose(Q.T @ Q, np.eye(2), atol=1e-15)
    np.testing.assert_allclose(Q @ R, A, atol=1e-15)
    assert R[0, 0] == 0.0 and R[0, 1] == 1.0 and R[1, 1] == pytest.approx(math.sqrt(8.0))


def test_hqr_vs_lapack(orc):
    """Thin Q, R (R_ii >= 0) equal LAPACK's up to rounding: catches a wrong reflector/sign."""
    rng = np.random.default_rng(4)
    A = rng.standard_normal((90, 31))
    Q, R = orc.hqr(A)
    Qn, Rn = np.linalg.qr(A)
    s = np.sign(np.diag(Rn))
    np.testing.assert_allclose(Q, Qn * s, atol=1e-14)
    np.testing.assert_allclose(R, (Rn.T * s).T, atol=1e-13)


def test_cpqr_closed_forms(orc):
    Q, R, perm = orc.cpqr(np.diag([1.0, 2.0, 3.0]))
    assert list(perm) == [2, 1, 0]
    np.testing.assert_allclose(np.abs(np.diag(R)), [3, 2, 1])
    Q, R, perm = orc.cpqr(np.zeros((4, 4)))
    assert list(perm) == [0, 1, 2, 3] and not R.any()
    # exact ties break to the lowest original column index (reading R5)
    Q, R, perm = orc.cpqr(np.diag([1.0, 2.0, 2.0, 1.0]))
    assert list(perm) == [1, 2, 0, 3]


@pytest.mark.parametrize("shape", [(40, 25), (25, 90), (60, 60)])
def test_cpqr_vs_lapack_geqp3(orc, shape):
    """Pivots and |R| equal LAPACK geqp3 (scipy), Q R = A Π: catches a wrong downdating rule,
    a missing swap or a wrong pivot criterion."""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    A = rng.standard_normal(shape) * np.logspace(0, -3, shape[1])
    Q, R, perm = orc.cpqr(A)
    _, R2, P2 = sla.qr(A, pivoting=True, mode="economic")
    s = min(shape)
    assert np.array_equal(perm[:s], P2[:s])
    np.testing.assert_allclose(np.abs(R[:, :s]), np.abs(R2[:, :s]), atol=1e-13)
    np.testing.assert_allclose(Q @ R, A[:, perm], atol=1e-13)
    assert (np.diag(R) >= 0).all()
    assert np.all(np.diff(np.abs(np.diag(R))) <= 1e-15)


def test_svd_brute_force(orc):
    phi = (1 + math.sqrt(5)) / 2
    np.testing.assert_allclose(orc.svd_values(np.array([[1.0, 1.0], [0.0, 1.0]])), [phi, 1 / phi], rtol=1e-14)
    np.testing.assert_allclose(orc.svd_values(np.diag([3.0, -2.0, 1.0])), [3, 2, 1], rtol=1e-15)
    rng = np.random.default_rng(5)
    A = rng.standard_normal((30, 12))
    np.testing.assert_allclose(orc.svd_values(A), np.linalg.svd(A, compute_uv=False), rtol=1e-13)
    # all 2x2 matrices with entries in {-2..2} vs the closed form
    vals = [-2.0, -1.0, 0.0, 1.0, 2.0]
    for a in vals:
        for b in vals:
            for c in vals[::2]:
                for d in vals[1::2]:
                    M = np.array([[a, b], [c, d]])
                    fro2, det = a * a + b * b + c * c + d * d, abs(a * d - b * c)
                    disc = math.sqrt(max(fro2 * fro2 - 4 * det * det, 0.0))
                    s1 = math.sqrt((fro2 + disc) / 2)
                    s2 = det / s1 if s1 > 0 else 0.0
                    np.testing.assert_allclose(orc.svd_values(M), [s1, s2], atol=1e-12)


# ------------------------------------------------------------------ the method
def test_rqlp_l_eq_n_is_stewart_qlp(orc):
    """ℓ = n: RQLP ≡ Stewart's pivoted QLP (eq. (2)) computed with two LAPACK
    geqp3 calls -- same Π0, Π1 and L-values (catches errors anywhere in the tail)."""
    m, n = 70, 30
    A = _rand_svd(m, n, np.logspace(0, -4, n), 6)
    out = orc.rqlp(A, k=25, p=5, q=0, d=0, seed=11)
    _, R, P0 = sla.qr(A, pivoting=True, mode="economic")
    _, Lt, P1 = sla.qr(R.T, pivoting=True, mode="economic")
    assert np.array_equal(out["piv0"], P0[:n])
    assert np.array_equal(out["piv1"], P1)
    np.testing.assert_allclose(np.diag(out["T"]), np.abs(np.diag(Lt)), rtol=1e-10)
    assert not out["t_is_upper"]
    np.testing.assert_allclose(np.triu(out["T"], 1), 0.0)


@pytest.mark.parametrize("d", [0, 1, 2, 3, 4])
def test_eq3_identity_and_reconstruction(orc, d):
    """eq.(3) ‖A−P_VA‖² = ‖A‖²−‖B‖² with B recomputed by numpy from the oracle's
    V, QLPᵀ = VB (eq. (5)), T triangular with the corrected parity (reading R9)."""
    A = _rand_svd(300, 200, np.arange(1, 201.0) ** -2, 7)
    out = orc.rqlp(A, k=20, p=5, q=1, d=d, seed=3, stages=True)
    V, Q, T, P = out["V"], out["Q"], out["T"], out["P"]
    B = V.T @ A
    np.testing.assert_allclose(out["B"], B, atol=1e-14)
    direct = np.linalg.norm(A - V @ B)
    assert direct**2 == pytest.approx(np.linalg.norm(A) ** 2 - np.linalg.norm(B) ** 2, abs=1e-13)
    np.testing.assert_allclose(Q @ T @ P.T, V @ B, atol=1e-14)
    assert orc.residual(A, Q, T, P) == pytest.approx(direct, rel=1e-11)
    l = 25
    assert np.abs(Q.T @ Q - np.eye(l)).max() < 1e-13 * l
    assert np.abs(P.T @ P - np.eye(l)).max() < 1e-13 * l
    upper = d >= 2 and d % 2 == 0
    assert out["t_is_upper"] == upper
    assert not (np.tril(T, -1) if upper else np.triu(T, 1)).any()
    assert (np.diag(T) >= 0).all()


def test_paper_literal_even_d_assembly_is_wrong(orc):
    """Documents reading R9: Alg.2 l.9 literally (L = [R^(d)]ᵀ for even d) does NOT reproduce B."""
    rng = np.random.default_rng(8)
    B = rng.standard_normal((10, 40))
    t = orc.qlp_tail(B, d=2)
    np.testing.assert_allclose(t["QB"] @ t["T"] @ t["PB"].T, B, atol=1e-13)
    assert np.linalg.norm(t["QB"] @ t["T"].T @ t["PB"].T - B) > 1e-3 * np.linalg.norm(B)


def test_residual_invariant_across_d(orc):
    """Same seed => same V; inner QRs are orthogonal => identical residual."""
    A = _rand_svd(200, 150, np.arange(1, 151.0) ** -1.5, 9)
    res = [orc.residual(A, *(lambda o: (o["Q"], o["T"], o["P"]))(orc.rqlp(A, 15, 5, q=0, d=d, seed=4)))
           for d in range(5)]
    assert max(res) - min(res) < 1e-14 * np.linalg.norm(A)


def test_exact_rank_recovery(orc):
    """rank r ≤ k: residual ~ 0 (eq. (3) optimum) and L-values -> σ_j for large d."""
    sig = np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125])
    A = _rand_svd(120, 90, sig, 10)
    for d in (0, 2):
        out = orc.rqlp(A, k=8, p=4, q=0, d=d, seed=5)
        assert orc.residual(A, out["Q"], out["T"], out["P"]) < 1e-13 * np.linalg.norm(A)
    out = orc.rqlp(A, k=8, p=4, q=0, d=40, seed=5)
    np.testing.assert_allclose(np.abs(np.diag(out["T"]))[:6], sig, rtol=1e-10)


def test_power_iteration_reaches_optimal_residual(orc):
    """With a spectral gap at ℓ, q subspace iterations drive the residual to the Eckart-Young
    optimum sqrt(Σ_{j>ℓ} σ_j²) (closed form from the constructed σ; reading R12)."""
    l = 12
    sig = np.concatenate([np.linspace(1.0, 0.5, l), 1e-3 * np.linspace(1.0, 0.5, 188)])
    A = _rand_svd(300, 200, sig, 12)
    opt = math.sqrt(np.sum(sig[l:] ** 2))
    gaps = []
    for q in (0, 1, 4):
        out = orc.rqlp(A, k=8, p=4, q=q, d=0, seed=6)
        gaps.append(orc.residual(A, out["Q"], out["T"], out["P"]) / opt - 1)
    assert gaps[0] > 1e-2 and gaps[1] < 1e-3 and abs(gaps[2]) < 1e-10


def test_large_d_converges_to_singular_values_of_B(orc):
    """Huckaby-Chan: |diag R^(d)| -> σ(B) on a gapped spectrum."""
    A = _rand_svd(200, 150, 2.0 ** -np.arange(1, 151.0), 13)
    out = orc.rqlp(A, k=10, p=5, q=0, d=30, seed=7, stages=True)
    sB = np.linalg.svd(out["B"], compute_uv=False)
    np.testing.assert_allclose(np.abs(np.diag(out["T"])), sB, rtol=1e-12)
    d2 = orc.rqlp(A, k=10, p=5, q=0, d=2, seed=7)
    d4 = orc.rqlp(A, k=10, p=5, q=0, d=4, seed=7)
    e = [np.max(np.abs(np.abs(np.diag(o["T"])) - sB) / sB) for o in (d2, d4)]
    assert e[1] < e[0]


def test_interlacing(orc):
    """σ_j(L) = σ_j(B) ≤ σ_j(A) (Lemma)."""
    sig = np.arange(1, 101.0) ** -1.0
    A = _rand_svd(150, 100, sig, 14)
    out = orc.rqlp(A, k=20, p=5, q=1, d=2, seed=8)
    sL = np.linalg.svd(out["T"], compute_uv=False)
    assert np.all(sL <= sig[:25] * (1 + 1e-10))


def test_brqlp_single_block_is_rqlp(orc):
    """h = 1 (b = ℓ): Alg. 3 degenerates to Alg. 1 on the same Ω."""
    A = _rand_svd(160, 120, np.arange(1, 121.0) ** -2, 15)
    r = orc.rqlp(A, k=16, p=4, q=0, d=0, seed=9)
    b = orc.brqlp(A, k=16, p=4, b=20, q=0, seed=9)
    for key in ("Q", "T", "P"):
        np.testing.assert_allclose(b[key], r[key], atol=1e-12)
    assert np.array_equal(b["piv0"], r["piv0"]) and np.array_equal(b["piv1"], r["piv1"])


@pytest.mark.parametrize("b", [7, 8, 25])
def test_brqlp_projector_identity(orc, b):
    """Fixed Ω, q = 0: block and unblocked range finders give the same projector,
    and A − QLPᵀ = A − VVᵀA (eq. (21)).  b = 7 leaves a ragged last block."""
    sig = np.exp(-np.arange(1, 201.0) / 20)
    A = _rand_svd(300, 200, sig, 16)
    l = 25
    bl = orc.brqlp(A, k=20, p=5, b=b, q=0, seed=10, stages=True)
    rq = orc.rqlp(A, k=20, p=5, q=0, d=0, seed=10, stages=True)
    Vb, Vu = bl["V"], rq["V"]
    assert np.linalg.norm(Vb @ (Vb.T @ A) - Vu @ (Vu.T @ A)) < 1e-12 * np.linalg.norm(A)
    np.testing.assert_allclose(bl["Q"] @ bl["T"] @ bl["P"].T, Vb @ (Vb.T @ A), atol=1e-13)
    h = -(-l // b)
    for j in range(h):                   # L block diagonal, lower triangular blocks
        c0, c1 = j * b, min(l, (j + 1) * b)
        blk = bl["T"][c0:c1, c0:c1]
        assert not np.triu(blk, 1).any()
        off = bl["T"][c0:c1].copy()
        off[:, c0:c1] = 0
        assert not off.any()
        assert np.all(bl["piv1"][c0:c1] < c1 - c0)


def test_brqlp_deflated_power_step(orc):
    """q = 1 deflated steps (reading R16) improve the residual and keep Q orthonormal."""
    sig = np.exp(-np.arange(1, 201.0) / 30)
    A = _rand_svd(300, 200, sig, 17)
    r0 = orc.brqlp(A, 20, 6, 8, q=0, seed=2)
    r1 = orc.brqlp(A, 20, 6, 8, q=1, seed=2)
    e0 = orc.residual(A, r0["Q"], r0["T"], r0["P"])
    e1 = orc.residual(A, r1["Q"], r1["T"], r1["P"])
    assert e1 < e0
    assert np.abs(r1["Q"].T @ r1["Q"] - np.eye(26)).max() < 1e-13 * 26


@pytest.mark.parametrize("kind", ["rank_deficient", "gap"])
def test_brqlp_reorth_twice_keeps_q_orthonormal(orc, kind):
    """Reading R28: with Alg. 3 l.5 applied twice, Q stays orthonormal when a block lies (almost)
    inside span(V_<j) -- beyond rank(A), or past a spectral gap -- where one pass cannot (in exact
    arithmetic a block inside the span gives qr(0)); the residual is the exact-arithmetic one
    (rank(A) <= l: ~0), a value fixed by the construction, not by the oracle."""
    l = 30
    sig = (np.r_[1.0 / np.arange(1, 16.0), np.zeros(185)] if kind == "rank_deficient"
           else np.where(np.arange(1, 201) <= 20, 1.0, 1e-9) / np.arange(1, 201.0))
    A = _rand_svd(400, 200, sig, 31)
    out = orc.brqlp(A, 26, 4, b=4, q=0, seed=3)
    Q = out["Q"]
    assert np.abs(Q.T @ Q - np.eye(l)).max() < 1e-13 * l
    res = orc.residual(A, Q, out["T"], out["P"]) / np.linalg.norm(A)
    if kind == "rank_deficient":
        assert res < 1e-13


def test_corollary_expected_error_bound(orc):
    """Corollary (eq. (6)): E‖A−QLPᵀ‖_F ≤ (1+k/(p−1))^½ (Σ_{j>k} σ_j²)^½;
    sample mean over 20 seeds."""
    k, p = 10, 5
    sig = np.arange(1, 101.0) ** -1.0
    A = _rand_svd(150, 100, sig, 18)
    errs = []
    for s in range(20):
        out = orc.rqlp(A, k, p, q=0, d=0, seed=100 + s)
        errs.append(orc.residual(A, out["Q"], out["T"], out["P"]))
    bound = math.sqrt(1 + k / (p - 1)) * math.sqrt(np.sum(sig[k:] ** 2))
    assert np.mean(errs) <= bound


def test_rqlp_argument_errors(orc):
    A = np.zeros((10, 8))
    with pytest.raises(ValueError):
        orc.rqlp(A, k=1, p=5)         # k >= 2
    with pytest.raises(ValueError):
        orc.rqlp(A, k=4, p=1)         # p >= 2
    with pytest.raises(ValueError):
        orc.rqlp(A, k=6, p=4)         # ℓ > n


def test_zero_matrix(orc):
    """Zero A: τ = 0 reflectors, L = 0, identity pivots (reading R21)."""
    A = np.zeros((20, 15), order="F")
    out = orc.rqlp(A, k=3, p=2, q=0, d=0, seed=1)
    assert not out["T"].any()
    assert list(out["piv0"]) == [0, 1, 2, 3, 4]
    assert np.abs(out["Q"].T @ out["Q"] - np.eye(5)).max() < 1e-14


def test_sigma_helpers():
    s = sigma("poly2", 4).numpy()
    np.testing.assert_allclose(s, [1, 1 / 4, 1 / 9, 1 / 16])


# ------------------------------------------------------------------ NEXT-1: auto-rank RQLP
def test_autorank_indicator_is_direct_residual(orc):
    """The eq. (3) indicator, computed from ||A||^2 - sum ||B_j||^2, equals the
    directly computed ||A − QLPᵀ||_F / ||A||_F at every stopping point (catches a missing deflation
    of B_j, a wrong block offset, or an indicator on the wrong matrix)."""
    sig = np.exp(-np.arange(1, 151.0) / 15)
    A = _rand_svd(220, 150, sig, 41)
    nA = np.linalg.norm(A)
    prev = 0
    for eps in (1e-1, 1e-2, 1e-3):
        out = orc.autorank(A, b=8, l_max=144, eps=eps, q=1, seed=3)
        direct = orc.residual(A, out["Q"], out["T"], out["P"]) / nA
        assert out["err"] == pytest.approx(direct, rel=1e-6, abs=1e-13)
        assert out["err"] <= eps and out["l"] % 8 == 0 and out["l"] >= prev
        # one block fewer would not have met the tolerance (stops at the FIRST block)
        if out["l"] > 8:
            o2 = orc.autorank(A, b=8, l_max=out["l"] - 8, eps=0.0, q=1, seed=3)
            assert orc.residual(A, o2["Q"], o2["T"], o2["P"]) / nA > eps
        prev = out["l"]


def test_autorank_exact_rank(orc):
    """rank(A) = 24 = 3 blocks of 8: the indicator collapses to rounding at l = 24 and the loop
    stops there (a textbook property of the range finder on an exactly low-rank matrix)."""
    sig = np.linspace(4.0, 1.0, 24)
    A = _rand_svd(200, 140, sig, 42)
    out = orc.autorank(A, b=8, l_max=80, eps=1e-10, q=0, seed=5)
    assert out["l"] == 24
    assert out["err"] < 1e-12
    Q = out["Q"]
    assert np.abs(Q.T @ Q - np.eye(24)).max() < 1e-13 * 24
    np.testing.assert_allclose(Q @ out["T"] @ out["P"].T, A, atol=1e-12 * np.linalg.norm(A))


def test_autorank_limits_and_equivalence(orc):
    """eps >= 1 stops after one block; eps = 0 runs to l_max; the result at l_out is the
    BRQLP of Alg. 3 with k + p = l_out on the same Ω (Ω columns do not depend on l)."""
    sig = np.arange(1, 121.0) ** -1.5
    A = _rand_svd(180, 120, sig, 43)
    one = orc.autorank(A, b=10, l_max=60, eps=1.0, q=0, seed=8)
    assert one["l"] == 10
    full = orc.autorank(A, b=10, l_max=60, eps=0.0, q=0, seed=8)
    assert full["l"] == 60
    mid = orc.autorank(A, b=10, l_max=60, eps=3e-2, q=1, seed=8)
    assert 10 < mid["l"] < 60
    ref = orc.brqlp(A, k=mid["l"] - 2, p=2, b=10, q=1, seed=8)
    for key in ("Q", "T", "P"):
        np.testing.assert_allclose(mid[key], ref[key], atol=1e-13)
    assert np.array_equal(mid["piv0"], ref["piv0"]) and np.array_equal(mid["piv1"], ref["piv1"])


# ------------------------------------------------------------------ NEXT-3: truncated pivoted QLP
@pytest.mark.parametrize("m,n,l", [(90, 70, 12), (70, 90, 25), (60, 40, 40)])
def test_tqlp_matches_lapack_pivoted_qlp(orc, m, n, l):
    """Truncated pivoted QLP against LAPACK's dgeqp3 via scipy: pivots of the
    first l steps, pivots of the CPQR of [R11 R12]^T, |L-values|, and the residual
    ||(I - Q_R Q_R^T) A||_F (catches a wrong truncation, a transposed R, a wrong Π0/Π1 assembly)."""
    sig = 2.0 ** -np.arange(min(m, n), dtype=float) * (1 + 0.1 * np.arange(min(m, n)) % 3)
    A = _rand_svd(m, n, np.sort(sig)[::-1], m * n)
    o = orc.tqlp(A, l)
    Qs, Rs, ps = sla.qr(A, pivoting=True, mode="economic")
    assert np.array_equal(o["piv0"], ps[:l])
    R1 = Rs[:l, :]
    Q2, R2, p2 = sla.qr(R1.T, pivoting=True, mode="economic")
    assert np.array_equal(o["piv1"], p2)
    np.testing.assert_allclose(np.abs(np.diag(o["T"])), np.abs(np.diag(R2)), rtol=1e-10, atol=1e-14)
    assert not np.triu(o["T"], 1).any()
    Ql = Qs[:, :l]
    direct = np.linalg.norm(A - Ql @ (Ql.T @ A))
    assert orc.residual(A, o["Q"], o["T"], o["P"]) == pytest.approx(direct, rel=1e-8, abs=1e-14)
    assert np.abs(o["Q"].T @ o["Q"] - np.eye(l)).max() < 1e-13 * l
    assert np.abs(o["P"].T @ o["P"] - np.eye(l)).max() < 1e-13 * l


def test_tqlp_full_rank_is_exact(orc):
    """l = min(m, n): the pivoted QLP is an exact factorisation A = Q L P^T (eq. (1))."""
    A = _rand_svd(50, 35, np.logspace(0, -6, 35), 77)
    o = orc.tqlp(A, 35)
    np.testing.assert_allclose(o["Q"] @ o["T"] @ o["P"].T, A, atol=1e-14)


def test_erqlp_more_inner_qr_tracks_better(orc):
    """Theorem 2: more inner QR iterations give L-values closer to the
    singular values (quadratic improvement per step for gapped spectra).  Max relative L-value
    error over j <= k for d = 0, 2, 4, 6 on a gapped spectrum, fixed seed."""
    k, p = 12, 4
    sig = 0.6 ** np.arange(40.0)
    A = _rand_svd(120, 40, sig, 55)
    errs = []
    for d in (0, 2, 4, 6):
        out = orc.rqlp(A, k, p, q=1, d=d, seed=3)
        lv = np.abs(np.diag(out["T"]))[:k]
        errs.append(np.max(np.abs(lv - sig[:k]) / sig[:k]))
    assert errs[1] < errs[0] and errs[2] < errs[1] and errs[3] <= errs[2] * 1.01, errs
