"""Seeded randomized sweep of the whole factorisation against the oracle: shapes (tall, wide,
square, ragged against every tile size), k, p, q, d, b and spectra (polynomial, exponential,
gapped, numerically rank-deficient, exactly rank-deficient) drawn from a fixed seed.  Every case
checks the north_star tolerances where they are well defined and the basis-invariant quantities
(residual, orthonormality) everywhere (readings R4, R26).  The grading is tests/parity.py's:
identical pivots (or a near-tie of the oracle's candidate norms, reading R30 -- anything else
FAILS), L-values to max(1e-10 relative, C_L u |L_1|) (reading R29), Q, T, P element-wise, the
residual to 1e-12 -- with a residual slack only for numerically rank-deficient sketches (R4)."""
import os

import numpy as np
import pytest
import torch
from parity import check_factorization

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1811_09334_b200 as rq
    return rq


def _cm(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda().t()


def _np(t):
    return np.asfortranarray(t.detach().cpu().numpy())


# RQLP_SWEEP_OFFSET=<int> draws a different set of random cases (the extended sweeps recorded in
# profiles/r02_extended_sweep.txt); the default 0 is the suite's fixed set
_OFFSET = int(os.environ.get("RQLP_SWEEP_OFFSET", "0"))


def _case(i):
    rng = np.random.default_rng(1000 + i + _OFFSET)
    k = int(rng.integers(2, 40))
    p = int(rng.integers(2, 12))
    l = k + p
    m = int(rng.integers(l, 900))
    n = int(rng.integers(l, 700))
    q = int(rng.integers(0, 3))
    variant = ["rqlp", "erqlp", "brqlp"][int(rng.integers(0, 3))]
    d = int(rng.integers(1, 5)) if variant == "erqlp" else 0
    b = int(rng.integers(1, l + 1)) if variant == "brqlp" else None
    kind = ["poly", "exp", "gap", "numdef", "exactdef"][int(rng.integers(0, 5))]
    r = min(m, n)
    j = np.arange(1, r + 1.0)
    if kind == "poly":
        sig = j ** -float(rng.uniform(0.5, 2.5))
    elif kind == "exp":
        sig = np.exp(-j / float(rng.uniform(3, 60)))
    elif kind == "gap":
        sig = np.where(j <= k, 1.0, 1e-6) * j ** -1.0
    elif kind == "numdef":
        sig = np.where(j <= max(2, l // 2), j ** -1.0, 1e-17)
    else:
        sig = np.where(j <= max(2, l // 2), j ** -1.0, 0.0)
    U, _ = np.linalg.qr(rng.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    A = np.asfortranarray((U * sig) @ V.T)
    return dict(m=m, n=n, k=k, p=p, q=q, d=d, b=b, variant=variant, kind=kind, A=A, sig=sig, seed=int(rng.integers(0, 2**62)))


@pytest.mark.parametrize("i", range(96))
def test_random_sweep(rq, orc, i):
    c = _case(i)
    A, l = c["A"], c["k"] + c["p"]
    g = rq.factorize(_cm(A), c["k"], c["p"], q=c["q"], d=c["d"], b=c["b"], seed=c["seed"])
    if c["variant"] == "brqlp":
        o = orc.brqlp(A, c["k"], c["p"], b=c["b"], q=c["q"], seed=c["seed"], stages=True)
        B_o = o["V"].T @ A
    else:
        o = orc.rqlp(A, c["k"], c["p"], q=c["q"], d=c["d"], seed=c["seed"], stages=True)
        B_o = o["B"]
        if c["d"] >= 1:
            o["piv1"] = None
    tag = f"case {i}: {c['variant']} m={c['m']} n={c['n']} k={c['k']} p={c['p']} q={c['q']} d={c['d']} b={c['b']} {c['kind']}"
    _grade(orc, A, g, o, l, c["sig"], c["kind"], c["b"], B_o, tag)


def _grade(orc, A, g, o, l, sig, kind, block, B_o, tag):
    """Full grading where the factorisation is unique (a sketch of full numerical rank); the
    basis-invariant quantities (residual with the R4 slack, orthonormality) otherwise."""
    rank = int((sig > 1e-14 * sig[0]).sum())
    if rank >= l and kind in ("poly", "exp", "gap"):
        check_factorization(orc, A, g, o, l, sig_ratio=sig[:l] / sig[0], block=block, B_oracle=B_o, tag=tag)
        return
    Q, T, P = _np(g["Q"]), _np(g["T"]), _np(g["P"])
    nA = np.linalg.norm(A)
    rg, ro = orc.residual(A, Q, T, P) / nA, orc.residual(A, o["Q"], o["T"], o["P"]) / nA
    lq = Q.shape[1]
    assert np.abs(Q.T @ Q - np.eye(lq)).max() <= 1e-13 * lq, tag
    if block is None:   # BRQLP's P is orthonormal per block only (reading R17)
        assert np.abs(P.T @ P - np.eye(lq)).max() <= 1e-13 * lq, tag
    assert abs(rg - ro) <= 1e-12 or rg <= 2 * ro + 1e-14, (tag, rg, ro)


def _spectrum(rng, r, k, l):
    j = np.arange(1, r + 1.0)
    kind = ["poly", "exp", "gap", "numdef"][int(rng.integers(0, 4))]
    if kind == "poly":
        return kind, j ** -float(rng.uniform(0.5, 2.0))
    if kind == "exp":
        return kind, np.exp(-j / float(rng.uniform(10, 80)))
    if kind == "gap":
        return kind, np.where(j <= k, 1.0, 1e-6) * j ** -1.0
    return kind, np.where(j <= max(2, l // 2), j ** -1.0, 1e-17)


def _rand_A(rng, m, n, sig):
    r = len(sig)
    U, _ = np.linalg.qr(rng.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((U * sig) @ V.T)


@pytest.mark.parametrize("i", range(24))
def test_random_sweep_large(rq, orc, i):
    """Larger shapes (multi-tile GEMMs: split-K and the balanced split, the grid-mode CPQR engine
    with several columns per CTA, the blocked Cholesky for l > 128)."""
    rng = np.random.default_rng(5000 + i)
    k = int(rng.integers(20, 200))
    p = int(rng.integers(2, 16))
    l = k + p
    m = int(rng.integers(max(l, 1500), 4200))
    n = int(rng.integers(max(l, 1200), 3600))
    q = int(rng.integers(0, 2))
    d = int(rng.integers(0, 3))
    kind, sig = _spectrum(rng, min(m, n, 3 * l), k, l)
    A = _rand_A(rng, m, n, sig)
    seed = int(rng.integers(0, 2**62))
    g = rq.factorize(_cm(A), k, p, q=q, d=d, seed=seed)
    o = orc.rqlp(A, k, p, q=q, d=d, seed=seed, stages=True)
    if d >= 1:
        o["piv1"] = None
    tag = f"large {i}: m={m} n={n} k={k} p={p} q={q} d={d} {kind}"
    _grade(orc, A, g, o, l, sig, kind, None, o["B"], tag)


@pytest.mark.parametrize("i", range(24))
def test_random_sweep_autorank_tqlp(rq, orc, i):
    """Auto-rank RQLP (NEXT-1) and the truncated QLP (NEXT-3) on random shapes."""
    rng = np.random.default_rng(9000 + i)
    m = int(rng.integers(60, 900))
    n = int(rng.integers(60, 700))
    kind, sig = _spectrum(rng, min(m, n), 20, 40)
    A = _rand_A(rng, m, n, sig)
    nA = np.linalg.norm(A)
    if i % 2 == 0:
        b = int(rng.integers(1, 24))
        l_max = int(rng.integers(b, min(m, n) + 1))
        eps = float(10 ** rng.uniform(-6, -1))
        q = int(rng.integers(0, 3))
        seed = int(rng.integers(0, 2**62))
        g = rq.autorank(_cm(A), b=b, l_max=l_max, eps=eps, q=q, seed=seed)
        o = orc.autorank(A, b, l_max, eps, q=q, seed=seed)
        tag = f"autorank {i}: m={m} n={n} b={b} l_max={l_max} eps={eps:.1e} q={q} {kind}"
        assert g["l"] == o["l"], (tag, g["l"], o["l"])
        _grade(orc, A, g, o, g["l"], sig, kind, b, None, tag)
    else:
        l = int(rng.integers(2, min(m, n, 160) + 1))
        g = rq.tqlp(_cm(A), l)
        o = orc.tqlp(A, l)
        tag = f"tqlp {i}: m={m} n={n} l={l} {kind}"
        _grade(orc, A, g, o, l, sig, kind, None, A, tag)


def test_truncate_views(rq, orc):
    """Rank-k views: the truncated factors are views of the l-sized ones and the rank-k
    approximation error is bounded by the l-sized residual plus the dropped L-values; BRQLP
    truncation is refused off a block boundary."""
    rng = np.random.default_rng(7)
    sig = np.exp(-np.arange(1, 301.0) / 15)
    A = _rand_A(rng, 500, 300, sig)
    g = rq.factorize(_cm(A), 20, 8, q=1, d=2, seed=3)
    t = rq.truncate(g, 20)
    assert t["Q"].data_ptr() == g["Q"].data_ptr() and t["Q"].shape == (500, 20)
    Q, T, P = _np(t["Q"]), _np(t["T"]), _np(t["P"])
    nA = np.linalg.norm(A)
    err = np.linalg.norm(A - Q @ T @ P.T) / nA
    assert err <= 3 * sig[20] / sig[0] * np.sqrt(300) + orc.residual(A, _np(g["Q"]), _np(g["T"]), _np(g["P"])) / nA
    gb = rq.factorize(_cm(A), 24, 8, q=1, b=8, seed=3)
    assert rq.truncate(gb, 16, b=8)["T"].shape == (16, 16)
    with pytest.raises(ValueError):
        rq.truncate(gb, 20, b=8)


@pytest.mark.parametrize("i", range(24))
def test_random_sweep_large_blocks(rq, orc, i):
    """Larger BRQLP and auto-rank cases: many blocks (ragged last), q up to 2, l up to ~300 (the
    blocked Cholesky past 128 columns inside the block orths' reorthogonalisation)."""
    rng = np.random.default_rng(12000 + i)
    k = int(rng.integers(40, 260))
    p = int(rng.integers(2, 24))
    l = k + p
    m = int(rng.integers(max(l, 1200), 3600))
    n = int(rng.integers(max(l, 900), 2800))
    q = int(rng.integers(0, 3))
    b = int(rng.integers(8, min(150, l) + 1))   # 1 <= b <= l
    kind, sig = _spectrum(rng, min(m, n, 3 * l), k, l)
    A = _rand_A(rng, m, n, sig)
    seed = int(rng.integers(0, 2**62))
    nA = np.linalg.norm(A)
    tag = f"large-blocks {i}: m={m} n={n} k={k} p={p} q={q} b={b} {kind}"
    if i % 3 == 2:
        eps = float(10 ** rng.uniform(-5, -1))
        g = rq.autorank(_cm(A), b=b, l_max=l, eps=eps, q=q, seed=seed)
        o = orc.autorank(A, b, l, eps, q=q, seed=seed)
        assert g["l"] == o["l"], (tag, g["l"], o["l"])
        _grade(orc, A, g, o, g["l"], sig, kind, b, None, tag)
    else:
        g = rq.factorize(_cm(A), k, p, q=q, b=b, seed=seed)
        o = orc.brqlp(A, k, p, b=b, q=q, seed=seed, stages=True)
        _grade(orc, A, g, o, l, sig, kind, b, o["V"].T @ A, tag)


_EDGE = [(l, sh, q, d) for l in (4, 32, 33, 128, 129, 257) for sh in ("square", "tall", "wide", "l_plus_1")
         for (q, d) in ((0, 0), (2, 3))]


@pytest.mark.parametrize("l,shape,q,d", _EDGE)
def test_edge_shapes(rq, orc, l, shape, q, d):
    """Shapes at the path switches: m or n equal to l (square sketch / B), l at the one-warp CPQR
    limit (32/33), at the fused Cholesky limit (128/129), past the one-CTA engine (257)."""
    m, n = {"square": (l, l), "tall": (3 * l, l), "wide": (l, 3 * l), "l_plus_1": (l + 1, l + 1)}[shape]
    rng = np.random.default_rng(l * 7 + len(shape) + q + d)
    sig = np.exp(-np.arange(1, min(m, n) + 1.0) / max(4.0, l / 4))
    A = _rand_A(rng, m, n, sig)
    k, p = l - 2, 2
    g = rq.factorize(_cm(A), k, p, q=q, d=d, seed=5)
    o = orc.rqlp(A, k, p, q=q, d=d, seed=5, stages=True)
    if d >= 1:
        o["piv1"] = None
    tag = f"edge l={l} {shape} q={q} d={d}"
    check_factorization(orc, A, g, o, l, sig_ratio=sig[:l] / sig[0], B_oracle=o["B"], tag=tag)


def test_two_handles_on_two_streams_concurrently(rq):
    """Two handles on two CUDA streams run factorisations concurrently (cooperative engine and
    rescue launches, graph replays) and reproduce their sequential results bit for bit."""
    rng = np.random.default_rng(77)
    A1 = _cm(_rand_A(rng, 2048, 1500, np.exp(-np.arange(1, 1501.0) / 40)))
    A2 = _cm(_rand_A(rng, 1800, 1700, np.arange(1, 1701.0) ** -1.0))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h1, h2 = rq.Handle(stream=s1), rq.Handle(stream=s2)
    ref = []
    for A, h, kw in ((A1, h1, dict(q=1, d=2)), (A2, h2, dict(q=1, d=0))):
        g = rq.factorize(A, 90, 10, seed=4, handle=h, **kw)
        torch.cuda.synchronize()
        ref.append({k: g[k].clone() for k in ("Q", "T", "P", "piv0")})
    torch.cuda.synchronize()
    for _ in range(3):   # eager, capture, replay -- interleaved on the two streams
        with torch.cuda.stream(s1):
            g1 = rq.factorize(A1, 90, 10, q=1, d=2, seed=4, handle=h1)
        with torch.cuda.stream(s2):
            g2 = rq.factorize(A2, 90, 10, q=1, d=0, seed=4, handle=h2)
        torch.cuda.synchronize()
        for g, r in ((g1, ref[0]), (g2, ref[1])):
            for k in ("Q", "T", "P", "piv0"):
                assert torch.equal(g[k], r[k]), k
