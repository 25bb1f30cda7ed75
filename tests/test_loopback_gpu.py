"""librqlp's row-sharded path at p > 1 ranks on ONE GPU: p loopback
handles (rqlp_create_loopback) act as the ranks -- one host thread per rank calls the real
rqlp_ex / erqlp_ex / brqlp_ex / rqlp_autorank_ex / rqlp_factorize with its row block of A; every
exchange step (Grams, A^T V, B = V^T A, ||A||^2) is a sum over the ranks in fixed rank order.
Graded against the oracle on the whole matrix at north_star tolerance (tests/parity.py), and the
replicated outputs (L/T, P, pivots) must be bitwise equal on every rank."""
import threading

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


_RARE_SEEN: dict = {}


def _rand_A(rng, m, n, sig):
    r = len(sig)
    U, _ = np.linalg.qr(rng.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return np.asfortranarray((U * sig) @ V.T)


def _blocks(m, p):
    from paper_1811_09334_b200.dist import row_block
    return [row_block(m, r, p) for r in range(p)]


def run_ranks(rq, A_np, p, call):
    """call(rank, A_block, handle) on p threads; returns the per-rank results in rank order."""
    A = torch.from_numpy(np.ascontiguousarray(A_np.T)).cuda().t()        # column-major, lda = m
    hs = rq.Handle.loopback(p)
    out, err = [None] * p, [None] * p

    def job(r, r0, r1):
        try:
            out[r] = call(r, A[r0:r1], hs[r])      # row block: a column-major view with lda = m
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ths = [threading.Thread(target=job, args=(r, r0, r1)) for r, (r0, r1) in enumerate(_blocks(A_np.shape[0], p))]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=900)
    torch.cuda.synchronize()
    for e in err:
        if e is not None:
            raise e
    flags = [h.sync() for h in hs]
    run_ranks.reruns = [h.careful_reruns() for h in hs]
    return out, flags


def _gather(out):
    g = dict(out[0])
    g["Q"] = torch.cat([o["Q"] for o in out], dim=0)
    return g


def _replicated_equal(out, keys):
    for o in out[1:]:
        for k in keys:
            if out[0].get(k) is not None:
                assert torch.equal(o[k], out[0][k]), f"replicated {k} differs between ranks"


VARIANTS = {
    "rqlp": dict(q=1, d=0),
    "erqlp": dict(q=2, d=2),
    "brqlp": dict(q=1, b=16),
    "brqlp_q0": dict(q=0, b=24),
}


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_loopback_ranks_match_oracle(rq, orc, p, variant):
    kw = VARIANTS[variant]
    rng = np.random.default_rng(100 + p)
    m, n, k, pp = 2003, 700, 56, 8            # ragged row blocks (m % p != 0 for p = 2, 4, 8)
    sig = np.exp(-np.arange(1, 501.0) / 60)
    A = _rand_A(rng, m, n, sig)
    out, flags = run_ranks(rq, A, p, lambda r, Ab, h: rq.factorize(Ab, k, pp, seed=9, handle=h, **kw))
    _replicated_equal(out, ("T", "P", "piv0", "piv1"))
    g = _gather(out)
    l = k + pp
    if "b" in kw:
        o = orc.brqlp(A, k, pp, b=kw["b"], q=kw["q"], seed=9, stages=True)
        check_factorization(orc, A, g, o, l, sig_ratio=sig[:l] / sig[0], block=kw["b"], B_oracle=o["V"].T @ A,
                            tag=f"loopback p={p} {variant}")
    else:
        o = orc.rqlp(A, k, pp, q=kw["q"], d=kw["d"], seed=9, stages=True)
        if kw["d"]:
            o["piv1"] = None
        check_factorization(orc, A, g, o, l, sig_ratio=sig[:l] / sig[0], B_oracle=o["B"],
                            tag=f"loopback p={p} {variant}")
    assert all(f == 0 for f in flags), flags
    assert run_ranks.reruns == [0] * p     # the optimistic run (no per-orth readback) stood


@pytest.mark.parametrize("p", [2, 3])
def test_loopback_autorank(rq, orc, p):
    """Auto-rank on row shards: ||A||_F^2 is a sum over ranks, the per-block indicator is read back
    on every rank (identical), and every rank stops at the same block as the oracle."""
    rng = np.random.default_rng(7)
    sig = np.exp(-np.arange(1, 401.0) / 30)
    A = _rand_A(rng, 1501, 600, sig)
    out, _ = run_ranks(rq, A, p, lambda r, Ab, h: rq.autorank(Ab, b=16, l_max=160, eps=1e-3, q=1, seed=4, handle=h))
    ls = {o["l"] for o in out}
    errs = {o["err"] for o in out}
    assert len(ls) == 1 and len(errs) == 1, (ls, errs)
    o = orc.autorank(A, 16, 160, 1e-3, q=1, seed=4)
    assert out[0]["l"] == o["l"]
    _replicated_equal(out, ("T", "P", "piv0", "piv1"))
    g = _gather(out)
    check_factorization(orc, A, g, o, o["l"], sig_ratio=sig[:o["l"]] / sig[0], block=16, tag=f"loopback autorank p={p}")
    assert out[0]["err"] == pytest.approx(o["err"], rel=1e-8, abs=1e-13)


@pytest.mark.parametrize("mode", ["optimistic", "careful"])
@pytest.mark.parametrize("kind", ["illcond", "deficient", "zero"])
def test_loopback_rare_branch(rq, orc, kind, mode, monkeypatch):
    """Sketches beyond CholeskyQR2's reach on 3 ranks: the host-driven shifted passes with summed
    Grams take the same decisions on every rank (identical COND words) and return an orthonormal
    Q with the oracle's residual.  optimistic (the default): the run without per-orth readbacks
    records the breakdown and every rank repeats the factorisation on the careful path;
    careful (RQLP_SHARDED_OPTIMISTIC=0): the careful path from the start -- bitwise the same result."""
    monkeypatch.setenv("RQLP_SHARDED_OPTIMISTIC", "1" if mode == "optimistic" else "0")
    rng = np.random.default_rng(11)
    m, n = 900, 400
    sig = {"illcond": np.logspace(0, -13, 16), "deficient": np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125]),
           "zero": np.zeros(4)}[kind]
    A = _rand_A(rng, m, n, sig)
    out, flags = run_ranks(rq, A, 3, lambda r, Ab, h: rq.factorize(Ab, 12, 4, q=1, d=0, seed=5, handle=h))
    _replicated_equal(out, ("T", "P", "piv0"))
    assert len(set(flags)) == 1 and flags[0] & 1, flags
    assert run_ranks.reruns == [1 if mode == "optimistic" else 0] * 3, run_ranks.reruns
    g = _gather(out)
    Q, T, P = (np.asfortranarray(g[k].cpu().numpy()) for k in ("Q", "T", "P"))
    key = (kind,)
    if key in _RARE_SEEN:   # the two modes end on the same careful path: identical bits
        for a, b in zip(_RARE_SEEN[key], (Q, T, P)):
            assert np.array_equal(a, b)
    _RARE_SEEN[key] = (Q, T, P)
    assert np.abs(Q.T @ Q - np.eye(16)).max() <= 1e-13 * 16
    assert np.abs(P.T @ P - np.eye(16)).max() <= 1e-13 * 16
    o = orc.rqlp(A, 12, 4, q=1, d=0, seed=5)
    r_g, r_o = orc.residual(A, Q, T, P), orc.residual(A, o["Q"], o["T"], o["P"])
    assert r_g <= 10 * r_o + 1e-13 * max(np.linalg.norm(A), 1.0)


@pytest.mark.parametrize("mode", ["optimistic", "careful"])
def test_loopback_rare_branch_brqlp(rq, orc, mode, monkeypatch):
    """BRQLP on a rank-6 matrix with l = 24 in blocks of 8 on 2 ranks: the blocks beyond rank(A) are
    rounding noise, their sketches break CholeskyQR2 -- the optimistic run must notice on every rank,
    the careful rerun must return an orthonormal Q (reading R28) and the oracle's residual."""
    monkeypatch.setenv("RQLP_SHARDED_OPTIMISTIC", "1" if mode == "optimistic" else "0")
    rng = np.random.default_rng(21)
    m, n = 700, 300
    sig = np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125])
    A = _rand_A(rng, m, n, sig)
    out, flags = run_ranks(rq, A, 2, lambda r, Ab, h: rq.factorize(Ab, 20, 4, q=1, b=8, seed=5, handle=h))
    _replicated_equal(out, ("T", "P", "piv0", "piv1"))
    assert len(set(flags)) == 1 and flags[0] & 1, flags
    assert run_ranks.reruns == [1 if mode == "optimistic" else 0] * 2, run_ranks.reruns
    g = _gather(out)
    Q, T, P = (np.asfortranarray(g[k].cpu().numpy()) for k in ("Q", "T", "P"))
    assert np.abs(Q.T @ Q - np.eye(24)).max() <= 1e-13 * 24
    o = orc.brqlp(A, 20, 4, b=8, q=1, seed=5)
    r_g, r_o = orc.residual(A, Q, T, P), orc.residual(A, o["Q"], o["T"], o["P"])
    assert r_g <= 10 * r_o + 1e-13 * np.linalg.norm(A)
    np.testing.assert_allclose(np.abs(np.diag(T))[:6], np.abs(np.diag(o["T"]))[:6], rtol=1e-8)


@pytest.mark.parametrize("variant", ["erqlp", "brqlp", "brqlp_q0"])
def test_loopback_replica_mismatch_is_flagged(rq, variant, monkeypatch):
    """The replicated tail relies on every rank holding the same bits of the summed B; the library
    compares a hash of B across the ranks after the sum.  With one rank pretending to hold other bits
    (RQLP_DEBUG_REPLICA_FLIP) EVERY rank must report RQLP_FLAG_REPLICA_MISMATCH (4); without it none
    does (the other loopback tests assert flags == 0)."""
    rng = np.random.default_rng(8)
    A = _rand_A(rng, 600, 300, np.arange(1, 201.0) ** -1.5)
    kw = dict(erqlp=dict(q=1, d=2), brqlp=dict(q=1, b=8), brqlp_q0=dict(q=0, b=8))[variant]
    monkeypatch.setenv("RQLP_DEBUG_REPLICA_FLIP", "1")
    _, flags = run_ranks(rq, A, 3, lambda r, Ab, h: rq.factorize(Ab, 20, 4, seed=5, handle=h, **kw))
    assert all(f & 4 for f in flags), flags
    monkeypatch.delenv("RQLP_DEBUG_REPLICA_FLIP")
    _, flags = run_ranks(rq, A, 3, lambda r, Ab, h: rq.factorize(Ab, 20, 4, seed=5, handle=h, **kw))
    assert all(f == 0 for f in flags), flags


def test_loopback_host_buffers(rq, orc):
    """rqlp_factorize (the e2e entry point) on loopback ranks with pinned host row blocks."""
    rng = np.random.default_rng(5)
    sig = np.arange(1, 301.0) ** -1.5
    A = _rand_A(rng, 1200, 500, sig)
    p, k, pp = 4, 30, 6
    l = k + pp
    hs = rq.Handle.loopback(p)
    res = [None] * p

    def job(r, r0, r1):
        Ah = torch.from_numpy(np.ascontiguousarray(A[r0:r1].T)).pin_memory().t()
        res[r] = rq.factorize_host(Ah, k, pp, q=1, d=2, seed=3, handle=hs[r])

    ths = [threading.Thread(target=job, args=(r, r0, r1)) for r, (r0, r1) in enumerate(_blocks(A.shape[0], p))]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    assert all(x is not None for x in res)
    for x in res[1:]:
        assert torch.equal(x[1], res[0][1]) and torch.equal(x[2], res[0][2])
    g = dict(Q=torch.cat([x[0] for x in res], 0), T=res[0][1], P=res[0][2], piv0=None)
    o = orc.rqlp(A, k, pp, q=1, d=2, seed=3)
    Q, T, P = (np.asfortranarray(g[k_].numpy()) for k_ in ("Q", "T", "P"))
    nA = np.linalg.norm(A)
    assert abs(orc.residual(A, Q, T, P) - orc.residual(A, o["Q"], o["T"], o["P"])) / nA <= 1e-12
    np.testing.assert_allclose(np.abs(np.diag(T)), np.abs(np.diag(o["T"])), rtol=1e-10)


def test_loopback_rank_failure_aborts_group(rq):
    """A rank whose call fails (too small a workspace) aborts the group: the other ranks' calls
    return an error instead of waiting forever."""
    rng = np.random.default_rng(1)
    A = _rand_A(rng, 400, 200, np.arange(1, 101.0) ** -1.0)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
    hs = rq.Handle.loopback(2)
    tiny = torch.empty(1024, dtype=torch.uint8, device="cuda")
    import ctypes
    rq.lib().rqlp_set_workspace(hs[1].h, ctypes.c_void_p(tiny.data_ptr()), 1024)
    hs[1]._ws_key = ("pinned",)           # keep the binding from replacing the tiny workspace
    errs = [None, None]

    def job(r, r0, r1):
        try:
            h = hs[r]
            Q = rq.cm_empty(r1 - r0, 20, "cuda")
            L = rq.cm_empty(20, 20, "cuda")
            P = rq.cm_empty(200, 20, "cuda")
            lib = rq.lib()
            Ab = At[r0:r1]
            if r == 0:
                h.workspace(rq.VARIANT_RQLP, r1 - r0, 200, 16, 4, 1, 0, 0)
            rc = lib.rqlp_ex(h.h, r1 - r0, 200, 16, 4, 1, ctypes.c_void_p(Ab.data_ptr()), 400, 1,
                             ctypes.c_void_p(Q.data_ptr()), r1 - r0, ctypes.c_void_p(L.data_ptr()), 20,
                             ctypes.c_void_p(P.data_ptr()), 200, None, None)
            errs[r] = rc
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ths = [threading.Thread(target=job, args=(r, r0, r1)) for r, (r0, r1) in enumerate(_blocks(400, 2))]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=120)
    assert errs[1] == 3          # RQLP_ERR_WORKSPACE on the failing rank
    assert errs[0] == 2          # RQLP_ERR_NCCL (group aborted) on the other
