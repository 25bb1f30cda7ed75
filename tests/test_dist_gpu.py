"""The row-sharded NCCL path of librqlp on one GPU (world size 1): rqlp_create_dist, the NCCL
allreduces at every exchange point (Grams, A^T V, B) and the replicated tail.  With one rank the
sums are identities, so the results must be bit-identical to the single-GPU handle."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def world1():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    if own:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["rqlp", "erqlp", "brqlp", "autorank"])
def test_nccl_world1_bit_identical(world1, variant):
    dist = world1
    import paper_1811_09334_b200 as rq
    rng = np.random.default_rng(3)
    U, _ = np.linalg.qr(rng.standard_normal((1200, 300)))
    V, _ = np.linalg.qr(rng.standard_normal((500, 300)))
    A = torch.from_numpy(np.ascontiguousarray(((U * np.arange(1, 301.0) ** -1.5) @ V.T).T)).cuda().t()
    hd = rq.Handle(group=dist.group.WORLD)
    if variant == "autorank":   # the sharded path also allreduces ||A||_F^2
        g1 = rq.autorank(A, b=16, l_max=64, eps=1e-3, q=1, seed=5, handle=hd)
        g0 = rq.autorank(A, b=16, l_max=64, eps=1e-3, q=1, seed=5, handle=rq.Handle())
        assert g0["l"] == g1["l"] and g0["err"] == g1["err"]
    else:
        kw = dict(rqlp=dict(q=1), erqlp=dict(q=1, d=2), brqlp=dict(q=1, b=16))[variant]
        g1 = rq.factorize(A, 40, 8, seed=5, handle=hd, **kw)
        g0 = rq.factorize(A, 40, 8, seed=5, handle=rq.Handle(), **kw)
    torch.cuda.synchronize()
    for key in ("Q", "T", "P", "piv0"):
        assert torch.equal(g0[key], g1[key]), key
    assert hd.careful_reruns() == 0


@pytest.mark.parametrize("variant", ["erqlp", "brqlp"])
def test_nccl_world1_graph_replay(world1, variant, monkeypatch):
    """RQLP_SHARDED_GRAPHS=1 (opt-in): the optimistic sharded run, ncclAllReduce calls included, is
    captured on the second call and replayed from the third; every call returns the bits of the
    single-GPU handle, and a sketch that breaks CholeskyQR2 still ends on the careful path."""
    dist = world1
    import paper_1811_09334_b200 as rq
    monkeypatch.setenv("RQLP_SHARDED_GRAPHS", "1")
    rng = np.random.default_rng(4)
    U, _ = np.linalg.qr(rng.standard_normal((1500, 200)))
    V, _ = np.linalg.qr(rng.standard_normal((600, 200)))
    A = torch.from_numpy(np.ascontiguousarray(((U * np.arange(1, 201.0) ** -1.2) @ V.T).T)).cuda().t()
    kw = dict(erqlp=dict(q=1, d=2), brqlp=dict(q=1, b=16))[variant]
    g0 = rq.factorize(A, 40, 8, seed=5, handle=rq.Handle(), **kw)
    hd = rq.Handle(group=dist.group.WORLD)
    g1 = None
    for _ in range(4):       # eager, capture + replay, replay, replay (the freed outputs are handed out
        g1 = None            # again by the caching allocator: same pointers, same graph key)
        g1 = rq.factorize(A, 40, 8, seed=5, handle=hd, **kw)
        torch.cuda.synchronize()
        for key in ("Q", "T", "P", "piv0"):
            assert torch.equal(g0[key], g1[key]), key
    assert hd.careful_reruns() == 0


@pytest.mark.parametrize("kind", ["illcond", "deficient", "zero"])
@pytest.mark.parametrize("d", [0, 2])
def test_nccl_world1_rare_branch(world1, kind, d):
    """Sketches beyond CholeskyQR2's reach on the row-sharded path: its host-driven shifted passes
    (allreduced Grams) must give an orthonormal Q and the residual of the single-GPU handle
    (whose rescue is one cooperative kernel -- same algorithm, different reduction order)."""
    dist = world1
    import oracle as orc

    import paper_1811_09334_b200 as rq
    rng = np.random.default_rng(11)
    m, n = 600, 400
    sig = {"illcond": np.logspace(0, -13, 16), "deficient": np.array([3.0, 2.0, 1.0, 0.5, 0.25, 0.125]),
           "zero": np.zeros(4)}[kind]
    U, _ = np.linalg.qr(rng.standard_normal((m, len(sig))))
    V, _ = np.linalg.qr(rng.standard_normal((n, len(sig))))
    A_np = np.asfortranarray((U * sig) @ V.T)
    A = torch.from_numpy(np.ascontiguousarray(A_np.T)).cuda().t()
    hd = rq.Handle(group=dist.group.WORLD)
    g1 = rq.factorize(A, 12, 4, q=1, d=d, seed=5, handle=hd)
    flags = hd.sync()
    assert hd.careful_reruns() == 1   # the optimistic run recorded the breakdown -> careful rerun
    g0 = rq.factorize(A, 12, 4, q=1, d=d, seed=5, handle=rq.Handle())
    torch.cuda.synchronize()
    Q1, T1, P1 = (np.asfortranarray(g1[k].cpu().numpy()) for k in ("Q", "T", "P"))
    Q0, T0, P0 = (np.asfortranarray(g0[k].cpu().numpy()) for k in ("Q", "T", "P"))
    assert np.abs(Q1.T @ Q1 - np.eye(16)).max() <= 1e-13 * 16
    assert np.abs(P1.T @ P1 - np.eye(16)).max() <= 1e-13 * 16
    r1, r0 = orc.residual(A_np, Q1, T1, P1), orc.residual(A_np, Q0, T0, P0)
    assert r1 <= 10 * r0 + 1e-13 * max(np.linalg.norm(A_np), 1.0)
    assert flags & 1  # the shifted passes ran
    k = len(sig) if kind != "illcond" else 6
    if kind != "zero":
        np.testing.assert_allclose(np.abs(np.diag(T1))[:k], np.abs(np.diag(T0))[:k], rtol=1e-8)


def test_nccl_world1_graph_replay_rare_branch(world1, monkeypatch):
    """With RQLP_SHARDED_GRAPHS=1 a sketch beyond CholeskyQR2's reach sets the sticky word in the
    eager run AND in every replay: each call is repeated on the careful path and returns the same
    bits as the careful path from the start."""
    dist = world1
    import paper_1811_09334_b200 as rq
    rng = np.random.default_rng(11)
    sig = np.logspace(0, -13, 16)
    U, _ = np.linalg.qr(rng.standard_normal((600, 16)))
    V, _ = np.linalg.qr(rng.standard_normal((400, 16)))
    A = torch.from_numpy(np.ascontiguousarray(((U * sig) @ V.T).T)).cuda().t()
    monkeypatch.setenv("RQLP_SHARDED_OPTIMISTIC", "0")
    ref = rq.factorize(A, 12, 4, q=1, d=2, seed=5, handle=rq.Handle(group=dist.group.WORLD))
    torch.cuda.synchronize()
    monkeypatch.setenv("RQLP_SHARDED_OPTIMISTIC", "1")
    monkeypatch.setenv("RQLP_SHARDED_GRAPHS", "1")
    hd = rq.Handle(group=dist.group.WORLD)
    g1 = None
    for i in range(3):
        g1 = None
        g1 = rq.factorize(A, 12, 4, q=1, d=2, seed=5, handle=hd)
        assert hd.sync() & 1
        assert hd.careful_reruns() == i + 1
        for key in ("Q", "T", "P", "piv0"):
            assert torch.equal(ref[key], g1[key]), key
