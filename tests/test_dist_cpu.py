"""World-size-2 CPU (gloo) tests of the row-sharded host logic: the row partition,
the NCCL unique-id bootstrap over torch.distributed, the max-over-ranks timing reduction, shard
generation, and a model of the sharded exchange schedule (Gram / A^T V / V^T A row-sums, the
rest replicated) checked against the unsharded oracle."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_09334_b200.dist import exchange_unique_id, max_over_ranks, row_block


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    out = tempfile.mkdtemp()
    mp.spawn(_entry, args=(world, port, out, fn, args), nprocs=world, join=True)
    return [np.load(os.path.join(out, f"r{r}.npy"), allow_pickle=True).item() for r in range(world)]


def _entry(rank, world, port, out, fn, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = fn(rank, world, *args)
    finally:
        dist.destroy_process_group()
    np.save(os.path.join(out, f"r{rank}.npy"), res, allow_pickle=True)


def test_row_block_partition():
    for m in (1, 7, 4096, 1048577):
        for world in (1, 2, 3, 8):
            blocks = [row_block(m, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == m
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def _uid_job(rank, world):
    uid = exchange_unique_id()   # real librqlp rqlp_get_unique_id on rank 0 (works without a GPU)
    t = max_over_ranks(10.0 + rank)
    return {"uid": uid, "max": t}


def test_unique_id_exchange_and_max_gloo():
    res = _run(2, _uid_job)
    assert len(res[0]["uid"]) == 128 and res[0]["uid"] == res[1]["uid"]
    assert any(res[0]["uid"])
    assert res[0]["max"] == res[1]["max"] == 11.0


def _shard_job(rank, world, m, n):
    from synthetic import make_A, sigma
    r0, r1 = row_block(m, rank, world)
    A = make_A(m, n, sigma("inv", 40), rank=40, noise=1e-6, seed=3, row_range=(r0, r1), chunk=64)
    return {"rows": (r0, r1), "A": A.numpy().copy()}


def test_synthetic_shards_are_slices_of_the_global_matrix():
    from synthetic import make_A, sigma
    m, n = 301, 120
    res = _run(2, _shard_job, m, n)
    full = make_A(m, n, sigma("inv", 40), rank=40, noise=1e-6, seed=3, chunk=64).numpy()
    for r in res:
        r0, r1 = r["rows"]
        assert np.array_equal(r["A"], full[r0:r1])


def _model_job(rank, world, m, n, k, p, q, d, seed):
    """Model of librqlp's sharded schedule: local A-passes on the row block, row-sums (allreduce)
    at exactly the exchange points of api.cu/orth.cu, everything else replicated."""
    import oracle as orc
    from synthetic import make_A, sigma
    r0, r1 = row_block(m, rank, world)
    A = make_A(m, n, sigma("poly2", min(m, n)), seed=11, row_range=(r0, r1)).numpy()
    l = k + p

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    def cholqr2_sharded(Y):            # Gram row-sum, replicated Cholesky, local Y R^-1
        for _ in range(2):
            G = allreduce(Y.T @ Y)
            R = np.linalg.cholesky(G).T
            Y = Y @ np.linalg.inv(R)
        return Y

    Om = orc.omega(seed, n, l)                       # replicated (same seed on every rank)
    V = cholqr2_sharded(A @ Om)
    for _ in range(q):
        Z = allreduce(A.T @ V)                       # power step: A^T V row-sum
        W, _ = orc.hqr(Z)                            # replicated
        V = cholqr2_sharded(A @ W)
    B = allreduce(V.T @ A)                           # projection row-sum
    t = orc.qlp_tail(B, d=d)                         # replicated tail (identical bits everywhere)
    Q = V @ t["QB"]                                  # local rows of Q
    return {"rows": (r0, r1), "Q": Q, "T": t["T"], "P": t["PB"], "piv0": t["piv0"]}


@pytest.mark.parametrize("q,d", [(0, 0), (1, 2)])
def test_sharded_schedule_matches_unsharded_oracle(q, d):
    import oracle as orc
    from synthetic import make_A, sigma
    m, n, k, p, seed = 401, 150, 12, 4, 5
    res = _run(2, _model_job, m, n, k, p, q, d, seed)
    A = make_A(m, n, sigma("poly2", min(m, n)), seed=11).numpy()
    o = orc.rqlp(np.asfortranarray(A), k, p, q=q, d=d, seed=seed)
    for r in res:  # replicated outputs identical on every rank
        assert np.array_equal(r["T"], res[0]["T"]) and np.array_equal(r["piv0"], res[0]["piv0"])
    assert np.array_equal(res[0]["piv0"], o["piv0"])
    np.testing.assert_allclose(np.diag(res[0]["T"]), np.diag(o["T"]), rtol=1e-10)
    Q = np.vstack([r["Q"] for r in sorted(res, key=lambda r: r["rows"][0])])
    np.testing.assert_allclose(Q, o["Q"], atol=1e-11)
    np.testing.assert_allclose(res[0]["P"], o["P"], atol=1e-11)
