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
