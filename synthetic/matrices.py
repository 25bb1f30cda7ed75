"""Test-matrix construction (see package docstring).  No RQLP arithmetic lives here."""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (or a scaled-down parity variant of it)."""

    name: str
    m: int
    n: int
    k: int
    p: int
    q: int
    d: int                 # 0 = RQLP (Alg. 1); >= 1 = ERQLP inner QR iterations (Alg. 2)
    b: int | None          # block size for BRQLP (Alg. 3), None otherwise
    spectrum: str          # "poly2" | "exp50" | "inv" | "exp100" | "poly1.5"
    rank: int | None       # r of the low-rank part (None = full SVD form)
    noise: float           # coefficient c of c·G, G_ij ~ N(0, 1/n)
    seed: int

    @property
    def l(self) -> int:
        return self.k + self.p

    @property
    def variant(self) -> str:
        if self.b is not None:
            return "brqlp"
        return "erqlp" if self.d >= 1 else "rqlp"


def sigma(spectrum: str, count: int, dtype=torch.float64) -> torch.Tensor:
    """Singular values σ_1..σ_count of BASELINE.json's configs (1-based j)."""
    j = torch.arange(1, count + 1, dtype=dtype)
    if spectrum == "poly2":      # C1: σ_j = j^-2 (pds with t=1, s=2)
        return j ** -2.0
    if spectrum == "exp50":      # C2: σ_j = exp(-j/50) (eds family)
        return torch.exp(-j / 50.0)
    if spectrum == "inv":        # C3: σ_j = 1/j
        return 1.0 / j
    if spectrum == "exp100":     # C4: σ_j = exp(-j/100)
        return torch.exp(-j / 100.0)
    if spectrum == "poly1.5":    # C5: σ_j = j^-1.5
        return j ** -1.5
    if spectrum == "gap":        # test helper: σ_j = 2^-j (gapped, Huckaby-Chan pin)
        return 2.0 ** (-j)
    raise ValueError(spectrum)


def pds_sigma(n: int, t: int, s: float) -> torch.Tensor:
    """Polynomially decaying spectrum: diag(1,..,1, 2^-s, 3^-s, .., (n-t+1)^-s)."""
    tail = torch.arange(2, n - t + 2, dtype=torch.float64) ** (-s)
    return torch.cat([torch.ones(t, dtype=torch.float64), tail])[:n]


def eds_sigma(n: int, t: int, s: float) -> torch.Tensor:
    """Exponentially decaying spectrum: diag(1,..,1, 2^-s, 2^-2s, .., 2^-(n-t)s)."""
    tail = 2.0 ** (-s * torch.arange(1, n - t + 1, dtype=torch.float64))
    return torch.cat([torch.ones(t, dtype=torch.float64), tail])[:n]


def haar(rows: int, cols: int, gen: torch.Generator, device="cpu") -> torch.Tensor:
    """Orthonormal rows x cols from the Householder QR of an N(0,1) matrix, columns signed by
    sign(R_ii).  Returned row-major contiguous (rows, cols)."""
    G = torch.randn(rows, cols, generator=gen, dtype=torch.float64, device=device)
    Q, R = torch.linalg.qr(G, mode="reduced")
    s = torch.sign(torch.diagonal(R))
    s[s == 0] = 1.0
    del G, R
    return Q * s


def col_major(At: torch.Tensor) -> torch.Tensor:
    """(n, m) contiguous -> (m, n) column-major view (lda = m)."""
    return At.t()


def make_A(m: int, n: int, sig: torch.Tensor, rank: int | None = None, noise: float = 0.0,
           seed: int = 0, device="cpu", row_range: tuple[int, int] | None = None,
           chunk: int = 8192) -> torch.Tensor:
    """A = U_r diag(σ) V_rᵀ + noise·G with G_ij ~ N(0, 1/n); column-major (m, n) tensor.

    ``row_range=(r0, r1)`` returns only rows r0..r1-1 of the global A (row-sharded runs);
    U_r is generated globally so every shard is a slice of the same matrix.
    """
    r = min(m, n) if rank is None else rank
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(int(seed) * 7919 + 17)
    U = haar(m, r, g, dev)                      # m x r
    V = haar(n, r, g, dev)                      # n x r
    s = sig[:r].to(device=dev, dtype=torch.float64)
    r0, r1 = (0, m) if row_range is None else row_range
    Ul = U[r0:r1]
    del U
    At = torch.empty(n, r1 - r0, dtype=torch.float64, device=dev)   # A^T, row-major == A col-major
    Vs = V * s
    for c0 in range(0, r1 - r0, chunk):
        c1 = min(r1 - r0, c0 + chunk)
        torch.matmul(Vs, Ul[c0:c1].t(), out=At[:, c0:c1])
    if noise != 0.0:
        gn = torch.Generator(device=dev)
        # noise rows are generated in fixed global chunks, each from its own seed, so a shard's bits
        # do not depend on the sharding and a row block never generates the other blocks' noise
        scale = noise / math.sqrt(n)
        for g0 in range(0, m, chunk):
            g1 = min(m, g0 + chunk)
            a0, a1 = max(g0, r0), min(g1, r1)
            if a0 >= a1:
                continue
            gn.manual_seed(int(seed) * 104729 + 3 + 7 * (g0 // chunk))
            G = torch.randn(n, g1 - g0, generator=gn, dtype=torch.float64, device=dev)
            At[:, a0 - r0:a1 - r0].add_(G[:, a0 - g0:a1 - g0], alpha=scale)
            del G
    return col_major(At)


# BASELINE.json "configs" (index 0..4).  C1 is quoted both as RQLP q=0 and ERQLP q=1.
CONFIGS: dict[str, Config] = {
    "c1": Config("c1", 1000, 800, 20, 5, 0, 0, None, "poly2", None, 0.0, 1),
    "c1e": Config("c1e", 1000, 800, 20, 5, 1, 2, None, "poly2", None, 0.0, 1),
    "c2": Config("c2", 4096, 4096, 100, 10, 1, 2, None, "exp50", None, 0.0, 2),
    "c3": Config("c3", 65536, 8192, 256, 16, 2, 2, None, "inv", 512, 1e-6, 3),
    "c4": Config("c4", 262144, 16384, 512, 16, 1, 0, 64, "exp100", 1024, 1e-8, 4),
    "c5": Config("c5", 1048576, 16384, 1024, 32, 2, 2, None, "poly1.5", 2048, 1e-6, 5),
    "c5w": Config("c5w", 131072, 16384, 1024, 32, 2, 2, None, "poly1.5", 2048, 1e-6, 5),
}


def config(name: str) -> Config:
    return CONFIGS[name]


def small_config(name: str) -> Config:
    """Scaled-down variant of a config that the CPU oracle finishes in seconds, keeping its
    spectrum family, q, d, b and a ragged (non tile-multiple) m, n, ℓ."""
    c = CONFIGS[name]
    small = {
        "c1": dict(m=1000, n=800),
        "c1e": dict(m=1000, n=800),
        "c2": dict(m=1031, n=1030, k=100, p=10),
        "c3": dict(m=4133, n=1029, k=122, p=16, rank=300),
        "c4": dict(m=4133, n=1029, k=120, p=16, rank=300),
        "c5": dict(m=4133, n=1029, k=200, p=32, rank=400),
        "c5w": dict(m=4133, n=1029, k=200, p=32, rank=400),
    }[name]
    return dataclasses.replace(c, name=c.name + "_small", **small)


def make_A_config(c: Config, device="cpu", row_range=None) -> torch.Tensor:
    r = c.rank if c.rank is not None else min(c.m, c.n)
    return make_A(c.m, c.n, sigma(c.spectrum, r), rank=r, noise=c.noise, seed=c.seed, device=device,
                  row_range=row_range)
