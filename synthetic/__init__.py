"""Seeded synthetic input generators shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no Ω, no sketch, no QR of the method's
matrices): it only builds test matrices A = U·diag(σ)·Vᵀ (+ noise) with prescribed singular
values, shaped like the paper's test matrices (Example 1 "pds"/"eds") and
BASELINE.json's five configs.  Random numbers come from torch.Generator; orthonormal factors
come from torch.linalg.qr (LAPACK / cuSOLVER) with the Haar sign fix.

Matrices are returned column-major: a torch tensor of shape (m, n) with strides (1, m), i.e.
``At.T`` where ``At`` is a contiguous (n, m) tensor, so ``lda = m``.
"""
from .matrices import (  # noqa: F401
    CONFIGS,
    Config,
    col_major,
    config,
    eds_sigma,
    haar,
    make_A,
    make_A_config,
    pds_sigma,
    sigma,
    small_config,
)
