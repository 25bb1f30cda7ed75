"""paper_1811_09334_b200 -- B200-native (sm_100a) FP64 randomized QLP (arXiv:1811.09334).

Thin Python binding of librqlp.so (include/rqlp.h): argument marshalling only.  Every step of
RQLP / ERQLP / BRQLP runs in the library's CUDA kernels; PyTorch provides device memory,
streams and process groups.  There is no CPU fallback: if librqlp.so is missing or the device is
not a B200 the calls raise.

Matrices are column-major FP64 CUDA tensors: shape (rows, cols) with stride (1, ld), e.g.
``A = At.t()`` for a contiguous (n, m) tensor ``At`` (see ``col_major`` / ``cm_empty``).
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _capi

__all__ = ["Handle", "RQLPError", "rqlp", "erqlp", "brqlp", "factorize", "factorize_host", "autorank", "tqlp",
           "truncate",
           "omega", "gemm_nn", "gemm_tn", "orth", "cpqr", "qlp_tail", "residual", "rqlp_host", "cm_empty",
           "col_major", "lib", "VARIANT_RQLP", "VARIANT_ERQLP", "VARIANT_BRQLP"]

VARIANT_RQLP, VARIANT_ERQLP, VARIANT_BRQLP = 0, 1, 2
FLAG_SHIFTED_CHOLQR = 1


class RQLPError(RuntimeError):
    pass


def lib():
    return _capi.load()


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().rqlp_strerror(rc).decode()
        raise RQLPError(f"{what} failed: rc={rc} ({msg})")


def cm_empty(rows: int, cols: int, device, dtype=torch.float64) -> torch.Tensor:
    """Uninitialised column-major (rows, cols) tensor, ld = rows."""
    return torch.empty(cols, rows, dtype=dtype, device=device).t()


def col_major(t: torch.Tensor) -> torch.Tensor:
    """Column-major copy/view of a 2-D tensor."""
    if t.dim() == 2 and t.stride(0) == 1 and (t.shape[1] <= 1 or t.stride(1) >= max(1, t.shape[0])):
        return t
    return t.t().contiguous().t()


def _ld(t: torch.Tensor) -> int:
    if t.stride(0) != 1 and t.shape[0] > 1:
        raise ValueError("tensor must be column-major (stride(0) == 1)")
    return max(1, t.shape[0]) if t.shape[1] <= 1 else t.stride(1)


def _mat(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2:
        raise TypeError(f"{name} must be a 2-D float64 CUDA tensor")
    return t if t.stride(0) == 1 or t.shape[0] <= 1 else col_major(t)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class Handle:
    """librqlp handle bound to one device and one CUDA stream; owns a torch workspace tensor."""

    _cache: dict = {}
    _lock = threading.Lock()

    def __init__(self, device=None, stream=None, group=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        if group is None:
            _check(lib().rqlp_create(ctypes.byref(h), self.device.index, ctypes.c_void_p(self.stream.cuda_stream)),
                   "rqlp_create")
            self.rank, self.nranks = 0, 1
        else:
            import torch.distributed as dist

            from .dist import exchange_unique_id
            self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
            raw = ctypes.create_string_buffer(exchange_unique_id(group), 128)
            _check(lib().rqlp_create_dist(ctypes.byref(h), self.device.index,
                                          ctypes.c_void_p(self.stream.cuda_stream), raw, self.rank, self.nranks),
                   "rqlp_create_dist")
        self.h = h
        self._ws = None
        self.group = group

    @classmethod
    def loopback(cls, nranks: int, device=None, stream=None) -> list["Handle"]:
        """`nranks` virtual ranks of a row-sharded run in THIS process on ONE GPU
        (rqlp_create_loopback): one handle per rank, all on one stream.  Call the factorisations
        collectively, one host thread per rank, each with its rank's row block of A; the sums over
        ranks run in fixed rank order (bit-identical replicated outputs)."""
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        stream = stream if stream is not None else torch.cuda.current_stream(dev)
        arr = (ctypes.c_void_p * nranks)()
        _check(lib().rqlp_create_loopback(arr, nranks, dev.index, ctypes.c_void_p(stream.cuda_stream)),
               "rqlp_create_loopback")
        hs = []
        for r in range(nranks):
            h = cls.__new__(cls)
            h.device, h.stream, h.h, h._ws, h.group = dev, stream, ctypes.c_void_p(arr[r]), None, None
            h.rank, h.nranks = r, nranks
            hs.append(h)
        return hs

    @classmethod
    def default(cls, device=None) -> "Handle":
        dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
        stream = torch.cuda.current_stream(dev)
        key = (dev, stream.cuda_stream)
        with cls._lock:
            if key not in cls._cache:
                cls._cache[key] = cls(device=torch.device("cuda", dev), stream=stream)
            return cls._cache[key]

    def workspace(self, variant, m, n, k, p, q, d, b):
        key = (variant, m, n, k, p, q, d, b or 0)
        if key == getattr(self, "_ws_key", None):   # same problem, workspace already attached
            return
        sz = ctypes.c_size_t()
        _check(lib().rqlp_workspace_size(self.h, variant, m, n, k, p, q, d, b or 0, ctypes.byref(sz)),
               "rqlp_workspace_size")
        need = sz.value
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        _check(lib().rqlp_set_workspace(self.h, ctypes.c_void_p(self._ws.data_ptr()), self._ws.numel()),
               "rqlp_set_workspace")
        self._ws_key = key

    def clear_workspace(self):
        self._ws_key = None
        _check(lib().rqlp_set_workspace(self.h, None, 0), "rqlp_set_workspace")

    def sync(self) -> int:
        f = ctypes.c_uint(0)
        _check(lib().rqlp_sync(self.h, ctypes.byref(f)), "rqlp_sync")
        return f.value

    def indicator(self) -> dict:
        """eq. (3) of the last factorisation on this handle: ||A||_F^2, ||B||_F^2 (BRQLP: sum of the
        deflated ||B_j||_F^2) and err = sqrt(max(0, a2 - b2)) / ||A||_F."""
        a2, b2 = ctypes.c_double(0.0), ctypes.c_double(0.0)
        _check(lib().rqlp_get_indicator(self.h, ctypes.byref(a2), ctypes.byref(b2)), "rqlp_get_indicator")
        a, b = a2.value, b2.value
        return {"a2": a, "b2": b, "err": (max(0.0, a - b) ** 0.5 / a ** 0.5) if a > 0 else 0.0}

    def set_timing(self, on: bool):
        _check(lib().rqlp_set_timing(self.h, 1 if on else 0), "rqlp_set_timing")

    def timing(self) -> list[tuple[str, float]]:
        cap = 256
        names = (ctypes.c_char_p * cap)()
        ms = (ctypes.c_float * cap)()
        nout = lib().rqlp_get_timing(self.h, names, ms, cap)
        if nout < 0:
            raise RQLPError(f"rqlp_get_timing rc={-nout}")
        return [(names[i].decode(), float(ms[i])) for i in range(min(nout, cap))]

    def set_stage_outputs(self, Y=None, V=None, B=None):
        """Tests: copy the sketch Y, final V and projected B of subsequent factorisations."""
        _check(lib().rqlp_set_stage_outputs(self.h, _ptr(Y), _ld(Y) if Y is not None else 0, _ptr(V),
                                            _ld(V) if V is not None else 0, _ptr(B),
                                            _ld(B) if B is not None else 0), "rqlp_set_stage_outputs")

    def set_power_stage_outputs(self, Vpre=None, Z=None, W=None, Ypow=None):
        """Tests: copy each power step's V (before), Z = A^T V, W = orth(Z) and Y = A W of subsequent
        factorisations (iteration it at columns it*l ..; see rqlp.h)."""
        ld = lambda t: _ld(t) if t is not None else 0  # noqa: E731
        _check(lib().rqlp_set_power_stage_outputs(self.h, _ptr(Vpre), ld(Vpre), _ptr(Z), ld(Z), _ptr(W), ld(W),
                                                  _ptr(Ypow), ld(Ypow)), "rqlp_set_power_stage_outputs")

    def launches(self) -> int:
        return int(lib().rqlp_launch_count(self.h))

    def careful_reruns(self) -> int:
        """Row-sharded handles: factorisations repeated on the careful path after a Cholesky
        breakdown in the optimistic run (rqlp_careful_rerun_count)."""
        return int(lib().rqlp_careful_rerun_count(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                lib().rqlp_destroy(self.h)
        except Exception:
            pass


def _handle(handle):
    return handle if handle is not None else Handle.default()


class _ordered:
    """Stream ordering between torch's current stream and the handle's stream: the library's work
    starts after everything already enqueued on the current stream (inputs, the outputs' and the
    workspace's allocations) and the current stream waits for the library's work before it uses
    the outputs or lets the caching allocator recycle any of these buffers."""

    def __init__(self, h: "Handle"):
        self.h = h

    def __enter__(self):
        self.cur = torch.cuda.current_stream(self.h.device)
        self.same = self.cur.cuda_stream == self.h.stream.cuda_stream
        if not self.same:
            self.h.stream.wait_stream(self.cur)
        return self

    def __exit__(self, *exc):
        if not self.same:
            self.cur.wait_stream(self.h.stream)
        return False


def _outputs(m: int, n: int, l: int, npiv: int, device):
    """Q (m x l), T (l x l), P (n x l) column-major and `npiv` int64 pivot vectors of length l,
    carved from ONE allocation (a call's host cost is dominated by allocations at small sizes)."""
    tot = (m + l + n + npiv) * l
    buf = torch.empty(tot, dtype=torch.float64, device=device)
    out = [buf.as_strided((m, l), (1, m), 0), buf.as_strided((l, l), (1, l), m * l),
           buf.as_strided((n, l), (1, n), (m + l) * l)]
    if npiv:
        bi = buf.view(torch.int64)
        out += [bi.as_strided((l,), (1,), (m + l + n + i) * l) for i in range(npiv)]
    return out


# ------------------------------------------------------------------ factorisations
def rqlp(A: torch.Tensor, k: int, p: int, q: int = 0, seed: int = 0, handle: Handle | None = None):
    """RQLP (Alg. 1) + q subspace iterations.  Returns Q (m x l), L (l x l lower),
    P (n x l), piv0 (l), piv1 (l) with A ~= Q L P^T."""
    A = _mat(A, "A")
    h = _handle(handle)
    m, n = A.shape
    l = k + p
    h.workspace(VARIANT_RQLP, m, n, k, p, q, 0, 0)
    Q, L, P, piv0, piv1 = _outputs(m, n, l, 2, A.device)
    with _ordered(h):
        _check(lib().rqlp_ex(h.h, m, n, k, p, q, _ptr(A), _ld(A), seed, _ptr(Q), _ld(Q), _ptr(L), _ld(L), _ptr(P), _ld(P),
                             _ptr(piv0), _ptr(piv1)), "rqlp_ex")
    return Q, L, P, piv0, piv1


def erqlp(A: torch.Tensor, k: int, p: int, q: int = 0, d: int = 2, seed: int = 0, handle: Handle | None = None):
    """ERQLP (Alg. 2, corrected assembly) + q subspace iterations.  Returns
    Q, T, P, piv0, t_is_upper with A ~= Q T P^T."""
    A = _mat(A, "A")
    h = _handle(handle)
    m, n = A.shape
    l = k + p
    h.workspace(VARIANT_ERQLP, m, n, k, p, q, d, 0)
    Q, T, P, piv0 = _outputs(m, n, l, 1, A.device)
    tu = ctypes.c_int(0)
    with _ordered(h):
        _check(lib().erqlp_ex(h.h, m, n, k, p, q, d, _ptr(A), _ld(A), seed, _ptr(Q), _ld(Q), _ptr(T), _ld(T),
                              ctypes.byref(tu), _ptr(P), _ld(P), _ptr(piv0)), "erqlp_ex")
    return Q, T, P, piv0, bool(tu.value)


def brqlp(A: torch.Tensor, k: int, p: int, b: int, q: int = 0, seed: int = 0, handle: Handle | None = None):
    """BRQLP (Alg. 3) + q deflated subspace iterations per block."""
    A = _mat(A, "A")
    h = _handle(handle)
    m, n = A.shape
    l = k + p
    h.workspace(VARIANT_BRQLP, m, n, k, p, q, 0, b)
    Q, L, P, piv0, piv1 = _outputs(m, n, l, 2, A.device)
    with _ordered(h):
        _check(lib().brqlp_ex(h.h, m, n, k, p, b, q, _ptr(A), _ld(A), seed, _ptr(Q), _ld(Q), _ptr(L), _ld(L), _ptr(P),
                              _ld(P), _ptr(piv0), _ptr(piv1)), "brqlp_ex")
    return Q, L, P, piv0, piv1


def factorize(A, k, p, q=0, d=0, b=None, seed=0, handle=None) -> dict:
    """Dispatch: b -> BRQLP, d >= 1 -> ERQLP, else RQLP.  Returns a dict with Q, T, P, piv0,
    piv1 (None for ERQLP) and t_is_upper."""
    if b is not None:
        Q, L, P, p0, p1 = brqlp(A, k, p, b, q, seed, handle)
        return dict(Q=Q, T=L, P=P, piv0=p0, piv1=p1, t_is_upper=False)
    if d >= 1:
        Q, T, P, p0, tu = erqlp(A, k, p, q, d, seed, handle)
        return dict(Q=Q, T=T, P=P, piv0=p0, piv1=None, t_is_upper=tu)
    Q, L, P, p0, p1 = rqlp(A, k, p, q, seed, handle)
    return dict(Q=Q, T=L, P=P, piv0=p0, piv1=p1, t_is_upper=False)


def rqlp_host(A, k: int, p: int, q: int = 0, seed: int = 0):
    """North-star entry rqlp(m,n,k,p,q,A,lda,seed,Q,L,P) with HOST buffers (numpy, column-major
    float64 or pinned torch CPU tensors): host<->device copies happen inside the C call."""
    import numpy as np
    if isinstance(A, torch.Tensor):
        m, n = A.shape
        lda = _ld(A)
        Q, L, P = (torch.empty(k + p, m, dtype=torch.float64, pin_memory=A.is_pinned()).t(),
                   torch.empty(k + p, k + p, dtype=torch.float64, pin_memory=A.is_pinned()).t(),
                   torch.empty(k + p, n, dtype=torch.float64, pin_memory=A.is_pinned()).t())
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    else:
        A = np.asfortranarray(A, dtype=np.float64)
        m, n = A.shape
        lda = m
        Q = np.zeros((m, k + p), order="F")
        L = np.zeros((k + p, k + p), order="F")
        P = np.zeros((n, k + p), order="F")
        ptr = lambda t: ctypes.c_void_p(t.ctypes.data)  # noqa: E731
    _check(lib().rqlp(m, n, k, p, q, ptr(A), lda, seed, ptr(Q), ptr(L), ptr(P)), "rqlp")
    return Q, L, P


# ------------------------------------------------------------------ stage entry points
def omega(n: int, l: int, seed: int, device="cuda", handle=None) -> torch.Tensor:
    h = _handle(handle)
    Om = cm_empty(n, l, device)
    with _ordered(h):
        _check(lib().rqlp_omega(h.h, n, l, seed, _ptr(Om), _ld(Om)), "rqlp_omega")
    return Om


def gemm_nn(A, X, handle=None) -> torch.Tensor:
    A, X = _mat(A, "A"), _mat(X, "X")
    h = _handle(handle)
    h.clear_workspace()
    Y = cm_empty(A.shape[0], X.shape[1], A.device)
    with _ordered(h):
        _check(lib().rqlp_gemm_nn(h.h, A.shape[0], X.shape[1], A.shape[1], _ptr(A), _ld(A), _ptr(X), _ld(X), _ptr(Y),
                                  _ld(Y)), "rqlp_gemm_nn")
    return Y


def gemm_tn(A, V, trans_out: bool = False, handle=None) -> torch.Tensor:
    A, V = _mat(A, "A"), _mat(V, "V")
    h = _handle(handle)
    h.clear_workspace()
    m, kk = A.shape
    c = V.shape[1]
    Z = cm_empty(c, kk, A.device) if trans_out else cm_empty(kk, c, A.device)
    with _ordered(h):
        _check(lib().rqlp_gemm_tn(h.h, m, c, kk, _ptr(A), _ld(A), _ptr(V), _ld(V), _ptr(Z), _ld(Z),
                                  1 if trans_out else 0), "rqlp_gemm_tn")
    return Z


def orth(Y, return_r: bool = False, handle=None):
    Y = _mat(Y, "Y")
    h = _handle(handle)
    h.clear_workspace()
    m, c = Y.shape
    V = cm_empty(m, c, Y.device)
    R = cm_empty(c, c, Y.device) if return_r else None
    with _ordered(h):
        _check(lib().rqlp_orth(h.h, m, c, _ptr(Y), _ld(Y), _ptr(V), _ld(V), _ptr(R), _ld(R) if R is not None else 1),
               "rqlp_orth")
    return (V, R) if return_r else V


def cpqr(M, handle=None):
    M = _mat(M, "M")
    h = _handle(handle)
    h.clear_workspace()
    r, c = M.shape
    s = min(r, c)
    Q, R = cm_empty(r, s, M.device), cm_empty(s, c, M.device)
    perm = torch.empty(c, dtype=torch.int64, device=M.device)
    with _ordered(h):
        _check(lib().rqlp_cpqr(h.h, r, c, _ptr(M), _ld(M), _ptr(Q), _ld(Q), _ptr(R), _ld(R), _ptr(perm)), "rqlp_cpqr")
    return Q, R, perm


def qlp_tail(B, d: int = 0, handle=None) -> dict:
    B = _mat(B, "B")
    h = _handle(handle)
    h.clear_workspace()
    l, n = B.shape
    QB, T, PB = cm_empty(l, l, B.device), cm_empty(l, l, B.device), cm_empty(n, l, B.device)
    piv0 = torch.empty(l, dtype=torch.int64, device=B.device)
    piv1 = torch.empty(l, dtype=torch.int64, device=B.device)
    tu = ctypes.c_int(0)
    with _ordered(h):
        _check(lib().rqlp_qlp_tail(h.h, l, n, _ptr(B), _ld(B), d, _ptr(QB), _ld(QB), _ptr(T), _ld(T), _ptr(PB), _ld(PB),
                                   _ptr(piv0), _ptr(piv1), ctypes.byref(tu)), "rqlp_qlp_tail")
    return dict(QB=QB, T=T, PB=PB, piv0=piv0, piv1=piv1, t_is_upper=bool(tu.value))


def residual(A, Q, T, P, handle=None) -> float:
    """||A - Q T P^T||_F (validation kernel)."""
    A, Q, T, P = (_mat(x, nm) for x, nm in ((A, "A"), (Q, "Q"), (T, "T"), (P, "P")))
    h = _handle(handle)
    h.clear_workspace()
    out = torch.zeros(1, dtype=torch.float64, device=A.device)
    m, n = A.shape
    l = Q.shape[1]
    with _ordered(h):
        _check(lib().rqlp_residual_sq(h.h, m, n, l, _ptr(A), _ld(A), _ptr(Q), _ld(Q), _ptr(T), _ld(T), _ptr(P), _ld(P),
                                      _ptr(out)), "rqlp_residual_sq")
    return float(out.item()) ** 0.5


def truncate(out: dict, k: int, b: int | None = None) -> dict:
    """Rank-k view of a factorisation (SPEC's truncation rule; no copy): A_k = Q[:, :k] T[:k, :k]
    P[:, :k]^T with the first k pivots.  The factors are l-sized (the L-values are
    |diag T|); truncation is a caller view.  For BRQLP (`b` given) k must fall on a block boundary,
    since L = blkdiag(L_j) and P is orthonormal per block only (readings R14, R17)."""
    l = out["T"].shape[0]
    if not 1 <= k <= l:
        raise ValueError(f"k = {k} outside 1..{l}")
    if b is not None and k % b != 0 and k != l:
        raise ValueError(f"BRQLP truncation must fall on a block boundary (b = {b})")
    res = dict(out)
    res["Q"], res["T"], res["P"] = out["Q"][:, :k], out["T"][:k, :k], out["P"][:, :k]
    res["piv0"] = out["piv0"][:k]
    if out.get("piv1") is not None:
        res["piv1"] = out["piv1"][:k]
    return res


def factorize_host(A: torch.Tensor, k: int, p: int, q: int = 0, d: int = 0, b: int | None = None, seed: int = 0,
                   handle: Handle | None = None, out: tuple | None = None):
    """rqlp_factorize() with HOST operands (a column-major float64 CPU tensor A, ideally pinned):
    the C call copies A to the device, factorises, copies Q, T, P back and returns.  `out` may
    pass preallocated (pinned) column-major CPU tensors (Q, T, P)."""
    if A.is_cuda or A.dtype != torch.float64:
        raise TypeError("A must be a float64 CPU tensor")
    h = _handle(handle)
    m, n = A.shape
    l = k + p
    variant = VARIANT_BRQLP if b is not None else (VARIANT_ERQLP if d >= 1 else VARIANT_RQLP)
    if out is None:
        pin = A.is_pinned()
        out = tuple(torch.empty(c, r, dtype=torch.float64, pin_memory=pin).t() for r, c in ((m, l), (l, l), (n, l)))
    Q, T, P = out
    tu = ctypes.c_int(0)
    h.clear_workspace()
    with _ordered(h):
        _check(lib().rqlp_factorize(h.h, variant, m, n, k, p, q, d, b or 0, _ptr(A), _ld(A), seed, _ptr(Q), _ptr(T),
                                    _ptr(P), ctypes.byref(tu)), "rqlp_factorize")
    return Q, T, P, bool(tu.value)


def autorank(A: torch.Tensor, b: int, l_max: int, eps: float, q: int = 0, seed: int = 0,
             handle: Handle | None = None) -> dict:
    """Auto-rank RQLP (NEXT-1): grow blocks of b columns until the eq. (3)
    indicator sqrt(||A||^2 - sum ||B_j||^2) <= eps ||A||_F or l_max columns.  Returns the
    factorisation restricted to the l columns used, plus l and the final indicator."""
    A = _mat(A, "A")
    h = _handle(handle)
    h.clear_workspace()
    m, n = A.shape
    Q, L, P = cm_empty(m, l_max, A.device), cm_empty(l_max, l_max, A.device), cm_empty(n, l_max, A.device)
    piv0 = torch.empty(l_max, dtype=torch.int64, device=A.device)
    piv1 = torch.empty(l_max, dtype=torch.int64, device=A.device)
    lo, err = ctypes.c_int(0), ctypes.c_double(0.0)
    with _ordered(h):
        _check(lib().rqlp_autorank_ex(h.h, m, n, b, l_max, q, float(eps), _ptr(A), _ld(A), seed, _ptr(Q), _ld(Q), _ptr(L),
                                      _ld(L), _ptr(P), _ld(P), _ptr(piv0), _ptr(piv1), ctypes.byref(lo),
                                      ctypes.byref(err)), "rqlp_autorank_ex")
    l = lo.value
    return dict(Q=Q[:, :l], T=L[:l, :l], P=P[:, :l], piv0=piv0[:l], piv1=piv1[:l], l=l, err=err.value)


def tqlp(A: torch.Tensor, l: int, handle: Handle | None = None) -> dict:
    """Truncated pivoted QLP (NEXT-3): partial CPQR of A (l steps)
    then the CPQR of [R11 R12]^T.  Returns Q (m x l), T = L (l x l lower), P (n x l), piv0, piv1."""
    A = _mat(A, "A")
    h = _handle(handle)
    h.clear_workspace()
    m, n = A.shape
    Q, L, P = cm_empty(m, l, A.device), cm_empty(l, l, A.device), cm_empty(n, l, A.device)
    piv0 = torch.empty(l, dtype=torch.int64, device=A.device)
    piv1 = torch.empty(l, dtype=torch.int64, device=A.device)
    with _ordered(h):
        _check(lib().rqlp_tqlp_ex(h.h, m, n, l, _ptr(A), _ld(A), _ptr(Q), _ld(Q), _ptr(L), _ld(L), _ptr(P), _ld(P),
                                  _ptr(piv0), _ptr(piv1)), "rqlp_tqlp_ex")
    return dict(Q=Q, T=L, P=P, piv0=piv0, piv1=piv1, t_is_upper=False)
