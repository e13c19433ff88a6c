"""POD by the method of snapshots (SPEC mor.pod; arXiv 1704.04139 section 2.5).

The snapshot Gram matrix ``G = S^T W S`` and the other dense contractions of the
reduced-basis stage (basis projection, re-orthonormalisation, EI updates, ``B^T W``)
run on the FP64 tensor cores (``csrc/hc_pod.cu``, :func:`tc_matmul`); the small
eigenproblem of G and the small triangular / dense solves stay on the device.
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from .errors import ReductionError


def pod_gram(S, w=None):
    """``S^T diag(w) S`` for an (n_dof, n_snap) fp64 snapshot matrix (row- or column-major
    CUDA tensors are used in place; anything else is copied to the device)."""
    t = _dev.torch()
    rows = False
    if _dev.is_tensor(S) and S.is_cuda and S.dtype == t.float64 and S.dim() == 2 \
            and S.t().is_contiguous():
        Sc = S.t()                      # column-major storage of S: no copy
    else:
        Sc = _dev.to_dev(S)             # row-major storage (snapshots contiguous per DOF)
        if Sc.dim() != 2:
            raise ValueError("snapshot matrix must be 2-D (n_dof, n_snap)")
        rows = True
    n_dof, n_snap = (Sc.shape[1], Sc.shape[0]) if not rows else (Sc.shape[0], Sc.shape[1])
    wd = _dev.to_dev(w) if w is not None else None
    G = t.empty((n_snap, n_snap), dtype=t.float64, device="cuda")
    fn = _native.lib().hc_pod_gram_rows if rows else _native.lib().hc_pod_gram
    _native.check(fn(_dev.ptr(Sc), _dev.ptr(wd) if wd is not None else None, int(n_dof), int(n_snap),
                     _dev.ptr(G), _dev.stream()))
    G = G.t()  # column-major result -> row-major view
    return _dev.like_input(G.contiguous(), S)


def tc_matmul(X, Y, w=None):
    """``X @ diag(w) @ Y`` (fp64) on the FP64 tensor cores (``hc_dgemm``, csrc/hc_pod.cu).

    X (M, K) and Y (K, N) are CUDA fp64 tensors of any strides (transposed views and row
    slices are used in place); the result is a new contiguous (M, N) tensor."""
    t = _dev.torch()
    X, Y = _dev.to_dev_strided(X), _dev.to_dev_strided(Y)
    if X.dim() != 2 or Y.dim() != 2 or X.shape[1] != Y.shape[0]:
        raise ValueError(f"tc_matmul: incompatible shapes {tuple(X.shape)} @ {tuple(Y.shape)}")
    M, K = X.shape
    N = Y.shape[1]
    C = t.empty((M, N), dtype=t.float64, device="cuda")
    wd = _dev.to_dev(w) if w is not None else None
    _native.check(_native.lib().hc_dgemm(
        _dev.ptr(X) if X.numel() else None, X.stride(1), X.stride(0),
        _dev.ptr(Y) if Y.numel() else None, Y.stride(0), Y.stride(1),
        _dev.ptr(wd) if wd is not None else None, int(K), int(M), int(N), _dev.ptr(C), int(N),
        _dev.stream()))
    return C


def pod_basis(S, rel_tol: float, w=None):
    """Orthonormal POD basis keeping the smallest k with tail energy <= rel_tol^2.

    Returns (basis (n_dof, k), singular values (n_snap,)).
    """
    t = _dev.torch()
    Sd = _dev.to_dev(S)
    if not float(t.linalg.vector_norm(Sd)) > 0.0:
        raise ReductionError("all-zero snapshot set")
    G = _dev.to_dev(pod_gram(Sd, w))
    G = 0.5 * (G + G.t())
    lam, V = t.linalg.eigh(G)
    lam, V = lam.flip(0), V.flip(1)
    lam = t.clamp(lam, min=0.0)
    sig = t.sqrt(lam)
    tot = float(lam.sum())
    tail = t.flip(t.cumsum(t.flip(lam, [0]), 0), [0])  # tail[k] = sum_{i>=k} lam_i
    k = int(lam.numel())
    for kk in range(1, lam.numel() + 1):
        rest = float(tail[kk]) if kk < lam.numel() else 0.0
        if rest <= rel_tol ** 2 * tot:
            k = kk
            break
    B = tc_matmul(Sd, V[:, :k] / sig[:k])
    # one modified Gram-Schmidt pass (SPEC: re-orthonormalize output)
    for j in range(k):
        for i in range(j):
            B[:, j] -= (B[:, i] @ B[:, j]) * B[:, i]
        B[:, j] /= t.linalg.vector_norm(B[:, j])
    return _dev.like_input(B, S), (sig.cpu().numpy() if not _dev.is_tensor(S) else sig)
