"""Device-memory plumbing: PyTorch allocates, the C ABI computes."""

from __future__ import annotations

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def is_tensor(a) -> bool:
    t = torch()
    return isinstance(a, t.Tensor)


def to_dev(a, dtype=None):
    """fp64 (or ``dtype``) contiguous CUDA tensor view/copy of ``a``."""
    t = torch()
    dtype = dtype or t.float64
    if isinstance(a, t.Tensor):
        if a.device.type == "cuda" and a.dtype == dtype and a.is_contiguous():
            return a
        return a.to(device="cuda", dtype=dtype).contiguous()
    return t.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def to_dev_strided(a):
    """CUDA fp64 tensor of ``a`` keeping a strided CUDA fp64 view as it is (no copy)."""
    t = torch()
    if isinstance(a, t.Tensor) and a.device.type == "cuda" and a.dtype == t.float64:
        return a
    return to_dev(a)


def numel(a) -> int:
    """Element count of a numpy array or tensor."""
    return int(a.numel()) if is_tensor(a) else int(np.size(a))


def empty(n: int, dtype=None):
    t = torch()
    return t.empty(max(int(n), 0), dtype=dtype or t.float64, device="cuda")


def ptr(a) -> int | None:
    return a.data_ptr() if a is not None and a.numel() else None


def stream() -> int | None:
    t = torch()
    return t.cuda.current_stream().cuda_stream or None


def like_input(result, template):
    """Return ``result`` (CUDA tensor) as numpy when ``template`` was not a tensor."""
    if is_tensor(template):
        return result
    return result.cpu().numpy()
