"""GPU-test plumbing: a shared ctx, operand upload with controlled alignment."""
from __future__ import annotations

import numpy as np
import pytest
import torch

TORCH = {"f32": torch.float32, "f64": torch.float64, "u32": torch.uint32, "s64": torch.int64,
         "bf16": torch.bfloat16, "f16": torch.float16,
         "e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}
RTORCH = dict(TORCH, e4m3=torch.float32, e5m2=torch.float32)  # reduction result dtypes


def have_gpu() -> bool:
    return torch.cuda.is_available()


requires_gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")


def to_dev(a: np.ndarray, etype: str, offset: int = 0) -> torch.Tensor:
    """Upload to cuda:0 starting `offset` elements into a fresh allocation
    (offset controls the 16-byte misalignment of the data pointer)."""
    a = np.ascontiguousarray(a, dtype=_np_view(etype))
    if etype == "u32":
        t = torch.from_numpy(a.view(np.int32).copy()).view(torch.uint32)
    elif etype == "bf16":  # host arrays hold bf16 bit patterns (uint16)
        t = torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16)
    elif etype in ("e4m3", "e5m2"):  # host arrays hold 8-bit patterns (uint8)
        t = torch.from_numpy(a.copy()).view(TORCH[etype])
    else:
        t = torch.from_numpy(a.copy())
    base = torch.empty(a.size + offset + 8, dtype=TORCH[etype], device="cuda")
    dst = base[offset:offset + a.size]
    dst.copy_(t.to("cuda"))
    return dst


def _np_view(etype):
    return {"f32": np.float32, "f64": np.float64, "u32": np.uint32, "s64": np.int64,
            "bf16": np.uint16, "f16": np.float16, "e4m3": np.uint8, "e5m2": np.uint8}[etype]


def empty_dev(n: int, etype: str, offset: int = 0) -> torch.Tensor:
    base = torch.empty(n + offset + 8, dtype=TORCH[etype], device="cuda")
    return base[offset:offset + n]


def to_host(t: torch.Tensor, etype: str) -> np.ndarray:
    if etype == "u32":
        return t.cpu().view(torch.int32).numpy().view(np.uint32)
    if etype == "bf16":
        return t.cpu().view(torch.int16).numpy().view(np.uint16)
    if etype in ("e4m3", "e5m2") and t.dtype == TORCH[etype]:
        return t.cpu().view(torch.uint8).numpy()
    return t.cpu().numpy()


def half_ordinal(bits: np.ndarray) -> np.ndarray:
    b = np.asarray(bits).view(np.uint16).astype(np.int64)
    return np.where(b & 0x8000, -(b & 0x7FFF), b)


def half_ulp(a, b) -> np.ndarray:
    """Ordinal distance of 16-bit float bit patterns (NaN vs NaN -> 0)."""
    a = np.atleast_1d(np.asarray(a)).view(np.uint16)
    b = np.atleast_1d(np.asarray(b)).view(np.uint16)
    d = np.abs(half_ordinal(a) - half_ordinal(b))
    return d
