"""Device plumbing: CUDA availability, the current stream, host<->device
staging.  torch is used only for device memory and streams."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1811_08596_b200 runs its data path on a CUDA device (sm_100a); "
                           "no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def as_signal(values, name: str = "gradient"):
    """1-D float32/float64 device tensor + dtype code; the reference converts
    with ``np.asarray(values, dtype=float64)`` -- float32 input is kept as
    float32 (exactly representable, so results are identical)."""
    dev = require_cuda()
    if isinstance(values, torch.Tensor):
        t = values.detach()
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        t = t.to(dev).contiguous()
    else:
        a = np.asarray(values)
        if a.dtype != np.float32:
            a = np.asarray(values, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    code = _lib.DTYPE_F32 if t.dtype == torch.float32 else _lib.DTYPE_F64
    return aligned(t), code


def aligned(t: torch.Tensor) -> torch.Tensor:
    """The kernels load two samples at a time: a view starting off an 8-byte
    (f32) / 16-byte (f64) boundary is copied to a fresh allocation."""
    return t.clone() if t.data_ptr() % (2 * t.element_size()) else t


def flags_tensor() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=require_cuda())


def read_flags(flags: torch.Tensor) -> int:
    return int(flags.item()) & 0xFFFFFFFF


def raise_on_flags(f: int) -> None:
    if f & _lib.FLAG_NONFINITE:
        raise ValueError("gradient must be finite")
    if f & _lib.FLAG_HALF_OVERFLOW:
        raise ValueError("gradient overflowed binary16 during the half-precision pass")
    if f & _lib.FLAG_F32_RANGE:
        raise ValueError("gradient exceeds the float32 range the GPU codec computes in")
    if f & _lib.FLAG_CAPACITY:
        raise _lib.NativeError("message exceeded its fixed device capacity")
