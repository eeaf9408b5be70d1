"""Stream compaction -- drop-in for ``fgc.packer`` (pkg/src/fgc/packer.py).

``prefix_sum``, the bitmap byte conversions and ``pack`` / ``unpack`` (a
device scan, then the scatter / gather kernels fgc_compact / fgc_expand) run
as this package's CUDA kernels."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib

__all__ = ["PackedSparse", "pack", "unpack", "prefix_sum", "bitmap_to_bytes", "bitmap_from_bytes"]


@dataclass(frozen=True)
class PackedSparse:
    """packer.py:19-35."""

    bitmap: np.ndarray
    dense: np.ndarray
    original_len: int

    def __post_init__(self) -> None:
        bitmap = np.asarray(self.bitmap, dtype=bool)
        object.__setattr__(self, "bitmap", bitmap)
        object.__setattr__(self, "dense", np.asarray(self.dense))
        if bitmap.size != self.original_len:
            raise ValueError(f"bitmap covers {bitmap.size} elements, expected {self.original_len}")


def _device_scan(status01: torch.Tensor) -> torch.Tensor:
    n = status01.numel()
    out = torch.empty(n, dtype=torch.int64, device=status01.device)
    bad = torch.zeros(1, dtype=torch.int32, device=status01.device)
    tiles = (n + 4095) // 4096
    scratch = torch.empty(tiles + 1, dtype=torch.int64, device=status01.device)
    _lib.check(_lib.lib.fgc_prefix_sum(status01.data_ptr(), n, out.data_ptr(), bad.data_ptr(),
                                       scratch.data_ptr(), D.stream()))
    if int(bad.item()):
        raise ValueError("status entries must be 0 or 1")
    return out


def prefix_sum(status) -> np.ndarray:
    """packer.py:41-46: inclusive scan of a 0/1 vector (GPU)."""
    s = np.asarray(status)
    if s.size == 0:
        return np.zeros(0, dtype=np.int64)
    if s.dtype != bool and bool(((s != 0) & (s != 1)).any()):
        raise ValueError("status entries must be 0 or 1")
    dev = D.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(s.reshape(-1) != 0).astype(np.uint8)).to(dev)
    return _device_scan(t).cpu().numpy()


def _elem(values: np.ndarray) -> tuple:
    """(contiguous array, element bytes) for the device copy."""
    v = np.ascontiguousarray(values)
    if v.dtype.itemsize not in (1, 2, 4, 8):
        raise ValueError(f"unsupported element size {v.dtype.itemsize}")
    return v, v.dtype.itemsize


def pack(sparse) -> PackedSparse:
    """packer.py:49-58: status -> scan -> scatter to dense[loc-1]."""
    values = np.asarray(sparse)
    if values.size == 0:
        return PackedSparse(np.zeros(0, dtype=bool), np.empty(0, dtype=values.dtype), 0)
    dev = D.require_cuda()
    flat, eb = _elem(values.reshape(-1))
    status = torch.from_numpy((flat != 0).astype(np.uint8)).to(dev)
    loc = _device_scan(status)
    kept = int(loc[-1].item())
    src = torch.from_numpy(flat.view(np.uint8)).to(dev)
    dense = torch.empty(max(1, kept * eb), dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.fgc_compact(src.data_ptr(), status.data_ptr(), loc.data_ptr(), flat.size, eb,
                                    dense.data_ptr(), D.stream()))
    d = dense[:kept * eb].cpu().numpy().view(flat.dtype)
    return PackedSparse(bitmap=status.cpu().numpy().astype(bool), dense=d, original_len=values.size)


def unpack(packed: PackedSparse) -> np.ndarray:
    """packer.py:61-70."""
    kept = int(np.count_nonzero(packed.bitmap))
    if kept != packed.dense.size:
        raise ValueError(f"bitmap marks {kept} elements but dense payload has {packed.dense.size}")
    out = np.zeros(packed.original_len, dtype=packed.dense.dtype)
    if kept:
        dev = D.require_cuda()
        dense, eb = _elem(packed.dense)
        status = torch.from_numpy(np.ascontiguousarray(packed.bitmap).astype(np.uint8)).to(dev)
        loc = _device_scan(status)
        src = torch.from_numpy(dense.view(np.uint8)).to(dev)
        full = torch.empty(packed.original_len * eb, dtype=torch.uint8, device=dev)
        _lib.check(_lib.lib.fgc_expand(src.data_ptr(), status.data_ptr(), loc.data_ptr(), packed.original_len, eb,
                                       full.data_ptr(), D.stream()))
        out = full.cpu().numpy().view(dense.dtype).copy()
    return out


def bitmap_to_bytes(bitmap: np.ndarray) -> bytes:
    """packer.py:73-75: MSB-first, zero padded (GPU)."""
    b = np.asarray(bitmap, dtype=np.uint8).reshape(-1)
    if b.size == 0:
        return b""
    dev = D.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(b != 0).astype(np.uint8)).to(dev)
    out = torch.empty((b.size + 7) // 8, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.fgc_flags_to_bitmap(t.data_ptr(), b.size, out.data_ptr(), D.stream()))
    return out.cpu().numpy().tobytes()


def bitmap_from_bytes(data: bytes, length: int) -> np.ndarray:
    """packer.py:78-84 (GPU)."""
    need = (length + 7) // 8
    if len(data) < need:
        raise ValueError(f"bitmap buffer too short: {len(data)} < {need} bytes")
    if length == 0:
        return np.zeros(0, dtype=bool)
    dev = D.require_cuda()
    src = torch.frombuffer(bytearray(data[:need]), dtype=torch.uint8).to(dev)
    out = torch.empty(length, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.fgc_bitmap_to_flags(src.data_ptr(), length, out.data_ptr(), D.stream()))
    return out.cpu().numpy().astype(bool)
