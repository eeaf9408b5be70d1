"""Stream compaction -- drop-in for ``fgc.packer`` (pkg/src/fgc/packer.py).

``prefix_sum`` and the bitmap byte conversions run as CUDA kernels; ``pack``
/ ``unpack`` compact with a device scan + scatter (torch index ops on the
device for the value gather, the scan itself is ours)."""

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


def pack(sparse) -> PackedSparse:
    """packer.py:49-58: status -> scan -> scatter to dense[loc-1]."""
    values = np.asarray(sparse)
    if values.size == 0:
        return PackedSparse(np.zeros(0, dtype=bool), np.empty(0, dtype=values.dtype), 0)
    dev = D.require_cuda()
    flat = values.reshape(-1)
    status = torch.from_numpy(np.ascontiguousarray(flat != 0).astype(np.uint8)).to(dev)
    loc = _device_scan(status)
    kept = int(loc[-1].item())
    marked = status.bool()
    vals = torch.from_numpy(np.ascontiguousarray(flat)).to(dev) if flat.dtype != np.uint32 else \
        torch.from_numpy(flat.view(np.int32).copy()).to(dev)
    dense = torch.empty(kept, dtype=vals.dtype, device=dev)
    dense[loc[marked] - 1] = vals[marked]
    d = dense.cpu().numpy()
    if flat.dtype == np.uint32:
        d = d.view(np.uint32)
    return PackedSparse(bitmap=marked.cpu().numpy(), dense=d.astype(values.dtype, copy=False),
                        original_len=values.size)


def unpack(packed: PackedSparse) -> np.ndarray:
    """packer.py:61-70."""
    kept = int(np.count_nonzero(packed.bitmap))
    if kept != packed.dense.size:
        raise ValueError(f"bitmap marks {kept} elements but dense payload has {packed.dense.size}")
    out = np.zeros(packed.original_len, dtype=packed.dense.dtype)
    if kept:
        dev = D.require_cuda()
        mask = torch.from_numpy(np.ascontiguousarray(packed.bitmap)).to(dev)
        dense = packed.dense
        is_u32 = dense.dtype == np.uint32
        src = torch.from_numpy(dense.view(np.int32).copy() if is_u32 else np.ascontiguousarray(dense)).to(dev)
        full = torch.zeros(packed.original_len, dtype=src.dtype, device=dev)
        full[mask] = src
        r = full.cpu().numpy()
        out = r.view(np.uint32) if is_u32 else r
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
