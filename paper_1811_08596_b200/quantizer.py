"""Range-based N-bit float quantizer -- drop-in for the reference module
``fgc.quantizer`` (pkg/src/fgc/quantizer.py).

Configuration logic (``QuantizerConfig``, ``tune_eps``) runs in the host C
library; the element-wise codec (``encode_array`` ...) runs as CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib

__all__ = ["QuantizerConfig", "tune_eps", "encode", "decode", "encode_array", "decode_array",
           "encode_block", "decode_block", "pack_codes", "unpack_codes"]

MIN_EPS = 2.0 ** -126
MAX_F32_PATTERN = 0x7F7FFFFF
TUNE_MAX_ITERS = 64


def _f32(x) -> float:
    return float(np.float32(x))


@dataclass(frozen=True)
class QuantizerConfig:
    """One range-float lattice (quantizer.py:71-151).  Same fields, same
    validation; ``pbase`` / ``pos_count`` are derived by ``from_params``."""

    min: float
    max: float
    n_bits: int
    mantissa_bits: int
    eps: float
    pbase: int
    pos_count: int

    def __post_init__(self) -> None:
        n, m = self.n_bits, self.mantissa_bits
        # the float checks of quantizer.py:95-100 in float64, as the reference
        if 2 <= n <= 16 and 1 <= m < n:
            if not (np.isfinite(self.min) and np.isfinite(self.max)):
                raise ValueError("min/max must be finite")
            if not (self.min < 0.0 < self.max):
                raise ValueError(f"range must straddle zero, got [{self.min}, {self.max}]")
            if not (0.0 < self.eps < self.max):
                raise ValueError(f"eps must be in (0, max), got {self.eps}")
        if not (0 <= int(self.pbase) < 2 ** 32 and 0 <= int(self.pos_count) < 2 ** 32):
            raise ValueError("config leaves no room for positive or negative codes")
        s = _lib.Quantizer()
        s.min, s.max, s.eps = self.min, self.max, self.eps
        s.n_bits, s.mantissa_bits = int(n), int(m)
        s.pbase, s.pos_count = int(self.pbase), int(self.pos_count)
        _lib.check(_lib.lib.fgc_quantizer_validate(C.byref(s)))   # integer checks, derived fields
        object.__setattr__(self, "_c", s)

    @property
    def c_struct(self) -> _lib.Quantizer:
        return self._c

    @classmethod
    def from_params(cls, min: float, max: float, n_bits: int, mantissa_bits: int,
                    eps: float) -> "QuantizerConfig":
        """quantizer.py:108-135."""
        s = _lib.Quantizer()
        _lib.check(_lib.lib.fgc_quantizer_from_params(float(min), float(max), int(n_bits),
                                                      int(mantissa_bits), float(eps), C.byref(s)))
        return cls(float(s.min), float(s.max), int(n_bits), int(mantissa_bits), float(s.eps),
                   int(s.pbase), int(s.pos_count))

    @property
    def neg_count(self) -> int:
        return 2 ** self.n_bits - 1 - self.pos_count

    @property
    def actual_min(self) -> float:
        return float(self._c.actual_min)

    @property
    def actual_max(self) -> float:
        return float(self._c.actual_max)


def tune_eps(min: float, max: float, n_bits: int, mantissa_bits: int,
             eps_init: float = 0.002) -> QuantizerConfig:
    """quantizer.py:154-214 (host C)."""
    s = _lib.Quantizer()
    st = _lib.lib.fgc_tune_eps(float(min), float(max), int(n_bits), int(mantissa_bits),
                               float(eps_init), C.byref(s))
    _lib.check(st)
    return QuantizerConfig(float(s.min), float(s.max), int(n_bits), int(mantissa_bits), float(s.eps),
                           int(s.pbase), int(s.pos_count))


def _codes_to_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def encode_array(config: QuantizerConfig, values) -> np.ndarray:
    """quantizer.py:217-236 on the GPU; returns uint32 codes."""
    arr = np.asarray(values)
    if arr.size == 0:
        return np.zeros(arr.shape, dtype=np.uint32)
    t, code = D.as_signal(arr.reshape(-1), "values")
    out = torch.empty(t.numel(), dtype=torch.int32, device=t.device)
    first_nan = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=t.device)
    _lib.check(_lib.lib.fgc_quantize(C.byref(config.c_struct), t.data_ptr(), code, t.numel(),
                                     out.data_ptr(), first_nan.data_ptr(), D.stream()))
    if int(first_nan.item()) != np.iinfo(np.int64).max:
        raise ValueError("cannot encode NaN")
    return _codes_to_host(out).reshape(arr.shape)


def decode_array(config: QuantizerConfig, codes) -> np.ndarray:
    """quantizer.py:239-253 on the GPU; returns float32 values."""
    c = np.asarray(codes)
    if c.size == 0:
        return np.zeros(c.shape, dtype=np.float32)
    dev = D.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(c.astype(np.int64).reshape(-1))).to(dev)
    out = torch.empty(t.numel(), dtype=torch.float32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib.fgc_dequantize(C.byref(config.c_struct), t.data_ptr(), t.numel(),
                                       out.data_ptr(), bad.data_ptr(), D.stream()))
    if int(bad.item()):
        raise ValueError(f"code out of range for N={config.n_bits}")
    return out.cpu().numpy().reshape(c.shape)


def encode(config: QuantizerConfig, x: float) -> int:
    return int(encode_array(config, np.array([x]))[0])


def decode(config: QuantizerConfig, code: int) -> float:
    return float(decode_array(config, np.array([code]))[0])


def pack_codes(codes, n_bits: int) -> bytes:
    """quantizer.py:266-273: LSB-first ``n_bits`` fields (GPU)."""
    c = np.asarray(codes, dtype=np.uint32).reshape(-1)
    if c.size == 0:
        return b""
    dev = D.require_cuda()
    t = torch.from_numpy(c.view(np.int32).copy()).to(dev)
    nbytes = (c.size * n_bits + 7) // 8
    out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib.fgc_pack_bits(t.data_ptr(), c.size, int(n_bits), out.data_ptr(), D.stream()))
    return out.cpu().numpy().tobytes()


def unpack_codes(data: bytes, n_bits: int, count: int) -> np.ndarray:
    """quantizer.py:276-285 (GPU)."""
    if count == 0:
        return np.zeros(0, dtype=np.uint32)
    need = (count * n_bits + 7) // 8
    if len(data) < need:
        raise ValueError(f"packed code buffer too short: {len(data)} < {need} bytes")
    dev = D.require_cuda()
    src = torch.frombuffer(bytearray(data[:need]), dtype=torch.uint8).to(dev)
    out = torch.empty(count, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib.fgc_unpack_bits(src.data_ptr(), count, int(n_bits), out.data_ptr(), D.stream()))
    return _codes_to_host(out)


def encode_block(config: QuantizerConfig, values) -> bytes:
    """quantizer.py:288-294."""
    arr = np.asarray(values, dtype=np.float64)
    if arr.size:
        t, code = D.as_signal(arr.reshape(-1))
        out = torch.empty(t.numel(), dtype=torch.int32, device=t.device)
        first_nan = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=t.device)
        _lib.check(_lib.lib.fgc_quantize(C.byref(config.c_struct), t.data_ptr(), code, t.numel(),
                                         out.data_ptr(), first_nan.data_ptr(), D.stream()))
        bad = int(first_nan.item())
        if bad != np.iinfo(np.int64).max:
            raise ValueError(f"cannot encode NaN at index {bad}")
        nbytes = (t.numel() * config.n_bits + 7) // 8
        packed = torch.empty(nbytes, dtype=torch.uint8, device=t.device)
        _lib.check(_lib.lib.fgc_pack_bits(out.data_ptr(), t.numel(), config.n_bits, packed.data_ptr(),
                                          D.stream()))
        return packed.cpu().numpy().tobytes()
    return b""


def decode_block(config: QuantizerConfig, data: bytes, count: int) -> np.ndarray:
    """quantizer.py:297-299."""
    return decode_array(config, unpack_codes(data, config.n_bits, count))
