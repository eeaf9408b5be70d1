"""Gradient codec pipeline and FGC1 wire format -- drop-in for ``fgc.codec``
(pkg/src/fgc/codec.py), executed by the sm_100a kernels of libfgc_b200.

A ``CompressedMessage`` returned by ``compress`` / ``deserialize`` is backed
by a fixed-capacity device message; its
``chunks`` (``ChunkPayload`` bitmap/codes arrays, codec.py:112-125) are
materialized lazily by a device unpack kernel.  Messages built by hand from
``ChunkPayload`` objects are packed onto the device when first decoded.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from ._lib import (BitmapMismatchError, CodecFormatError, CorruptHeaderError,
                   TruncatedPayloadError)
from .quantizer import QuantizerConfig, tune_eps
from .spectral import SparsificationSpec

__all__ = ["CodecConfig", "ChunkPayload", "CompressedMessage", "CodecFormatError",
           "CorruptHeaderError", "TruncatedPayloadError", "BitmapMismatchError", "compress",
           "decompress", "reconstruct", "reconstruct_rows", "serialize", "deserialize",
           "calibrate", "compression_ratio", "Plan", "get_plan"]

MAGIC = b"FGC1"
VERSION = 1
FLAG_HALF_PASS, FLAG_ENERGY, FLAG_PASSTHROUGH = 0x01, 0x02, 0x04
HEADER_BYTES = 36
MIN_CHUNK_SIZE = 16
DEFAULT_CHUNK_SIZE = 1 << 16
_KEPT = struct.Struct("<I")


@dataclass(frozen=True)
class CodecConfig:
    """codec.py:92-109."""

    sparsification: SparsificationSpec
    quantizer: QuantizerConfig | None = None
    half_precision_pass: bool = False
    chunk_size: int = DEFAULT_CHUNK_SIZE

    def __post_init__(self) -> None:
        if self.chunk_size < MIN_CHUNK_SIZE:
            raise ValueError(f"chunk_size must be >= {MIN_CHUNK_SIZE}, got {self.chunk_size}")
        if self.sparsification.domain != "frequency":
            raise ValueError("codec sparsification must operate in the frequency domain")

    @property
    def n_bits(self) -> int:
        return 32 if self.quantizer is None else self.quantizer.n_bits


@dataclass(eq=False)
class ChunkPayload:
    """codec.py:112-125."""

    bitmap: np.ndarray
    codes: np.ndarray

    def __eq__(self, other) -> bool:
        if not isinstance(other, ChunkPayload):
            return NotImplemented
        return np.array_equal(self.bitmap, other.bitmap) and np.array_equal(self.codes, other.codes)


# ------------------------------------------------------------------ plans

def _desc(n: int, chunk: int, theta: float, mode: str, half: bool, quant: QuantizerConfig | None,
          full_capacity: bool) -> _lib.CodecDesc:
    d = _lib.CodecDesc()
    d.n = int(n)
    d.chunk_size = int(chunk)
    d.mode = _lib.MODE_ENERGY if mode == "energy" else _lib.MODE_COUNT
    d.theta = float(theta)
    d.half_pass = int(bool(half))
    d.passthrough = int(quant is None)
    d.full_capacity = int(bool(full_capacity))
    if quant is not None:
        d.quant = quant.c_struct
    return d


class Plan:
    """Owns one native plan (device tables + scratch) for a config/length."""

    def __init__(self, desc: _lib.CodecDesc):
        D.require_cuda()
        self.desc = desc
        h = C.c_void_p()
        _lib.check(_lib.lib.fgc_plan_create(C.byref(desc), C.byref(h)))
        self.handle = h
        info = _lib.PlanInfo()
        _lib.check(_lib.lib.fgc_plan_get_info(h, C.byref(info)))
        self.info = info
        self.n_chunks = int(info.n_chunks)
        self.message_bytes = int(info.message_bytes)
        self.n_bits = int(info.n_bits)
        offs = np.zeros(self.n_chunks + 1, dtype=np.uint64)
        _lib.check(_lib.lib.fgc_plan_segment_offsets(h, offs.ctypes.data))
        self.segment_offsets = offs
        bins = np.zeros(self.n_chunks + 1, dtype=np.uint64)
        _lib.check(_lib.lib.fgc_plan_bin_offsets(h, bins.ctypes.data))
        self.bin_offsets = bins

    def new_message(self) -> torch.Tensor:
        return torch.empty(self.message_bytes, dtype=torch.uint8, device=D.require_cuda())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.lib.fgc_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


_PLANS: "OrderedDict[tuple, Plan]" = OrderedDict()
_PLAN_CACHE = int(__import__("os").environ.get("FGC_PLAN_CACHE", "16"))


def get_plan(n: int, chunk: int, theta: float, mode: str, half: bool, quant: QuantizerConfig | None,
             full_capacity: bool = False) -> Plan:
    key = (int(n), int(chunk), float(theta), mode, bool(half), quant, bool(full_capacity),
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    p = _PLANS.get(key)
    if p is None:
        p = Plan(_desc(n, chunk, theta, mode, half, quant, full_capacity))
        _PLANS[key] = p
        while len(_PLANS) > _PLAN_CACHE:
            _PLANS.popitem(last=False)
    else:
        _PLANS.move_to_end(key)
    return p


def _chunk_lengths(n: int, chunk_size: int) -> list:
    """codec.py:163-167."""
    lengths = [chunk_size] * (n // chunk_size)
    if n % chunk_size:
        lengths.append(n % chunk_size)
    return lengths


def _slot_count(chunk_len: int) -> int:
    """codec.py:170-171."""
    return 2 * (chunk_len // 2 + 1)


# ------------------------------------------------------------------ message

class CompressedMessage:
    """codec.py:128-160; device-backed when produced by this package."""

    def __init__(self, original_len: int, chunk_size: int, theta: float, mode: str, half_pass: bool,
                 quantizer: QuantizerConfig | None, chunks: list | None = None, *,
                 _device: tuple | None = None):
        self.original_len = int(original_len)
        self.chunk_size = int(chunk_size)
        self.theta = float(theta)
        self.mode = mode
        self.half_pass = bool(half_pass)
        self.quantizer = quantizer
        self._chunks = chunks
        self._device = _device          # (Plan, uint8 device tensor)
        if chunks is None and _device is None:
            self._chunks = []

    # the reference exposes `chunks` as a plain list attribute
    @property
    def chunks(self) -> list:
        if self._chunks is None:
            self._chunks = _materialize(*self._device)
        return self._chunks

    @chunks.setter
    def chunks(self, value: list) -> None:
        self._chunks = value
        self._device = None

    @property
    def passthrough(self) -> bool:
        return self.quantizer is None

    @property
    def n_bits(self) -> int:
        return 32 if self.quantizer is None else self.quantizer.n_bits

    def __eq__(self, other) -> bool:
        if not isinstance(other, CompressedMessage):
            return NotImplemented
        return (self.original_len == other.original_len and self.chunk_size == other.chunk_size
                and self.theta == other.theta and self.mode == other.mode
                and self.half_pass == other.half_pass and self.quantizer == other.quantizer
                and self.chunks == other.chunks)

    __hash__ = None

    def __repr__(self) -> str:
        where = "device" if self._device is not None else "host"
        return (f"CompressedMessage(original_len={self.original_len}, chunk_size={self.chunk_size}, "
                f"theta={self.theta}, mode={self.mode!r}, half_pass={self.half_pass}, "
                f"quantizer={self.quantizer!r}, [{where}])")

    # -------- device view
    def device_message(self) -> tuple:
        """(Plan, device uint8 message) -- packing host chunks if needed."""
        if self._device is None:
            self._device = _pack_host(self)
        return self._device


def _materialize(plan: Plan, msg: torch.Tensor) -> list:
    dev = msg.device
    n = plan.n_chunks
    nnz = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib.fgc_message_counts(plan.handle, msg.data_ptr(), nnz.data_ptr(), D.stream()))
    counts = nnz.cpu().numpy().astype(np.int64)
    code_off = np.zeros(n + 1, dtype=np.uint64)
    code_off[1:] = np.cumsum(counts)
    total_slots = int(plan.info.total_slots)
    flags = torch.empty(total_slots, dtype=torch.uint8, device=dev)
    codes = torch.empty(max(1, int(code_off[-1])), dtype=torch.int32, device=dev)
    d_off = torch.from_numpy(code_off.view(np.int64)).to(dev)
    _lib.check(_lib.lib.fgc_message_unpack(plan.handle, msg.data_ptr(), d_off.data_ptr(), flags.data_ptr(),
                                           codes.data_ptr(), D.stream()))
    fl = flags.cpu().numpy().astype(bool)
    cd = codes.cpu().numpy().view(np.uint32)
    out, s0 = [], 0
    lengths = _chunk_lengths(int(plan.desc.n), int(plan.desc.chunk_size))
    for c, L in enumerate(lengths):
        slots = _slot_count(L)
        out.append(ChunkPayload(bitmap=fl[s0:s0 + slots].copy(),
                                codes=cd[int(code_off[c]):int(code_off[c + 1])].copy()))
        s0 += slots
    return out


def _pack_host(m: CompressedMessage) -> tuple:
    lengths = _chunk_lengths(m.original_len, m.chunk_size)
    chunks = m.chunks
    if len(lengths) != len(chunks):
        raise TruncatedPayloadError(f"message has {len(chunks)} chunks, expected {len(lengths)}")
    for L, ch in zip(lengths, chunks):
        bm = np.asarray(ch.bitmap)
        if bm.size != _slot_count(L):
            raise BitmapMismatchError(f"bitmap covers {bm.size} slots, expected {_slot_count(L)}")
    plan = get_plan(m.original_len, m.chunk_size, m.theta, m.mode, m.half_pass, m.quantizer,
                    full_capacity=True)
    dev = D.require_cuda()
    flags01 = np.concatenate([np.asarray(ch.bitmap, dtype=bool) for ch in chunks]).astype(np.uint8)
    counts = np.array([np.asarray(ch.codes).size for ch in chunks], dtype=np.int64)
    code_off = np.zeros(len(chunks) + 1, dtype=np.int64)
    code_off[1:] = np.cumsum(counts)
    allcodes = np.concatenate([np.asarray(ch.codes, dtype=np.uint32).reshape(-1) for ch in chunks]
                              + [np.zeros(1, dtype=np.uint32)])
    msg = plan.new_message()
    pops = torch.empty(plan.n_chunks, dtype=torch.int32, device=dev)
    fl = D.flags_tensor()
    t_flags = torch.from_numpy(flags01).to(dev)
    t_codes = torch.from_numpy(allcodes.view(np.int32)).to(dev)
    t_off = torch.from_numpy(code_off).to(dev)
    _lib.check(_lib.lib.fgc_message_pack(plan.handle, t_flags.data_ptr(), t_codes.data_ptr(), t_off.data_ptr(),
                                         msg.data_ptr(), pops.data_ptr(), fl.data_ptr(), D.stream()))
    p = pops.cpu().numpy().astype(np.int64)
    bad = np.nonzero(p != counts)[0]
    if bad.size:
        c = int(bad[0])
        raise BitmapMismatchError(f"bitmap marks {int(p[c])} slots but payload has {int(counts[c])} codes")
    D.raise_on_flags(D.read_flags(fl))
    return plan, msg


# ------------------------------------------------------------------ pipeline

def _compress_device(t: torch.Tensor, code: int, config: CodecConfig) -> tuple:
    spec = config.sparsification
    plan = get_plan(t.numel(), config.chunk_size, spec.theta, spec.mode, config.half_precision_pass,
                    config.quantizer)
    msg = plan.new_message()
    flags = D.flags_tensor()
    _lib.check(_lib.lib.fgc_compress(plan.handle, t.data_ptr(), code, msg.data_ptr(), flags.data_ptr(),
                                     D.stream()))
    return plan, msg, flags


def _validated_signal(gradient):
    if isinstance(gradient, torch.Tensor):
        if gradient.dim() != 1 or gradient.numel() == 0:
            raise ValueError("gradient must be a non-empty 1D sequence")
    else:
        a = np.asarray(gradient)
        if a.ndim != 1 or a.size == 0:
            raise ValueError("gradient must be a non-empty 1D sequence")
        if a.dtype.kind not in "fiub":
            a = np.asarray(gradient, dtype=np.float64)
        gradient = a
    return D.as_signal(gradient)


def compress(gradient, config: CodecConfig) -> CompressedMessage:
    """codec.py:220-243 on the GPU.  Accepts array-likes or torch tensors."""
    t, code = _validated_signal(gradient)
    plan, msg, flags = _compress_device(t, code, config)
    D.raise_on_flags(D.read_flags(flags))
    return CompressedMessage(t.numel(), config.chunk_size, float(np.float32(config.sparsification.theta)),
                             config.sparsification.mode, config.half_precision_pass, config.quantizer,
                             _device=(plan, msg))


def _decode(plan: Plan, messages: torch.Tensor, W: int, stride: int, weights) -> torch.Tensor:
    out = torch.empty(int(plan.desc.n), dtype=torch.float32, device=messages.device)
    w = None
    if weights is not None:
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if w.size != W:
            raise ValueError(f"need {W} weights, got {w.size}")
    _lib.check(_lib.lib.fgc_decode_average(plan.handle, messages.data_ptr(), W, stride,
                                           None if w is None else w.ctypes.data, out.data_ptr(), D.stream()))
    return out


def decompress_device(message: CompressedMessage) -> torch.Tensor:
    """decompress on the device, returning the float32 device tensor."""
    plan, msg = message.device_message()
    return _decode(plan, msg, 1, plan.message_bytes, None)


def decompress(message: CompressedMessage) -> np.ndarray:
    """codec.py:246-270 on the GPU; float64 numpy output like the reference."""
    return decompress_device(message).double().cpu().numpy()


def reconstruct(gradient, config: CodecConfig) -> np.ndarray:
    """codec.py:273-289: decompress(compress()) without the wire."""
    t, code = _validated_signal(gradient)
    plan, msg, flags = _compress_device(t, code, config)
    out = _decode(plan, msg, 1, plan.message_bytes, None)
    D.raise_on_flags(D.read_flags(flags))
    return out.double().cpu().numpy()


def reconstruct_rows(rows, config: CodecConfig) -> np.ndarray:
    """codec.py:292-337: row-wise reconstruct of a 2-D array.  All rows go
    through one plan on the device back to back (compress + decode per row,
    no host round trip in between) and come back in one copy."""
    if isinstance(rows, torch.Tensor):
        r = rows.detach()
        if r.dim() != 2 or r.shape[1] == 0:
            raise ValueError("rows must be a non-empty 2D array")
        if r.dtype not in (torch.float32, torch.float64):
            r = r.to(torch.float64)
    else:
        a = np.asarray(rows)
        if a.ndim != 2 or a.shape[1] == 0:
            raise ValueError("rows must be a non-empty 2D array")
        r = torch.from_numpy(np.ascontiguousarray(a if a.dtype == np.float32 else a.astype(np.float64)))
    dev = D.require_cuda()
    R, n = int(r.shape[0]), int(r.shape[1])
    if R == 0:
        return np.empty((0, n), dtype=np.float64)
    # rows padded to an even length: every row starts 8/16-byte aligned
    buf = torch.zeros((R, n + (n & 1)), dtype=r.dtype, device=dev)
    buf[:, :n] = r.to(dev)
    code = _lib.DTYPE_F32 if buf.dtype == torch.float32 else _lib.DTYPE_F64
    spec = config.sparsification
    plan = get_plan(n, config.chunk_size, spec.theta, spec.mode, config.half_precision_pass, config.quantizer)
    mb = plan.message_bytes
    msgs = torch.empty(R * mb, dtype=torch.uint8, device=dev)
    out = torch.empty((R, (n + 3) & ~3), dtype=torch.float32, device=dev)   # 16-byte aligned rows
    flags = D.flags_tensor()
    for i in range(R):
        _lib.check(_lib.lib.fgc_compress(plan.handle, buf[i].data_ptr(), code, msgs[i * mb:].data_ptr(),
                                         flags.data_ptr(), D.stream()))
        _lib.check(_lib.lib.fgc_decode_average(plan.handle, msgs[i * mb:].data_ptr(), 1, mb, None,
                                               out[i].data_ptr(), D.stream()))
    D.raise_on_flags(D.read_flags(flags))
    return out[:, :n].double().cpu().numpy()


def _header(message: CompressedMessage) -> bytes:
    flags = 0
    if message.half_pass:
        flags |= FLAG_HALF_PASS
    if message.mode == "energy":
        flags |= FLAG_ENERGY
    q = message.quantizer
    if q is None:
        flags |= FLAG_PASSTHROUGH
        vals = (0.0, 0.0, 0.0, 32, 0)
    else:
        vals = (q.min, q.max, q.eps, q.n_bits, q.mantissa_bits)
    return struct.pack("<4sBBQIffffBB", MAGIC, VERSION, flags, message.original_len, message.chunk_size,
                       message.theta, *vals)


def serialize(message: CompressedMessage) -> bytes:
    """codec.py:340-374: the FGC1 bytes, assembled by the device serializer."""
    plan, msg = message.device_message()
    dev = msg.device
    wire = torch.empty(int(plan.info.wire_bytes_max), dtype=torch.uint8, device=dev)
    wlen = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(_lib.lib.fgc_serialize(plan.handle, msg.data_ptr(), wire.data_ptr(), wlen.data_ptr(), D.stream()))
    n = int(wlen.item())
    blob = bytearray(wire[:n].cpu().numpy().tobytes())
    # the plan's header carries the plan theta (float64); the message stores
    # float32(theta) like the reference -- both pack to the same f32 field.
    blob[:HEADER_BYTES] = _header(message)
    return bytes(blob)


def deserialize(data: bytes) -> CompressedMessage:
    """codec.py:377-441: header + framing validated on the host, payloads
    unpacked and popcount-checked on the device."""
    data = bytes(data)
    d = _lib.CodecDesc()
    _lib.check(_lib.lib.fgc_parse_header(data, len(data), C.byref(d)))
    quant = None
    if not d.passthrough:
        quant = QuantizerConfig(float(d.quant.min), float(d.quant.max), int(d.quant.n_bits),
                                int(d.quant.mantissa_bits), float(d.quant.eps), int(d.quant.pbase),
                                int(d.quant.pos_count))
    n, chunk = int(d.n), int(d.chunk_size)
    n_chunks = len(_chunk_lengths(n, chunk))
    offs = np.zeros(max(1, n_chunks), dtype=np.uint64)
    nnz = np.zeros(max(1, n_chunks), dtype=np.uint32)
    n_valid = C.c_uint32(0)
    st = _lib.lib.fgc_wire_index(data, len(data), C.byref(d), offs.ctypes.data, nnz.ctypes.data, C.byref(n_valid))
    fatal = None
    if st != _lib.OK:
        try:
            _lib.check(st)
        except CodecFormatError as exc:
            fatal = exc
    check_upto = int(n_valid.value) if fatal is not None else n_chunks
    mode = "energy" if d.mode == _lib.MODE_ENERGY else "count"
    theta = float(d.theta)
    plan = get_plan(n, chunk, theta, mode, bool(d.half_pass), quant, full_capacity=True)
    if check_upto or fatal is None:
        dev = D.require_cuda()
        wire = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
        # chunks past the truncation point are not copied: point them at chunk 0
        offs_eff = offs.copy()
        offs_eff[check_upto:] = offs[0] if check_upto else 0
        d_offs = torch.from_numpy(offs_eff.view(np.int64)).to(dev)
        msg = plan.new_message()
        pops = torch.empty(max(1, n_chunks), dtype=torch.int32, device=dev)
        if check_upto:
            _lib.check(_lib.lib.fgc_deserialize(plan.handle, wire.data_ptr(), d_offs.data_ptr(), msg.data_ptr(),
                                                pops.data_ptr(), D.stream()))
            p = pops.cpu().numpy().view(np.uint32)[:check_upto]
            bad = np.nonzero(p != nnz[:check_upto])[0]
            if bad.size:
                c = int(bad[0])
                raise BitmapMismatchError(f"bitmap marks {int(p[c])} slots, header says {int(nnz[c])}")
    if fatal is not None:
        raise fatal
    return CompressedMessage(n, chunk, theta, mode, bool(d.half_pass), quant, _device=(plan, msg))


def calibrate(sample_gradients, n_bits: int, mantissa_bits: int, eps_init: float = 0.002) -> QuantizerConfig:
    """codec.py:444-470: peak |Re|/|Im| of each sample's whole-vector float64
    rfft (GPU), then tune_eps on [-peak, peak]."""
    dev = None
    peak_t = None
    count = 0
    for sample in sample_gradients:
        t, code = D.as_signal(np.asarray(sample, dtype=np.float64) if not isinstance(sample, torch.Tensor)
                              else sample)
        if t.dim() != 1 or t.numel() == 0:
            raise ValueError("each sample must be a non-empty 1D sequence")
        if dev is None:
            dev = t.device
            peak_t = torch.zeros(1, dtype=torch.float64, device=dev)
        flags = D.flags_tensor()
        _lib.check(_lib.lib.fgc_spectrum_peak(t.data_ptr(), code, t.numel(), peak_t.data_ptr(),
                                              flags.data_ptr(), D.stream()))
        if D.read_flags(flags) & _lib.FLAG_NONFINITE:
            raise ValueError("samples must be finite")
        count += 1
    if count == 0:
        raise ValueError("calibration needs at least one sample")
    peak = float(peak_t.item())
    if peak == 0.0:
        raise ValueError("cannot calibrate from all-zero samples")
    return tune_eps(-peak, peak, n_bits, mantissa_bits, eps_init)


def compression_ratio(config: CodecConfig, n: int, include_bitmap: bool = False) -> float:
    """codec.py:473-493 (analytic; host arithmetic)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    theta = config.sparsification.theta
    n_bits = config.n_bits
    if not include_bitmap:
        if theta >= 1.0:
            raise ValueError("ratio is unbounded at theta = 1 without bitmap accounting")
        return 32.0 / (n_bits * (1.0 - theta))
    total_bits = HEADER_BYTES * 8
    for length in _chunk_lengths(n, config.chunk_size):
        slots = _slot_count(length)
        kept = (1.0 - theta) * slots
        total_bits += _KEPT.size * 8 + math.ceil(slots / 8) * 8 + n_bits * kept
    return 32.0 * n / total_bits
