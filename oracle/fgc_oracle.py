"""CPU oracle: a numpy restatement of the reference ``fgc`` codec path.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The product package
never imports this module.

Every function names the reference location it restates (paths relative to
``/root/reference/pkg/src/fgc``).  The arithmetic boundary is numpy itself
(the reference's only dependency, unpinned ``numpy>=1.24``,
``pkg/pyproject.toml:10-12``; this image has numpy 2.3.5): ``np.fft.rfft`` /
``irfft`` (pocketfft), ``np.abs`` on complex128 (numpy's SIMD cabs loop), a
stable ``np.argsort``, ``np.cumsum`` and ``np.packbits``.  Those calls are
kept, so the oracle reproduces the reference bit-for-bit on the same host;
``magnitude_exact`` restates numpy's cabs formula independently so the hazard
"SSE-only numpy computes a different key" is
detectable on any host.

Parity is pinned against the reference's golden wire fixtures and against
vectors produced by importing the reference (``tests/golden/``).
"""

from __future__ import annotations

import math
import struct
from fractions import Fraction
from typing import NamedTuple

import numpy as np

__all__ = [
    "Lattice", "lattice", "search_eps", "quantize", "dequantize",
    "codes_to_bytes", "bytes_to_codes", "flags_to_bytes", "bytes_to_flags",
    "half_roundtrip", "magnitude", "magnitude_exact", "parseval_weights",
    "drop_set", "Chunk", "Message", "chunk_lengths", "slot_count",
    "encode_spectrum", "compress", "decompress", "reconstruct_rows",
    "average", "to_wire", "from_wire", "calibrate", "WireError",
    "keep_bins", "device_layout", "device_segments", "from_device", "DEFAULT_CHUNK",
]

DEFAULT_CHUNK = 1 << 16          # codec.py:73
_MIN_CHUNK = 16                  # codec.py:72
_MIN_EPS = 2.0 ** -126           # quantizer.py:48
_TOP_PATTERN = 0x7F7FFFFF        # quantizer.py:52
_EPS_STEPS = 64                  # quantizer.py:54
_HDR = struct.Struct("<4sBBQIffffBB")   # codec.py:67 (36 bytes)


# ---------------------------------------------------------------- quantizer

def _f32_pattern(x: float) -> int:
    return int(np.array(x, dtype=np.float32).view(np.uint32))


def _pattern_f32(p: int) -> float:
    return float(np.array(p, dtype=np.uint32).view(np.float32))


class Lattice(NamedTuple):
    """The range-float code lattice (quantizer.py:71-151)."""

    lo: float
    hi: float
    n_bits: int
    mbits: int
    eps: float
    pbase: int
    npos: int

    @property
    def nneg(self) -> int:                       # quantizer.py:137-139
        return (1 << self.n_bits) - 1 - self.npos

    @property
    def shift(self) -> int:
        return 23 - self.mbits

    @property
    def floor(self) -> float:                    # actual_min, quantizer.py:141-145
        return -_pattern_f32((self.pbase + self.nneg - 1) << self.shift)

    @property
    def ceil(self) -> float:                     # actual_max, quantizer.py:147-151
        return _pattern_f32((self.pbase + self.npos - 1) << self.shift)


def _check_lattice(lat: Lattice) -> Lattice:
    """The validation of QuantizerConfig.__post_init__ (quantizer.py:89-106)."""
    n, m = lat.n_bits, lat.mbits
    if not 2 <= n <= 16:
        raise ValueError(f"n_bits must be in [2, 16], got {n}")
    if not 1 <= m < n:
        raise ValueError(f"mantissa_bits must satisfy 1 <= m < n_bits, got m={m}, N={n}")
    if not (math.isfinite(lat.lo) and math.isfinite(lat.hi)):
        raise ValueError("min/max must be finite")
    if not lat.lo < 0.0 < lat.hi:
        raise ValueError(f"range must straddle zero, got [{lat.lo}, {lat.hi}]")
    if not 0.0 < lat.eps < lat.hi:
        raise ValueError(f"eps must be in (0, max), got {lat.eps}")
    if lat.pbase != _f32_pattern(lat.eps) >> (23 - m):
        raise ValueError("pbase inconsistent with eps")
    if not 1 <= lat.npos <= (1 << n) - 2:
        raise ValueError("config leaves no room for positive or negative codes")
    if lat.pbase + lat.nneg - 1 > _TOP_PATTERN >> (23 - m):
        raise ValueError("negative lattice runs past the float32 range")
    return lat


def lattice(lo: float, hi: float, n_bits: int, mbits: int, eps: float) -> Lattice:
    """QuantizerConfig.from_params (quantizer.py:108-135): snap eps onto the
    lattice, derive pbase and the positive-code count, round the bounds
    through float32."""
    shift = 23 - mbits
    eps_l = _pattern_f32((_f32_pattern(eps) >> shift) << shift)
    pbase = _f32_pattern(eps_l) >> shift
    npos = (_f32_pattern(hi) >> shift) - pbase + 1
    return _check_lattice(Lattice(float(np.float32(lo)), float(np.float32(hi)),
                                  n_bits, mbits, eps_l, pbase, npos))


def search_eps(lo: float, hi: float, n_bits: int, mbits: int,
               eps0: float = 0.002) -> Lattice:
    """tune_eps (quantizer.py:154-214): halve/double eps until the most
    negative code crosses ``lo``; keep the closest candidate."""
    if not (math.isfinite(lo) and math.isfinite(hi) and lo < 0.0 < hi):
        raise ValueError(f"bounds must be finite with min < 0 < max, got [{lo}, {hi}]")
    if not 2 <= n_bits <= 16:
        raise ValueError(f"n_bits must be in [2, 16], got {n_bits}")
    if not 1 <= mbits < n_bits:
        raise ValueError(f"mantissa_bits must satisfy 1 <= m < N, got m={mbits}, N={n_bits}")
    if not (math.isfinite(eps0) and eps0 > 0.0):
        raise ValueError(f"eps_init must be positive and finite, got {eps0}")
    shift = 23 - mbits
    top = _f32_pattern(hi) >> shift
    limit = _TOP_PATTERN >> shift
    # quantizer.py:183: clip in float32 (NEP 50: the float32 bound is strong)
    upper = np.nextafter(np.float32(hi), np.float32(0.0))
    start = np.float32(min(max(np.float32(eps0), np.float32(_MIN_EPS)), upper))
    eps = _pattern_f32((_f32_pattern(float(start)) >> shift) << shift)
    best, best_gap, last = None, math.inf, None
    for _ in range(_EPS_STEPS):
        pb = _f32_pattern(eps) >> shift
        nneg = (1 << n_bits) - 2 - (top - pb)
        if nneg < 1:
            eps *= 2.0
            last = None
            continue
        if pb + nneg - 1 > limit:
            eps /= 2.0
            last = None
            continue
        cand = lattice(lo, hi, n_bits, mbits, eps)
        gap = cand.floor - lo
        if abs(gap) < best_gap:
            best, best_gap = cand, abs(gap)
        if gap == 0.0:
            return cand
        if last is not None and (gap > 0.0) != (last > 0.0):
            break
        last = gap
        eps = eps / 2.0 if gap < 0.0 else eps * 2.0
        if not _MIN_EPS < eps < hi:
            break
    if best is None:
        raise ValueError("eps tuning found no valid configuration")
    return best


def quantize(lat: Lattice, values) -> np.ndarray:
    """encode_array (quantizer.py:217-236): truncating range-float codes."""
    x = np.asarray(values, dtype=np.float32)
    if np.isnan(x).any():
        raise ValueError("cannot encode NaN")
    mag = np.abs(x)
    pos_cap = np.float32(lat.hi)
    neg_cap = np.float32(-lat.floor)
    sh = np.uint32(lat.shift)
    off_pos = (np.minimum(mag, pos_cap).view(np.uint32) >> sh).astype(np.int64) - lat.pbase + 1
    off_neg = (np.minimum(mag, neg_cap).view(np.uint32) >> sh).astype(np.int64) - lat.pbase + 1
    out = np.where(x > 0, np.minimum(off_pos, lat.npos),
                   lat.npos + np.minimum(off_neg, lat.nneg))
    out[mag < np.float32(lat.eps)] = 0
    return out.astype(np.uint32)


def dequantize(lat: Lattice, codes) -> np.ndarray:
    """decode_array (quantizer.py:239-253)."""
    c = np.asarray(codes).astype(np.int64)
    if c.size and (c.max() >= (1 << lat.n_bits) or c.min() < 0):
        raise ValueError(f"code out of range for N={lat.n_bits}")
    neg = c > lat.npos
    idx = np.where(neg, c - lat.npos, c)
    vals = ((lat.pbase + idx - 1) << lat.shift).astype(np.uint32).view(np.float32).copy()
    vals[neg] = -vals[neg]
    vals[c == 0] = 0.0
    return vals


def codes_to_bytes(codes, width: int) -> bytes:
    """pack_codes (quantizer.py:266-273): LSB-first ``width``-bit fields."""
    c = np.asarray(codes, dtype=np.uint64)
    if c.size == 0:
        return b""
    bits = (c[:, None] >> np.arange(width, dtype=np.uint64)) & np.uint64(1)
    return np.packbits(bits.astype(np.uint8).ravel(), bitorder="little").tobytes()


def bytes_to_codes(data: bytes, width: int, count: int) -> np.ndarray:
    """unpack_codes (quantizer.py:276-285)."""
    if count == 0:
        return np.zeros(0, dtype=np.uint32)
    need = (count * width + 7) // 8
    if len(data) < need:
        raise ValueError(f"packed code buffer too short: {len(data)} < {need} bytes")
    bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8), bitorder="little")
    bits = bits[: count * width].reshape(count, width).astype(np.uint64)
    return (bits << np.arange(width, dtype=np.uint64)).sum(axis=1).astype(np.uint32)


def flags_to_bytes(flags) -> bytes:
    """bitmap_to_bytes (packer.py:73-75): MSB-first, zero padded."""
    return np.packbits(np.asarray(flags, dtype=np.uint8), bitorder="big").tobytes()


def bytes_to_flags(data: bytes, length: int) -> np.ndarray:
    """bitmap_from_bytes (packer.py:78-84)."""
    need = (length + 7) // 8
    if len(data) < need:
        raise ValueError(f"bitmap buffer too short: {len(data)} < {need} bytes")
    return np.unpackbits(np.frombuffer(data, dtype=np.uint8), bitorder="big")[:length].astype(bool)


# ---------------------------------------------------------------- spectral

def half_roundtrip(v) -> np.ndarray:
    """half_round_trip (spectral.py:189-196): binary16 RNE and back."""
    with np.errstate(over="ignore"):
        return np.asarray(v, dtype=np.float64).astype(np.float16).astype(np.float64)


def magnitude(coeffs) -> np.ndarray:
    """The selection key of spectral.py:147 / codec.py:315: ``np.abs`` on
    complex128, i.e. numpy's SIMD cabs loop."""
    return np.abs(np.asarray(coeffs, dtype=np.complex128))


def magnitude_exact(re: float, im: float) -> float:
    """numpy's cabs formula restated with exact rational arithmetic:
    ``sqrt(fma(s/b, s/b, 1)) * b`` with b = max(|re|,|im|), s = min, and 0
    when b == 0 (numpy ``loops_unary_complex.dispatch.c.src``,
    ``simd_cabsolute``).  Used to pin ``magnitude`` on the running host."""
    a, b = abs(float(re)), abs(float(im))
    big, small = max(a, b), min(a, b)
    if big == 0.0:
        return 0.0
    r = small / big
    inner = float(Fraction(r) * Fraction(r) + 1)       # one rounding = fma
    return math.sqrt(inner) * big


def parseval_weights(n: int) -> np.ndarray:
    """bin_weights (spectral.py:109-115)."""
    w = np.full(n // 2 + 1, 2.0)
    w[0] = 1.0
    if n % 2 == 0:
        w[-1] = 1.0
    return w


def drop_set(mag: np.ndarray, energy: np.ndarray, theta: float, mode: str) -> np.ndarray:
    """_drop_set (spectral.py:124-139): smallest-first, ties to the lower
    index (stable ascending argsort)."""
    order = np.argsort(mag, kind="stable")
    if mode == "count":
        return order[: int(np.ceil(theta * mag.size))]
    if theta == 0.0:
        return order[:0]
    budget = theta ** 2 * float(energy.sum())
    running = np.cumsum(energy[order])
    return order[: int(np.searchsorted(running, budget, side="right"))]


def keep_bins(bins: int, theta: float) -> int:
    """Bins a count-mode selection keeps (spectral.py:131-132)."""
    return bins - int(np.ceil(theta * bins))


# ---------------------------------------------------------------- codec

class WireError(ValueError):
    """Restates the CodecFormatError family (codec.py:76-89); ``kind`` is
    'header', 'truncated', 'bitmap' or 'format'."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class Chunk(NamedTuple):
    bitmap: np.ndarray     # bool[slots]  (ChunkPayload, codec.py:112-125)
    codes: np.ndarray      # uint32[nnz]


class Message(NamedTuple):
    n: int
    chunk: int
    theta32: float
    mode: str
    half: bool
    lat: Lattice | None
    chunks: list

    @property
    def width(self) -> int:
        return 32 if self.lat is None else self.lat.n_bits


def chunk_lengths(n: int, chunk: int) -> list:
    """_chunk_lengths (codec.py:163-167)."""
    out = [chunk] * (n // chunk)
    if n % chunk:
        out.append(n % chunk)
    return out


def slot_count(length: int) -> int:
    """_slot_count (codec.py:170-171)."""
    return 2 * (length // 2 + 1)


def _to_codes(slots: np.ndarray, lat: Lattice | None) -> np.ndarray:
    """_quantize_parts (codec.py:174-180); passthrough folds -0.0."""
    if lat is None:
        f = slots.astype(np.float32)
        f[f == 0.0] = 0.0
        return f.view(np.uint32)
    return quantize(lat, slots)


def _from_codes(codes: np.ndarray, lat: Lattice | None) -> np.ndarray:
    """_dequantize_codes (codec.py:183-186)."""
    if lat is None:
        return codes.astype(np.uint32).view(np.float32).astype(np.float64)
    return dequantize(lat, codes).astype(np.float64)


def encode_spectrum(coeffs, length: int, theta: float, mode: str,
                    lat: Lattice | None):
    """Stage-injection oracle: the part of _chunk_codes (codec.py:209-217)
    after the forward DFT -- truncate (spectral.py:142-156), interleave
    (codec.py:197-202), quantize, then pack (packer.py:49-58).

    Returns ``(kept_mask[bins], Chunk)``."""
    c = np.asarray(coeffs, dtype=np.complex128).copy()
    mag = magnitude(c)
    energy = parseval_weights(length) * mag ** 2
    dropped = drop_set(mag, energy, theta, mode)
    kept = np.ones(c.size, dtype=bool)
    kept[dropped] = False
    c[dropped] = 0.0
    slots = np.empty(2 * c.size, dtype=np.float64)
    slots[0::2] = c.real
    slots[1::2] = c.imag
    codes = _to_codes(slots, lat)
    nz = codes != 0
    return kept, Chunk(nz, codes[nz].astype(np.uint32))


def _check_gradient(v: np.ndarray) -> None:
    if v.ndim != 1 or v.size == 0:
        raise ValueError("gradient must be a non-empty 1D sequence")
    if not np.isfinite(v).all():
        raise ValueError("gradient must be finite")


def _chunk_signal(piece: np.ndarray, half: bool) -> np.ndarray:
    if half:
        piece = half_roundtrip(piece)
        if not np.isfinite(piece).all():
            raise ValueError("gradient overflowed binary16 during the half-precision pass")
    return piece


def compress(gradient, theta: float, mode: str = "count", lat: Lattice | None = None,
             half: bool = False, chunk: int = DEFAULT_CHUNK) -> Message:
    """compress (codec.py:220-243)."""
    if chunk < _MIN_CHUNK:
        raise ValueError(f"chunk_size must be >= {_MIN_CHUNK}, got {chunk}")
    v = np.asarray(gradient, dtype=np.float64)
    _check_gradient(v)
    chunks, pos = [], 0
    for length in chunk_lengths(v.size, chunk):
        piece = _chunk_signal(v[pos:pos + length], half)
        spec = np.fft.rfft(piece)                       # spectral.py:95
        chunks.append(encode_spectrum(spec, length, theta, mode, lat)[1])
        pos += length
    return Message(v.size, chunk, float(np.float32(theta)), mode, half, lat, chunks)


def decompress(msg: Message) -> np.ndarray:
    """decompress (codec.py:246-270): unpack, dequantize, irfft per chunk."""
    lengths = chunk_lengths(msg.n, msg.chunk)
    if len(lengths) != len(msg.chunks):
        raise WireError("truncated", f"message has {len(msg.chunks)} chunks, expected {len(lengths)}")
    out = np.empty(msg.n, dtype=np.float64)
    pos = 0
    for length, ch in zip(lengths, msg.chunks):
        slots = slot_count(length)
        bm = np.asarray(ch.bitmap, dtype=bool)
        if bm.size != slots or int(bm.sum()) != ch.codes.size:
            raise WireError("bitmap", "bitmap/payload mismatch")
        dense = np.zeros(slots, dtype=np.uint32)
        dense[bm] = ch.codes
        parts = _from_codes(dense, msg.lat)
        out[pos:pos + length] = np.fft.irfft(parts[0::2] + 1j * parts[1::2], n=length)
        pos += length
    return out


def reconstruct_rows(rows, theta: float, mode: str = "count", lat: Lattice | None = None,
                     half: bool = False, chunk: int = DEFAULT_CHUNK) -> np.ndarray:
    """reconstruct_rows (codec.py:292-337) == row-wise decompress(compress())
    (asserted bit-identical by the reference, test_codec.py:138-152)."""
    rows = np.asarray(rows, dtype=np.float64)
    if rows.ndim != 2 or rows.shape[1] == 0:
        raise ValueError("rows must be a non-empty 2D array")
    return np.stack([decompress(compress(r, theta, mode, lat, half, chunk)) for r in rows])


def average(rows, weights, theta: float, mode: str = "count", lat: Lattice | None = None,
            half: bool = False, chunk: int = DEFAULT_CHUNK) -> np.ndarray:
    """The simulator's averaging step (simulator.py:520-547): per-worker
    codec round trip, then ``shard_weights @ recon`` in worker order."""
    w = np.asarray(weights, dtype=np.float64)
    if theta == 0.0 and lat is None:                   # simulator.py:520,543-545
        return w @ np.asarray(rows, dtype=np.float64)
    return w @ reconstruct_rows(rows, theta, mode, lat, half, chunk)


def to_wire(msg: Message) -> bytes:
    """serialize (codec.py:340-374)."""
    flags = (1 if msg.half else 0) | (2 if msg.mode == "energy" else 0) | (4 if msg.lat is None else 0)
    if msg.lat is None:
        qlo = qhi = qeps = 0.0
        nb, mb = 32, 0
    else:
        qlo, qhi, qeps, nb, mb = msg.lat.lo, msg.lat.hi, msg.lat.eps, msg.lat.n_bits, msg.lat.mbits
    out = [_HDR.pack(b"FGC1", 1, flags, msg.n, msg.chunk, msg.theta32, qlo, qhi, qeps, nb, mb)]
    for ch in msg.chunks:
        out.append(struct.pack("<I", ch.codes.size))
        out.append(flags_to_bytes(ch.bitmap))
        out.append(codes_to_bytes(ch.codes, msg.width))
    return b"".join(out)


def from_wire(data: bytes) -> Message:
    """deserialize (codec.py:377-441) with the same validation order."""
    if len(data) < _HDR.size:
        raise WireError("truncated", f"buffer of {len(data)} bytes is shorter than the header")
    magic, ver, flags, n, chunk, theta, qlo, qhi, qeps, nb, mb = _HDR.unpack_from(data, 0)
    if magic != b"FGC1":
        raise WireError("header", f"bad magic {magic!r}")
    if ver != 1:
        raise WireError("header", f"unsupported version {ver}")
    if flags & ~0x07:
        raise WireError("header", f"unknown flag bits in 0x{flags:02x}")
    if n < 1:
        raise WireError("header", "original_len must be >= 1")
    if chunk < _MIN_CHUNK:
        raise WireError("header", f"chunk_size {chunk} below minimum {_MIN_CHUNK}")
    if not (np.isfinite(theta) and 0.0 <= theta <= 1.0):
        raise WireError("header", f"theta {theta} outside [0, 1]")
    passthrough = bool(flags & 4)
    if passthrough:
        if nb != 32:
            raise WireError("header", "passthrough flag requires N=32")
        lat = None
    else:
        try:
            lat = lattice(qlo, qhi, nb, mb, qeps)
        except ValueError as exc:
            raise WireError("header", f"invalid quantizer parameters: {exc}") from exc
    width = 32 if passthrough else nb
    pos, chunks = _HDR.size, []
    for length in chunk_lengths(n, chunk):
        slots = slot_count(length)
        if pos + 4 > len(data):
            raise WireError("truncated", "buffer ended before chunk header")
        (nnz,) = struct.unpack_from("<I", data, pos)
        pos += 4
        bmb = (slots + 7) // 8
        if pos + bmb > len(data):
            raise WireError("truncated", "buffer ended inside the bitmap")
        bm = bytes_to_flags(data[pos:pos + bmb], slots)
        pos += bmb
        if int(bm.sum()) != nnz:
            raise WireError("bitmap", f"bitmap marks {int(bm.sum())} slots, header says {nnz}")
        cb = (nnz * width + 7) // 8
        if pos + cb > len(data):
            raise WireError("truncated", "buffer ended inside the packed codes")
        chunks.append(Chunk(bm, bytes_to_codes(data[pos:pos + cb], width, nnz)))
        pos += cb
    if pos != len(data):
        raise WireError("format", f"{len(data) - pos} unexpected trailing bytes")
    return Message(n, chunk, float(theta), "energy" if flags & 2 else "count",
                   bool(flags & 1), lat, chunks)


def calibrate(samples, n_bits: int, mbits: int, eps0: float = 0.002) -> Lattice:
    """calibrate (codec.py:444-470): whole-vector rfft peak of |Re|, |Im|."""
    peak, count = 0.0, 0
    for s in samples:
        v = np.asarray(s, dtype=np.float64)
        if v.ndim != 1 or v.size == 0:
            raise ValueError("each sample must be a non-empty 1D sequence")
        if not np.isfinite(v).all():
            raise ValueError("samples must be finite")
        spec = np.fft.rfft(v)
        peak = max(peak, float(np.abs(spec.real).max()), float(np.abs(spec.imag).max()))
        count += 1
    if count == 0:
        raise ValueError("calibration needs at least one sample")
    if peak == 0.0:
        raise ValueError("cannot calibrate from all-zero samples")
    return search_eps(-peak, peak, n_bits, mbits, eps0)


# ------------------------------------------- device message layout (ours)
#
# The GPU keeps one fixed-capacity segment per chunk (DESIGN.md "Device
# message"): [u32 nnz][12 B zero][bitmap words, wire bit order][pad to 16]
# [codes, LSB-first words][pad to 16].  The first ceil(slots/8) bitmap bytes
# and the first ceil(nnz*N/8) code bytes are exactly the FGC1 wire bytes.

def _a16(x: int) -> int:
    return (x + 15) & ~15


def device_layout(n: int, chunk: int, theta: float, width: int, mode: str = "count"):
    """Per-chunk (offset, bitmap_offset, code_offset, capacity) list and the
    total message bytes, restating ``fgc_layout`` in csrc/plan.cpp."""
    out, off = [], 0
    for length in chunk_lengths(n, chunk):
        slots = slot_count(length)
        bins = length // 2 + 1
        maxnz = slots if mode != "count" else 2 * keep_bins(bins, theta)
        bm_words = (slots + 31) // 32
        code_off = 16 + _a16(4 * bm_words)
        cap = code_off + _a16(4 * ((maxnz * width + 31) // 32))
        out.append((off, 16, code_off, cap))
        off += cap
    return out, off


def from_device(buf: bytes, n: int, chunk: int, theta: float, lat: Lattice | None,
                mode: str = "count", half: bool = False) -> Message:
    """Parse a fixed-capacity device message back into a Message."""
    width = 32 if lat is None else lat.n_bits
    layout, total = device_layout(n, chunk, theta, width, mode)
    if len(buf) < total:
        raise ValueError("device message shorter than its layout")
    chunks = []
    for (off, bmo, co, cap), length in zip(layout, chunk_lengths(n, chunk)):
        slots = slot_count(length)
        nnz = struct.unpack_from("<I", buf, off)[0]
        bm = bytes_to_flags(buf[off + bmo: off + bmo + (slots + 7) // 8], slots)
        cb = (nnz * width + 7) // 8
        chunks.append(Chunk(bm, bytes_to_codes(buf[off + co: off + co + cb], width, nnz)))
    return Message(n, chunk, float(np.float32(theta)), mode, half, lat, chunks)


def device_segments(msg: Message, theta: float) -> bytes:
    """The valid bytes of each device segment, zero elsewhere."""
    layout, total = device_layout(msg.n, msg.chunk, theta, msg.width, msg.mode)
    buf = bytearray(total)
    for (off, bmo, co, cap), ch in zip(layout, msg.chunks):
        struct.pack_into("<I", buf, off, ch.codes.size)
        bm = flags_to_bytes(ch.bitmap)
        buf[off + bmo: off + bmo + len(bm)] = bm
        cb = codes_to_bytes(ch.codes, msg.width)
        if len(cb) > cap - co:
            raise ValueError("chunk exceeds its device capacity")
        buf[off + co: off + co + len(cb)] = cb
    return bytes(buf)
