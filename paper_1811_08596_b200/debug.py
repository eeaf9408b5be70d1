"""Stage-level entry points for parity testing (SURVEY.md 8c "stage
injection"): the forward coefficients the codec quantizes, encoding a given
spectrum, and decoding to a spectrum.  All run on the GPU through the C ABI.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _lib
from .codec import CodecConfig, CompressedMessage, Plan, _validated_signal, get_plan

__all__ = ["forward_spectrum", "encode_spectrum", "decode_spectrum", "inverse_spectrum", "plan_for",
           "message_bytes"]


def plan_for(n: int, config: CodecConfig) -> Plan:
    s = config.sparsification
    return get_plan(n, config.chunk_size, s.theta, s.mode, config.half_precision_pass, config.quantizer)


def forward_spectrum(gradient, config: CodecConfig) -> np.ndarray:
    """Chunk-major complex64 coefficients exactly as compress() computes them."""
    t, code = _validated_signal(gradient)
    plan = plan_for(t.numel(), config)
    out = torch.empty((int(plan.info.spectrum_bins), 2), dtype=torch.float32, device=t.device)
    flags = D.flags_tensor()
    _lib.check(_lib.lib.fgc_forward_spectrum(plan.handle, t.data_ptr(), code, out.data_ptr(), flags.data_ptr(),
                                             D.stream()))
    D.raise_on_flags(D.read_flags(flags))
    return out.cpu().numpy().view(np.complex64).reshape(-1)


def encode_spectrum(spectrum, n: int, config: CodecConfig):
    """Quantize + pack a given chunk-major complex64 spectrum.
    Returns (CompressedMessage, kept_mask[bins] bool)."""
    plan = plan_for(n, config)
    sp = np.ascontiguousarray(np.asarray(spectrum, dtype=np.complex64)).view(np.float32)
    if sp.size != 2 * int(plan.info.spectrum_bins):
        raise ValueError("spectrum does not match the plan's bin count")
    dev = D.require_cuda()
    t = torch.from_numpy(sp.copy()).to(dev)
    msg = plan.new_message()
    mask = torch.empty(int(plan.info.spectrum_bins), dtype=torch.uint8, device=dev)
    flags = D.flags_tensor()
    _lib.check(_lib.lib.fgc_encode_spectrum(plan.handle, t.data_ptr(), msg.data_ptr(), mask.data_ptr(),
                                            flags.data_ptr(), D.stream()))
    D.raise_on_flags(D.read_flags(flags))
    s = config.sparsification
    m = CompressedMessage(n, config.chunk_size, float(np.float32(s.theta)), s.mode, config.half_precision_pass,
                          config.quantizer, _device=(plan, msg))
    return m, mask.cpu().numpy().astype(bool)


def message_bytes(message: CompressedMessage) -> bytes:
    """The raw fixed-capacity device message."""
    plan, msg = message.device_message()
    return msg.cpu().numpy().tobytes()


def decode_spectrum(messages: list, weights=None) -> np.ndarray:
    """Weighted frequency-domain average of messages sharing one plan."""
    plan, _ = messages[0].device_message()
    stacked = torch.cat([m.device_message()[1] for m in messages])
    W = len(messages)
    out = torch.empty((int(plan.info.spectrum_bins), 2), dtype=torch.float32, device=stacked.device)
    w = None if weights is None else np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    _lib.check(_lib.lib.fgc_decode_spectrum(plan.handle, stacked.data_ptr(), W, plan.message_bytes,
                                            None if w is None else w.ctypes.data, out.data_ptr(), D.stream()))
    return out.cpu().numpy().view(np.complex64).reshape(-1)


def decode_average(messages: list, weights=None) -> np.ndarray:
    """fgc_decode_average over stacked device messages (one plan)."""
    plan, _ = messages[0].device_message()
    stacked = torch.cat([m.device_message()[1] for m in messages])
    W = len(messages)
    out = torch.empty(int(plan.desc.n), dtype=torch.float32, device=stacked.device)
    w = None if weights is None else np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    _lib.check(_lib.lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes,
                                           None if w is None else w.ctypes.data, out.data_ptr(), D.stream()))
    return out.cpu().numpy()


def inverse_spectrum(spectrum, n: int, config: CodecConfig) -> np.ndarray:
    plan = plan_for(n, config)
    sp = np.ascontiguousarray(np.asarray(spectrum, dtype=np.complex64)).view(np.float32)
    dev = D.require_cuda()
    t = torch.from_numpy(sp.copy()).to(dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(_lib.lib.fgc_inverse_spectrum(plan.handle, t.data_ptr(), out.data_ptr(), D.stream()))
    return out.cpu().numpy()
