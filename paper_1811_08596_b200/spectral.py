"""Real DFT and magnitude truncation -- drop-in for the hot-path part of
``fgc.spectral`` (pkg/src/fgc/spectral.py).

``dft_forward`` / ``dft_inverse`` run a float64 GPU DFT (any length, like
numpy's pocketfft); ``truncate`` runs the GPU selection -- count mode, or
energy mode (numpy's pairwise total, stable order and sequential cumulative
energy, csrc/energy.cu) -- with numpy's exact complex-abs key and the stable
index tie-break.  The time-domain audit helpers (``sparsify_time``,
``assumption_check``) are outside this build's scope.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib

__all__ = ["Spectrum", "SparsificationSpec", "dft_forward", "dft_inverse", "truncate",
           "half_round_trip", "bin_weights", "spectrum_energy"]


@dataclass(frozen=True)
class Spectrum:
    """Half spectrum of a length-n real signal (spectral.py:43-56)."""

    coefficients: np.ndarray
    n: int

    def __post_init__(self) -> None:
        object.__setattr__(self, "coefficients", np.asarray(self.coefficients, dtype=np.complex128))
        if self.n < 1:
            raise ValueError("signal length must be >= 1")

    @property
    def bins(self) -> int:
        return self.coefficients.shape[0]


@dataclass(frozen=True)
class SparsificationSpec:
    """Dropout ratio theta plus mode and domain (spectral.py:61-76)."""

    theta: float
    mode: str = "count"
    domain: str = "frequency"

    def __post_init__(self) -> None:
        if not (0.0 <= self.theta <= 1.0):
            raise ValueError(f"theta must be in [0, 1], got {self.theta}")
        if self.mode not in ("count", "energy"):
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.domain not in ("frequency", "time"):
            raise ValueError(f"unknown domain {self.domain!r}")


def dft_forward(signal) -> Spectrum:
    """spectral.py:88-95 on the GPU (float64)."""
    v = np.asarray(signal, dtype=np.float64)
    if v.ndim != 1 or v.size == 0:
        raise ValueError("signal must be a non-empty 1D sequence")
    t, code = D.as_signal(v)
    out = torch.empty((v.size // 2 + 1, 2), dtype=torch.float64, device=t.device)
    flags = D.flags_tensor()
    _lib.check(_lib.lib.fgc_rfft(t.data_ptr(), code, v.size, out.data_ptr(), flags.data_ptr(), D.stream()))
    if D.read_flags(flags) & _lib.FLAG_NONFINITE:
        raise ValueError("signal must be finite")
    return Spectrum(out.cpu().numpy().view(np.complex128).reshape(-1), v.size)


def dft_inverse(spectrum: Spectrum) -> np.ndarray:
    """spectral.py:98-106 on the GPU (float64; Im of DC/Nyquist ignored)."""
    expected = spectrum.n // 2 + 1
    if spectrum.bins != expected:
        raise ValueError(f"half spectrum of a length-{spectrum.n} signal needs {expected} bins, "
                         f"got {spectrum.bins}")
    dev = D.require_cuda()
    src = torch.from_numpy(np.ascontiguousarray(spectrum.coefficients).view(np.float64).copy()).to(dev)
    out = torch.empty(spectrum.n, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib.fgc_irfft(src.data_ptr(), spectrum.n, out.data_ptr(), D.stream()))
    return out.cpu().numpy()


def bin_weights(n: int) -> np.ndarray:
    """spectral.py:109-115 (Parseval weights)."""
    w = np.full(n // 2 + 1, 2.0)
    w[0] = 1.0
    if n % 2 == 0:
        w[-1] = 1.0
    return w


def spectrum_energy(spectrum: Spectrum) -> float:
    """spectral.py:118-121 (reporting helper)."""
    w = bin_weights(spectrum.n)
    return float(np.sum(w * np.abs(spectrum.coefficients) ** 2) / spectrum.n)


def truncate(spectrum: Spectrum, spec: SparsificationSpec) -> tuple[Spectrum, np.ndarray]:
    """spectral.py:142-156 on the GPU.  count: zero the ceil(theta*bins)
    smallest-magnitude bins (ties to the lower index); energy: zero the
    smallest bins whose cumulative Parseval energy stays within theta**2 of
    the total (spectral.py:134-139)."""
    if spec.domain != "frequency":
        raise ValueError(f"truncate expects a frequency-domain spec, got {spec.domain!r}")
    dev = D.require_cuda()
    bins = spectrum.bins
    src = torch.from_numpy(np.ascontiguousarray(spectrum.coefficients).view(np.float64).copy()).to(dev)
    out = torch.empty_like(src)
    mask = torch.empty(bins, dtype=torch.uint8, device=dev)
    mode = _lib.MODE_ENERGY if spec.mode == "energy" else _lib.MODE_COUNT
    _lib.check(_lib.lib.fgc_truncate_mode(src.data_ptr(), bins, spectrum.n, float(spec.theta), mode, out.data_ptr(),
                                          mask.data_ptr(), D.stream()))
    coeffs = out.cpu().numpy().view(np.complex128).reshape(-1)
    return Spectrum(coeffs, spectrum.n), mask.cpu().numpy().astype(bool)


def half_round_trip(signal) -> np.ndarray:
    """spectral.py:189-196 on the GPU: binary16 RNE and back."""
    v = np.asarray(signal, dtype=np.float64)
    if v.size == 0:
        return v.copy()
    dev = D.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(v.reshape(-1))).to(dev)
    out = torch.empty_like(t)
    _lib.check(_lib.lib.fgc_half_round_trip(t.data_ptr(), t.numel(), out.data_ptr(), D.stream()))
    return out.cpu().numpy().reshape(v.shape)
