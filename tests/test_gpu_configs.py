"""Bit-exact parity at every BASELINE.json configuration, full size.

For C2 (25.6M floats), C3 (61M, theta_drop in {0.99, 0.95, 0.9, 0.7}) and
C4 (138M, (N, m) in {(4,2), (6,2), (8,3), (16,9)}) the WHOLE device message
of ``compress`` (every one of the 391 / 931 / 2106 chunk segments: nnz,
bitmap bytes, packed code bytes) is compared byte for byte with the oracle's
encoding (truncate -> interleave -> quantize -> pack, codec.py:209-217,
spectral.py:124-156, quantizer.py:217-236, packer.py:49-58) of the GPU's own
forward coefficients (the fp32 FFT is checked against numpy's float64 rfft
in test_gpu_codec.py).  The decoded gradient of every chunk is compared with
the oracle's float64 decode of the same payload (rel-L2 <= 1e-5 per chunk,
codec.py:246-270).

The oracle runs chunk-parallel on the host's cores (fork pool; the GPU
spectrum, message and decode are inherited copy-on-write), so a 2106-chunk
configuration takes seconds.
"""

import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import oracle as O
from oracle import fgc_oracle as OO

pytestmark = pytest.mark.gpu

F = pytest.importorskip("paper_1811_08596_b200")
from paper_1811_08596_b200 import debug  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

CHUNK = 65536
_S = {}          # state inherited by the fork workers


def _check_chunk(c):
    """Worker: (chunk, byte_equal, kept_flips, code_diffs, rel_l2 of the decode)."""
    s = _S
    L = s["lengths"][c]
    b0, b1 = s["bin_off"][c], s["bin_off"][c + 1]
    kept, ch = O.encode_spectrum(s["spec"][b0:b1], L, s["theta"], s["mode"], s["lat"])
    off, bmo, co, _ = s["layout"][c]
    buf = s["msg"]
    nnz = int.from_bytes(buf[off:off + 4], "little")
    bmb = (2 * (L // 2 + 1) + 7) // 8
    bm = buf[off + bmo:off + bmo + bmb]
    cb = buf[off + co:off + co + (nnz * s["width"] + 7) // 8]
    want_bm = O.flags_to_bytes(ch.bitmap)
    want_cb = O.codes_to_bytes(ch.codes, s["width"])
    equal = nnz == ch.codes.size and bm == want_bm and cb == want_cb
    flips = codes = 0
    if not equal:
        got_bm = O.bytes_to_flags(bm, 2 * (L // 2 + 1))
        flips = int(np.count_nonzero(got_bm != ch.bitmap))
        if flips == 0 and nnz == ch.codes.size:
            codes = int(np.count_nonzero(O.bytes_to_codes(cb, s["width"], nnz) != ch.codes))
    # decode parity: the oracle's float64 decode of the GPU payload
    dense = np.zeros(2 * (L // 2 + 1), dtype=np.uint32)
    got_bm = O.bytes_to_flags(bm, 2 * (L // 2 + 1))
    dense[got_bm] = O.bytes_to_codes(cb, s["width"], nnz)
    parts = OO._from_codes(dense, s["lat"])
    ref = np.fft.irfft(parts[0::2] + 1j * parts[1::2], n=L)
    got = s["out"][s["in_off"][c]:s["in_off"][c] + L]
    nr = np.linalg.norm(ref)
    rel = float(np.linalg.norm(got - ref) / nr) if nr else float(np.linalg.norm(got))
    return c, equal, flips, codes, rel


def _pool_map(fn, items):
    ctx = mp.get_context("fork")
    cores = max(1, min(32, len(os.sched_getaffinity(0))))
    with ctx.Pool(cores) as pool:
        return pool.map(fn, items, chunksize=max(1, len(items) // (8 * cores)))


def _full_message_parity(n, theta, nm, seed=0, mode="count", half=False, f64=False):
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(seed)) * 1e-2
    if f64:
        g = g.double()
    q = F.calibrate([g[:CHUNK * 4].double().cpu().numpy()], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q, half_precision_pass=half, chunk_size=CHUNK)
    m1 = F.compress(g, cfg)
    m2 = F.compress(g, cfg)
    b1, b2 = debug.message_bytes(m1), debug.message_bytes(m2)
    assert b1 == b2                                   # deterministic across runs
    out1 = F.codec.decompress_device(m1)
    out2 = F.codec.decompress_device(m2)
    assert torch.equal(out1, out2)
    spec = debug.forward_spectrum(g, cfg)
    lengths = O.chunk_lengths(n, CHUNK)
    bins = [L // 2 + 1 for L in lengths]
    layout, total = O.device_layout(n, CHUNK, theta, nm[0], mode)
    assert len(b1) == total
    _S.update(spec=spec, msg=b1, out=out1.double().cpu().numpy(), theta=theta, width=nm[0], mode=mode,
              lat=O.lattice(q.min, q.max, q.n_bits, q.mantissa_bits, q.eps), lengths=lengths,
              bin_off=np.concatenate([[0], np.cumsum(bins)]), in_off=np.concatenate([[0], np.cumsum(lengths)]),
              layout=layout)
    try:
        res = _pool_map(_check_chunk, list(range(len(lengths))))
    finally:
        _S.clear()
    bad = [r for r in res if not r[1]]
    worst = max(r[4] for r in res)
    print(f"n={n} theta={theta} nm={nm} mode={mode} half={half} f64={f64}: {len(res)} chunks, {len(bad)} differ "
          f"(kept flips {sum(r[2] for r in bad)}, code diffs {sum(r[3] for r in bad)}), "
          f"worst per-chunk decode rel-L2 {worst:.2e}")
    assert not bad, bad[:5]
    assert worst <= 1e-5


def test_c2_resnet50_full_message_bit_exact():
    """BASELINE config 2: 25.6M floats, keep 0.1, (8,3); all 391 chunks."""
    _full_message_parity(25_600_000, 0.9, (8, 3))


@pytest.mark.parametrize("mode,half,f64", [("energy", False, False), ("count", True, False), ("count", False, True)])
def test_c2_variants_full_message_bit_exact(mode, half, f64):
    """C2 through the other code paths of the fused kernels: energy mode
    (the energy drop set on the fused forward transform), the binary16
    half-precision pass (the HALF load), float64 input (the double load)."""
    _full_message_parity(25_600_000, 0.9, (8, 3), seed=3, mode=mode, half=half, f64=f64)


@pytest.mark.parametrize("theta", [0.99, 0.95, 0.9, 0.7])
def test_c3_alexnet_theta_sweep_full_message_bit_exact(theta):
    """BASELINE config 3: 61M floats, keep ratio 0.01 / 0.05 / 0.1 / 0.3."""
    _full_message_parity(61_000_000, theta, (8, 3), seed=1)


@pytest.mark.parametrize("nm", [(4, 2), (6, 2), (8, 3), (16, 9)])
def test_c4_vgg16_bit_sweep_full_message_bit_exact(nm):
    """BASELINE config 4: 138M floats, 4/6/8/16-bit range floats."""
    _full_message_parity(138_000_000, 0.9, nm, seed=2)


@pytest.mark.parametrize("kernel", [1, 4])
def test_alternative_compress_kernels_full_message(kernel):
    """The selectable compress variants (FGC_COMPRESS_KERNEL): 1 = 1024-thread
    CTAs with lane-pair FFT columns (fused_w.cu), 4 = 4-CTA clusters
    (fused4.cu).  Each is byte-exact against the oracle's encoding of its own
    coefficients at C2 size; the 1024-thread kernel computes the same
    coefficients as the default, so its message is byte-equal to the
    default's too."""
    import ctypes
    from paper_1811_08596_b200 import _lib
    setk = _lib.lib.fgc_debug_set_compress_kernel
    setk.argtypes = [ctypes.c_int]
    n = 25_600_000
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
    q = F.calibrate([g[:CHUNK * 4].double().cpu().numpy()], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=CHUNK)
    default = debug.message_bytes(F.compress(g, cfg))
    try:
        setk(kernel)
        if kernel == 1:
            assert debug.message_bytes(F.compress(g, cfg)) == default
        _full_message_parity(n, 0.9, (8, 3))
    finally:
        setk(2)
