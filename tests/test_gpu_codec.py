"""GPU parity tests: the CUDA path through the C ABI against the CPU oracle
(oracle/, pinned to the reference) and the reference's golden vectors.

Bars (SURVEY.md 8c / DESIGN.md "Parity"):
  * bitmap, codes, kept mask: BIT-EXACT given identical coefficients
    (stage injection);
  * forward coefficients vs numpy's float64 rfft: max error <= 2e-6 x the
    chunk's coefficient RMS-scale (fp32 FFT);
  * decoded / averaged gradients vs the oracle on the same message:
    rel-L2 <= 1e-5;
  * wire bytes: byte-exact round trips of the reference fixtures.
"""

import hashlib

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

F = pytest.importorskip("paper_1811_08596_b200")
from paper_1811_08596_b200 import debug  # noqa: E402

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def lat_of(q):
    return None if q is None else O.lattice(q.min, q.max, q.n_bits, q.mantissa_bits, q.eps)


def q_of(rec):
    if rec is None:
        return None
    return F.QuantizerConfig.from_params(rec["min"], rec["max"], rec["n_bits"], rec["mantissa_bits"], rec["eps"])


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    a = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)
    b = b.astype(np.complex128 if np.iscomplexobj(b) else np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)


def segments_valid_bytes(dev: bytes, n, chunk, theta, width, mode="count"):
    """Per chunk: nnz, wire bitmap bytes, wire code bytes from a device message."""
    layout, _ = O.device_layout(n, chunk, theta, width, mode)
    out = []
    for (off, bmo, co, cap), L in zip(layout, O.chunk_lengths(n, chunk)):
        nnz = int.from_bytes(dev[off:off + 4], "little")
        bmb = (O.slot_count(L) + 7) // 8
        cb = (nnz * width + 7) // 8
        out.append((nnz, dev[off + bmo:off + bmo + bmb], dev[off + co:off + co + cb]))
    return out


# ---------------------------------------------------------------- injection

def test_injection_golden_vectors(golden):
    meta, arr = golden
    for rec in meta["injection"]:
        L, theta = rec["length"], rec["theta"]
        q = q_of(rec["quantizer"])
        cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=max(16, L))
        coeffs = arr[rec["key"] + "_coeffs"]
        msg, mask = debug.encode_spectrum(coeffs, L, cfg)
        np.testing.assert_array_equal(mask, arr[rec["key"] + "_mask"], err_msg=rec["key"])
        width = 32 if q is None else q.n_bits
        (nnz, bm, cb), = segments_valid_bytes(debug.message_bytes(msg), L, max(16, L), theta, width)
        assert nnz == rec["kept"], rec["key"]
        assert bm.hex() == rec["bitmap_hex"], rec["key"]
        assert cb.hex() == rec["codes_hex"], rec["key"]


def _random_spectrum(rng, n, chunk, ties=True):
    bins = [L // 2 + 1 for L in O.chunk_lengths(n, chunk)]
    parts = []
    for b in bins:
        scale = np.exp(rng.uniform(-3, 3))
        c = (rng.standard_normal(b) + 1j * rng.standard_normal(b)) * scale
        c[0] = c[0].real
        if ties:
            c[5::97] = c[5]                 # exact magnitude ties
            c[7::131] = np.conj(c[7])       # conjugate twins: equal key
            c[11::53] = 0                   # zeros
            c[13::211] = c[13] * 1e-30      # tiny values
        parts.append(c.astype(np.complex64))
    return np.concatenate(parts)


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.9, 0.99, 1.0])
@pytest.mark.parametrize("nm", [(8, 3), (4, 2), (6, 2), (16, 9), None])
def test_injection_random_bit_exact(theta, nm):
    rng = np.random.default_rng(int(theta * 100) + (0 if nm is None else nm[0]))
    n, chunk = 300_000, 65536
    spec = _random_spectrum(rng, n, chunk)
    q = None if nm is None else F.tune_eps(-3.0 * np.abs(spec).max(), 3.0 * np.abs(spec).max(), *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=chunk)
    msg, mask = debug.encode_spectrum(spec, n, cfg)
    got = debug.message_bytes(msg)
    lat = lat_of(q)
    width = 32 if q is None else q.n_bits
    pos = 0
    gsegs = segments_valid_bytes(got, n, chunk, theta, width)
    for L, (nnz, bm, cb) in zip(O.chunk_lengths(n, chunk), gsegs):
        b = L // 2 + 1
        kept, ch = O.encode_spectrum(spec[pos:pos + b], L, theta, "count", lat)
        np.testing.assert_array_equal(mask[pos:pos + b], kept)
        assert nnz == ch.codes.size
        assert bm == O.flags_to_bytes(ch.bitmap)
        assert cb == O.codes_to_bytes(ch.codes, width)
        pos += b


def test_injection_degenerate_chunks():
    """All-equal magnitudes, all zeros and sub-2^-50 values force the exact
    fallback selection; the stable index tie-break must still hold."""
    n, chunk = 4 * 4096, 4096
    b = chunk // 2 + 1
    parts = [np.full(b, 1.5 + 0j), np.zeros(b), np.full(b, 3e-30 - 1e-30j),
             np.where(np.arange(b) % 2 == 0, 1e-20 + 0j, 0j)]
    spec = np.concatenate(parts).astype(np.complex64)
    q = F.tune_eps(-10.0, 10.0, 8, 3)
    for theta in (0.3, 0.5, 0.77):
        cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=chunk)
        _, mask = debug.encode_spectrum(spec, n, cfg)
        for i in range(4):
            kept, _ = O.encode_spectrum(spec[i * b:(i + 1) * b], chunk, theta, "count", lat_of(q))
            np.testing.assert_array_equal(mask[i * b:(i + 1) * b], kept)


# ---------------------------------------------------------------- FFTs

# tails of the benchmark configs: 40960 (5 x 2^12 mixed), 16960 (265 x 2^5 mixed),
# 46720 (365 x 2^6 mixed), 51520 / 5402 (Bluestein), plus odd and tiny chunks
@pytest.mark.parametrize("n,chunk", [(1_000_000, 65536), (65536 * 3, 65536), (40960 + 65536, 65536),
                                     (16960, 65536), (46720, 65536), (51520, 65536), (5402, 65536),
                                     (5000, 1024), (777, 64), (100, 17), (33, 16), (65537, 65536)])
def test_forward_coefficients_match_float64_rfft(n, chunk):
    rng = np.random.default_rng(n)
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), F.tune_eps(-5, 5, 8, 3), chunk_size=chunk)
    spec = debug.forward_spectrum(g, cfg)
    pos = 0
    off = 0
    for L in O.chunk_lengths(n, chunk):
        ref = np.fft.rfft(g[off:off + L].astype(np.float64))
        got = spec[pos:pos + ref.size]
        scale = np.sqrt(np.mean(np.abs(ref) ** 2)) + 1e-30
        err = np.abs(got.astype(np.complex128) - ref).max() / scale
        assert err <= 2e-6, (L, err)
        assert got[0].imag == 0 and (L % 2 or got[-1].imag == 0)
        pos += ref.size
        off += L


@pytest.mark.parametrize("n,chunk", [(1_000_000, 65536), (40960 + 65536, 65536), (46720, 65536), (51520, 65536),
                                     (5000, 1024), (777, 64), (101, 17)])
def test_inverse_matches_float64_irfft(n, chunk):
    rng = np.random.default_rng(n + 1)
    bins = [L // 2 + 1 for L in O.chunk_lengths(n, chunk)]
    spec = np.concatenate([(rng.standard_normal(b) + 1j * rng.standard_normal(b)) for b in bins]).astype(np.complex64)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), None, chunk_size=chunk)
    out = debug.inverse_spectrum(spec, n, cfg)
    pos = off = 0
    for L, b in zip(O.chunk_lengths(n, chunk), bins):
        ref = np.fft.irfft(spec[pos:pos + b].astype(np.complex128), n=L)   # ignores Im of DC/Nyquist too
        assert rel_l2(out[off:off + L], ref) <= 1e-6, L
        pos += b
        off += L


# ---------------------------------------------------------------- decode

@pytest.mark.parametrize("theta,nm", [(0.9, (8, 3)), (0.0, None), (0.5, (6, 2)), (0.99, (16, 9))])
def test_decode_matches_oracle_on_same_message(theta, nm):
    rng = np.random.default_rng(7)
    n, chunk = 200_000, 65536
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    q = None if nm is None else F.calibrate([g], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=chunk)
    msg = F.compress(g, cfg)
    wire = F.serialize(msg)
    ref = O.decompress(O.from_wire(wire))
    got = F.decompress(msg)
    assert got.dtype == np.float64
    assert rel_l2(got, ref) <= 1e-5


def test_compress_matches_oracle_given_gpu_coefficients():
    """Full K1->K3: the GPU message equals the oracle's message built from
    the GPU's own coefficients (bit-exact), and those coefficients match the
    float64 rfft (test above)."""
    rng = np.random.default_rng(8)
    n, chunk = 1_000_000, 65536
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    q = F.calibrate([g], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=chunk)
    spec = debug.forward_spectrum(g, cfg)
    msg = F.compress(g, cfg)
    got = segments_valid_bytes(debug.message_bytes(msg), n, chunk, 0.9, 8)
    pos = 0
    for L, (nnz, bm, cb) in zip(O.chunk_lengths(n, chunk), got):
        b = L // 2 + 1
        _, ch = O.encode_spectrum(spec[pos:pos + b], L, 0.9, "count", lat_of(q))
        assert (nnz, bm, cb) == (ch.codes.size, O.flags_to_bytes(ch.bitmap), O.codes_to_bytes(ch.codes, 8))
        pos += b


def _flip_account(gpu_msg, ref_msg, n, chunk):
    """Kept-set flips (bitmap slots that differ) and code differences on the
    common slots between the GPU's message and the reference's, plus the
    bins where they sit, chunk by chunk."""
    flips = codes = 0
    bins_hit = []
    for c, (L, a, b) in enumerate(zip(O.chunk_lengths(n, chunk), gpu_msg.chunks, ref_msg.chunks)):
        da = np.zeros(a.bitmap.size, dtype=np.int64)
        db = np.zeros(b.bitmap.size, dtype=np.int64)
        da[a.bitmap] = a.codes
        db[b.bitmap] = b.codes
        flips += int(np.count_nonzero(a.bitmap != b.bitmap))
        codes += int(np.count_nonzero((da != db) & a.bitmap & b.bitmap))
        bins_hit.append(np.unique(np.nonzero(da != db)[0] // 2))
    return flips, codes, bins_hit


def _explained_by_flips(got_ref_decode, ref_out, bins_hit, n, chunk, tol=1e-9):
    """The end-to-end difference between the reference's output and the
    float64 decode of the GPU's message lives only in the bins where the two
    messages differ (fp32-vs-f64 FFT moved a coefficient across a selection
    or lattice boundary): zero those bins and the rest agrees to `tol`."""
    off = 0
    for L, hit in zip(O.chunk_lengths(n, chunk), bins_hit):
        d = np.fft.rfft(got_ref_decode[off:off + L] - ref_out[off:off + L])
        d[hit] = 0
        scale = max(np.linalg.norm(np.fft.rfft(ref_out[off:off + L])), 1e-300)
        if np.linalg.norm(d) / scale > tol:
            return False
        off += L
    return True


def test_end_to_end_against_reference_vectors(golden):
    """Reference outputs (decompress(compress(g)) of the reference itself):
    rel-L2 <= 1e-5 whenever the GPU's message equals the
    reference's; kept-set flips and code differences are reported, and where
    they occur the remaining difference must sit in exactly those bins."""
    meta, arr = golden
    report = []
    for rec in meta["e2e"]:
        g = arr[rec["key"] + "_g"]
        q = q_of(rec["quantizer"])
        cfg = F.CodecConfig(F.SparsificationSpec(rec["theta"]), q, half_precision_pass=rec["half"],
                            chunk_size=rec["chunk"])
        msg = F.compress(g, cfg)
        wire = F.serialize(msg)
        ref_out = arr[rec["key"] + "_out"]
        got = F.decompress(msg)
        gm = O.from_wire(wire)
        rm = O.compress(np.asarray(g, dtype=np.float64), rec["theta"], "count", lat_of(q), rec["half"], rec["chunk"])
        assert hashlib.sha256(O.decompress(rm).tobytes()).hexdigest() == rec["out_sha256"]   # oracle pinned
        flips, codes, hit = _flip_account(gm, rm, rec["n"], rec["chunk"])
        rel = rel_l2(got, ref_out)
        report.append((rec["key"], flips, codes, rel))
        assert rel_l2(got, O.decompress(gm)) <= 1e-5, rec["key"]      # decode parity on the same message
        if flips == 0 and codes == 0:
            assert rel <= 1e-5, rec["key"]
            assert wire == O.to_wire(rm), rec["key"]
        else:
            assert _explained_by_flips(O.decompress(gm), ref_out, hit, rec["n"], rec["chunk"]), rec["key"]
    print("e2e vs reference (key, kept flips, code diffs, rel-L2):", report)


def test_average_matches_reference_vectors(golden):
    """simulator.py:547 averages (reference-generated): rel-L2 <= 1e-5 when
    every GPU message equals the reference's, flips reported otherwise."""
    meta, arr = golden
    report = []
    for rec in meta["average"]:
        rows = arr[rec["key"] + "_rows"]
        q = q_of(rec["quantizer"])
        if rec["theta"] == 0 and q is None:
            continue           # simulator bypass (exact identity), not a codec path
        cfg = F.CodecConfig(F.SparsificationSpec(rec["theta"]), q, chunk_size=rec["chunk"])
        msgs = [F.compress(r, cfg) for r in rows]
        spec = debug.decode_spectrum(msgs, rec["weights"])
        got = debug.inverse_spectrum(spec, rows.shape[1], cfg)
        ref = O.average(rows, rec["weights"], rec["theta"], "count", lat_of(q), False, rec["chunk"])
        ref_v = arr[rec["key"] + "_vhat"]
        np.testing.assert_array_equal(ref, ref_v)
        n = rows.shape[1]
        flips = codes = 0
        gms = [O.from_wire(F.serialize(m)) for m in msgs]
        for r, gm in zip(rows, gms):
            rm = O.compress(np.asarray(r, dtype=np.float64), rec["theta"], "count", lat_of(q), False, rec["chunk"])
            f, c, _ = _flip_account(gm, rm, n, rec["chunk"])
            flips += f
            codes += c
        same_msg = sum(w * O.decompress(gm) for w, gm in zip(rec["weights"], gms))
        assert rel_l2(got, same_msg) <= 1e-5, rec["key"]
        rel = rel_l2(got, ref)
        report.append((rec["key"], flips, codes, rel))
        if flips == 0 and codes == 0:
            assert rel <= 1e-5, rec["key"]
    print("average vs reference (key, kept flips, code diffs, rel-L2):", report)


def test_decode_average_multi_message_exact_messages():
    rng = np.random.default_rng(9)
    n, chunk, W = 300_000, 65536, 5
    rows = (rng.standard_normal((W, n)) * 1e-2).astype(np.float32)
    q = F.calibrate([rows[0]], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=chunk)
    w = F.shard_weights(17, W)
    msgs = [F.compress(r, cfg) for r in rows]
    spec = debug.decode_spectrum(msgs, w)
    got = debug.inverse_spectrum(spec, n, cfg)
    ref = sum(wi * O.decompress(O.from_wire(F.serialize(m))) for wi, m in zip(w, msgs))
    assert rel_l2(got, ref) <= 1e-5


def _oracle_message_from_gpu_coeffs(g, cfg, n, chunk, theta, q):
    spec = debug.forward_spectrum(g, cfg)
    chunks, pos = [], 0
    for L in O.chunk_lengths(n, chunk):
        b = L // 2 + 1
        chunks.append(O.encode_spectrum(spec[pos:pos + b], L, theta, "count", lat_of(q))[1])
        pos += b
    return O.Message(n, chunk, float(np.float32(theta)), "count", False, lat_of(q), chunks)


@pytest.mark.parametrize("theta", [0.0, 0.5, 0.9, 0.99, 1.0])
def test_fused_degenerate_and_mixed_chunks(theta):
    """Chunks that force every branch of the fused selection: all zero,
    constant (one non-zero bin), impulses (flat spectrum: heavy ties),
    tiny values (fallback to the exact generic select), random."""
    rng = np.random.default_rng(11)
    L = 65536
    parts = [np.zeros(L), np.full(L, 0.25), np.zeros(L), (rng.standard_normal(L) * 1e-30),
             rng.standard_normal(L) * 1e-2, rng.standard_normal(L) * 1e-2]
    parts[2][::4096] = 1.0
    parts[5][::7] = 0.0
    g = np.concatenate(parts).astype(np.float32)
    q = F.calibrate([g], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
    msg = F.compress(g, cfg)
    om = _oracle_message_from_gpu_coeffs(g, cfg, g.size, L, theta, q)
    assert F.serialize(msg) == O.to_wire(om)


@pytest.mark.parametrize("theta", [0.0, 0.5, 0.9, 1.0])
def test_overlapped_average_with_degenerate_chunks(theta):
    """The averaging step launches the decode as the compress grid's
    programmatic dependent; chunks selected in place by the generic code
    (tiny values), all-zero and tie-heavy chunks, over 200 chunks (several
    waves) plus a tail, give the same bits as compress then decompress."""
    from paper_1811_08596_b200.comm import GradientAverager
    rng = np.random.default_rng(5)
    L = 65536
    g = (rng.standard_normal(200 * L + 999) * 1e-2).astype(np.float32)
    g[3 * L:4 * L] = 0.0
    g[50 * L:51 * L] = (rng.standard_normal(L) * 1e-30).astype(np.float32)
    g[120 * L:121 * L] = 0.0
    g[120 * L:121 * L:4096] = 1.0
    g[199 * L:200 * L] = (rng.standard_normal(L) * 1e-30).astype(np.float32)
    q = F.calibrate([g], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
    ref = F.codec.decompress_device(F.compress(g, cfg))
    avg = GradientAverager(g.size, cfg, [1.0])
    t = torch.from_numpy(g).cuda()
    for _ in range(3):                          # tags advance per step
        assert torch.equal(avg.step(t), ref)
    avg.check()


@pytest.mark.parametrize("W", [1, 3, 8])
def test_fused_decode_average_matches_oracle(W):
    rng = np.random.default_rng(12 + W)
    n, chunk = 65536 * 3 + 777, 65536
    rows = (rng.standard_normal((W, n)) * 1e-2).astype(np.float32)
    q = F.calibrate([rows[0]], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q, chunk_size=chunk)
    w = rng.random(W)
    msgs = [F.compress(r, cfg) for r in rows]
    got = debug.decode_average(msgs, w)
    ref = sum(wi * O.decompress(O.from_wire(F.serialize(m))) for wi, m in zip(w, msgs))
    assert rel_l2(got, ref) <= 1e-5
    # deterministic: identical bits on a second run
    np.testing.assert_array_equal(got, debug.decode_average(msgs, w))


# ---------------------------------------------------------------- wire

def test_golden_fixtures_round_trip(golden):
    meta, arr = golden
    for rec in meta["fixtures"]:
        blob = bytes.fromhex(rec["hex"])
        m = F.deserialize(blob)
        assert F.serialize(m) == blob
        assert m.original_len == arr[f"fix_{rec['name']}_input"].size
        assert [c.codes.size for c in m.chunks] == rec["kept_per_chunk"]
        ref = O.decompress(O.from_wire(blob))
        assert hashlib.sha256(ref.tobytes()).hexdigest() == rec["decompressed_sha256"]
        assert rel_l2(F.decompress(m), ref) <= 1e-6
        om = O.from_wire(blob)
        for a, b in zip(m.chunks, om.chunks):
            np.testing.assert_array_equal(a.bitmap, b.bitmap)
            np.testing.assert_array_equal(a.codes, b.codes)


def test_compress_serialize_matches_oracle_wire_from_same_message():
    rng = np.random.default_rng(10)
    g = rng.standard_normal(5000)
    q = F.calibrate([g], 6, 2)
    cfg = F.CodecConfig(F.SparsificationSpec(0.7), q, chunk_size=1024)
    m = F.compress(g, cfg)
    blob = F.serialize(m)
    om = O.from_wire(blob)
    assert O.to_wire(om) == blob
    m2 = F.deserialize(blob)
    assert m2 == m
    assert F.serialize(m2) == blob
    # a message rebuilt from host ChunkPayloads decodes identically
    m3 = F.CompressedMessage(m.original_len, m.chunk_size, m.theta, m.mode, m.half_pass, m.quantizer,
                             [F.ChunkPayload(c.bitmap.copy(), c.codes.copy()) for c in m.chunks])
    np.testing.assert_array_equal(F.decompress(m3), F.decompress(m))


def test_wire_errors():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    blob = F.serialize(F.compress(np.ones(20), F.CodecConfig(F.SparsificationSpec(0.0), q)))
    with pytest.raises(F.CorruptHeaderError):
        F.deserialize(b"NOPE" + bytes(40))
    with pytest.raises(F.TruncatedPayloadError):
        F.deserialize(blob[:-3])
    with pytest.raises(F.TruncatedPayloadError):
        F.deserialize(blob[:10])
    b = bytearray(blob)
    b[36] ^= 1
    with pytest.raises(F.BitmapMismatchError):
        F.deserialize(bytes(b))
    with pytest.raises(F.CodecFormatError):
        F.deserialize(blob + b"\x00")
    # a raised or lowered `kept` field is a bitmap mismatch in the reference
    # (codec.py:424-433), whether or not the code bytes would also overrun
    for delta in (1, -1, 3):
        b = bytearray(blob)
        kept = int.from_bytes(b[36:40], "little")
        b[36:40] = (kept + delta).to_bytes(4, "little")
        with pytest.raises(O.WireError) as ref:
            O.from_wire(bytes(b))
        assert ref.value.kind == "bitmap"
        with pytest.raises(F.BitmapMismatchError):
            F.deserialize(bytes(b))


def test_input_errors():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.5), q)
    with pytest.raises(ValueError):
        F.compress(np.array([1.0, np.nan]), cfg)
    with pytest.raises(ValueError):
        F.compress(np.array([]), cfg)
    hcfg = F.CodecConfig(F.SparsificationSpec(0.0), None, half_precision_pass=True)
    with pytest.raises(ValueError, match="binary16"):
        F.compress(np.array([1e39] * 16), hcfg)


def test_zero_gradient_and_clamp():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    m = F.compress(np.zeros(100), F.CodecConfig(F.SparsificationSpec(0.5), q))
    assert all(c.codes.size == 0 for c in m.chunks)
    np.testing.assert_array_equal(F.decompress(m), np.zeros(100))
    cfg = F.CodecConfig(F.SparsificationSpec(0.0), q, chunk_size=16)
    np.testing.assert_allclose(F.decompress(F.compress(np.full(16, -2.0), cfg)), q.actual_min / 16, rtol=1e-6)
    np.testing.assert_allclose(F.decompress(F.compress(np.full(16, 2.0), cfg)), q.actual_max / 16, rtol=1e-6)


def test_chunk_independence():
    rng = np.random.default_rng(4)
    v = rng.standard_normal(100)
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.5), q, chunk_size=32)
    whole = F.decompress(F.compress(v, cfg))
    pieces = np.concatenate([F.decompress(F.compress(v[s:s + 32], cfg)) for s in range(0, 100, 32)])
    np.testing.assert_allclose(whole, pieces, rtol=0, atol=1e-6)


# ---------------------------------------------------------------- primitives

def test_quantizer_primitives(golden):
    meta, arr = golden
    for rec in meta["encode"]:
        q = q_of(rec["q"])
        q = F.QuantizerConfig(rec["q"]["min"], rec["q"]["max"], rec["q"]["n_bits"], rec["q"]["mantissa_bits"],
                              rec["q"]["eps"], rec["q"]["pbase"], rec["q"]["pos_count"])
        np.testing.assert_array_equal(F.encode_array(q, arr[rec["key"] + "_x"]), arr[rec["key"] + "_codes"])
        np.testing.assert_array_equal(F.decode_array(q, np.arange(2 ** q.n_bits)), arr[rec["key"] + "_decoded"])
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    with pytest.raises(ValueError, match="index 1"):
        F.encode_block(q, [0.1, float("nan"), 0.3])
    with pytest.raises(ValueError):
        F.decode(q, 256)
    assert F.pack_codes(np.array([1, 2], dtype=np.uint32), 3) == bytes([0b00010001])
    for w in (2, 3, 5, 7, 8, 11, 16, 32):
        c = np.random.default_rng(w).integers(0, 2 ** w, 257, dtype=np.uint64).astype(np.uint32)
        packed = F.pack_codes(c, w)
        assert packed == O.codes_to_bytes(c, w)
        np.testing.assert_array_equal(F.unpack_codes(packed, w, c.size), c)


def test_packer_primitives():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, size=1_000_003)
    np.testing.assert_array_equal(F.prefix_sum(bits), np.cumsum(bits))
    with pytest.raises(ValueError):
        F.prefix_sum([0, 2, 1])
    p = F.pack(np.array([7.0, 0.0, 8.0, 0.0, 9.0, 0.0, 0.0]))
    np.testing.assert_array_equal(p.bitmap, [1, 0, 1, 0, 1, 0, 0])
    np.testing.assert_array_equal(p.dense, [7.0, 8.0, 9.0])
    np.testing.assert_array_equal(F.unpack(p), [7.0, 0.0, 8.0, 0.0, 9.0, 0.0, 0.0])
    bm = rng.random(1000) < 0.4
    assert F.bitmap_to_bytes(bm) == O.flags_to_bytes(bm)
    np.testing.assert_array_equal(F.bitmap_from_bytes(F.bitmap_to_bytes(bm), 1000), bm)
    assert F.bitmap_to_bytes(np.ones(3, dtype=bool)) == bytes([0b11100000])


def test_spectral_primitives(golden):
    rng = np.random.default_rng(0)
    for n in [1, 2, 3, 17, 128, 1000, 1024, 4097, 40960, 46720, 100_003]:
        v = rng.standard_normal(n)
        ref = np.fft.rfft(v)
        got = F.dft_forward(v).coefficients
        assert np.abs(got - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), n
        back = F.dft_inverse(F.Spectrum(ref, n))
        assert np.abs(back - np.fft.irfft(ref, n=n)).max() <= 1e-12 * max(1.0, np.abs(v).max()) * np.sqrt(n)
    meta, arr = golden
    for rec in meta["injection"]:
        c = arr[rec["key"] + "_coeffs"].astype(np.complex128)
        out, mask = F.truncate(F.Spectrum(c, rec["length"]), F.SparsificationSpec(rec["theta"]))
        np.testing.assert_array_equal(mask, arr[rec["key"] + "_mask"])
        np.testing.assert_array_equal(out.coefficients, np.where(mask, c, 0))
    mask = F.truncate(F.Spectrum(np.array([3.0, 1.0, 1.0, 5.0, 1.0 + 0j]), 8), F.SparsificationSpec(0.4))[1]
    np.testing.assert_array_equal(mask, [True, False, False, True, True])
    assert F.half_round_trip([2049.0])[0] == 2048.0 and F.half_round_trip([2051.0])[0] == 2052.0


def test_calibrate_matches_reference(golden):
    meta, arr = golden
    for rec in meta["calibrate"]:
        q = F.calibrate([arr[rec["key"] + "_g"]], *rec["nm"])
        r = rec["q"]
        assert (q.min, q.max, q.eps, q.pos_count) == (r["min"], r["max"], r["eps"], r["pos_count"])


# ---------------------------------------------------------------- scale

def test_resnet50_size_properties():
    """25.6M floats (BASELINE config 2): size-independent properties."""
    _size_properties(25_600_000, 0.9, (8, 3))


@pytest.mark.parametrize("n,theta,nm", [
    # BASELINE config 3: AlexNet-sized gradient, keep ratio 0.01 / 0.05 / 0.1 / 0.3
    (61_000_000, 0.99, (8, 3)), (61_000_000, 0.95, (8, 3)), (61_000_000, 0.9, (8, 3)), (61_000_000, 0.7, (8, 3)),
    # BASELINE config 4: VGG-16-sized gradient, 4/6/8/16-bit range floats
    (138_000_000, 0.9, (4, 2)), (138_000_000, 0.9, (6, 2)), (138_000_000, 0.9, (8, 3)), (138_000_000, 0.9, (16, 9)),
])
def test_large_config_properties(n, theta, nm):
    _size_properties(n, theta, nm)


def _size_properties(n, theta, nm):
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
    q = F.calibrate([g[:65536 * 4].double().cpu().numpy()], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
    m1 = F.compress(g, cfg)
    m2 = F.compress(g, cfg)
    b1, b2 = debug.message_bytes(m1), debug.message_bytes(m2)
    assert b1 == b2                                   # deterministic
    segs = segments_valid_bytes(b1, n, 65536, theta, nm[0])
    for L, (nnz, bm, _) in zip(O.chunk_lengths(n, 65536), segs):
        bins = L // 2 + 1
        assert nnz <= 2 * O.keep_bins(bins, theta)
        assert int.from_bytes(bm, "big").bit_count() == nnz
    out1 = F.codec.decompress_device(m1)
    out2 = F.codec.decompress_device(m2)
    assert torch.equal(out1, out2)
    # spot-check three chunks against the oracle decode of the same payloads
    host = g.double().cpu().numpy()
    spec = debug.forward_spectrum(g, cfg)
    last = len(O.chunk_lengths(n, 65536)) - 1
    for c in (0, last // 2, last):
        L = O.chunk_lengths(n, 65536)[c]
        off = c * 65536
        b0 = c * 32769
        _, ch = O.encode_spectrum(spec[b0:b0 + L // 2 + 1], L, theta, "count", lat_of(q))
        ref = O.decompress(O.Message(L, 65536, theta, "count", False, lat_of(q), [ch]))
        assert rel_l2(out1[off:off + L].cpu().numpy(), ref) <= 1e-5
        assert rel_l2(np.fft.rfft(host[off:off + L]), spec[b0:b0 + L // 2 + 1]) <= 1e-6


# ---------------------------------------------------------------- energy mode

@pytest.fixture(params=[False, True], ids=["window", "exact-fallback"])
def energy_path(request):
    """Energy mode decides each chunk's cut from a small exactly-sorted window
    unless numpy's sequential rounding could matter; the exact fallback (full
    in-place sort + sequential cumsum) is forced here to test it as well."""
    import ctypes
    from paper_1811_08596_b200 import _lib
    f = _lib.lib.fgc_debug_energy_force_exact
    f.argtypes = [ctypes.c_int]
    f(1 if request.param else 0)
    yield request.param
    f(0)


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.7, 0.95, 1.0])
@pytest.mark.parametrize("n,chunk,nm", [(3 * 65536 + 40960, 65536, (8, 3)), (5000, 1024, (6, 2)), (71, 16, None)])
def test_energy_mode_injection_bit_exact(theta, n, chunk, nm, energy_path):
    """spectral.py:134-139 given identical coefficients: kept mask, bitmap and
    codes equal the oracle's (numpy pairwise sum, stable order, sequential
    cumulative energy)."""
    rng = np.random.default_rng(int(theta * 100) + n)
    lens = O.chunk_lengths(n, chunk)
    spec = np.concatenate([(rng.standard_normal(L // 2 + 1) * rng.random(L // 2 + 1) ** 3
                            + 1j * rng.standard_normal(L // 2 + 1)) for L in lens]).astype(np.complex64)
    q = None if nm is None else F.tune_eps(-5.0, 5.0, *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta, "energy"), q, chunk_size=chunk)
    msg, mask = debug.encode_spectrum(spec, n, cfg)
    got = segments_valid_bytes(debug.message_bytes(msg), n, chunk, theta, 32 if q is None else nm[0],
                               mode="energy")
    pos = 0
    for L, (nnz, bm, cb) in zip(lens, got):
        b = L // 2 + 1
        kept, ch = O.encode_spectrum(spec[pos:pos + b], L, theta, "energy", lat_of(q))
        np.testing.assert_array_equal(mask[pos:pos + b], kept)
        nb = 32 if q is None else nm[0]
        assert (nnz, bm, cb) == (ch.codes.size, O.flags_to_bytes(ch.bitmap), O.codes_to_bytes(ch.codes, nb))
        pos += b


def test_energy_mode_round_trip_and_wire():
    rng = np.random.default_rng(5)
    n, chunk = 2 * 65536 + 1000, 65536
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    q = F.calibrate([g], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.8, "energy"), q, chunk_size=chunk)
    spec = debug.forward_spectrum(g, cfg)
    msg = F.compress(g, cfg)
    wire = F.serialize(msg)
    back = F.deserialize(wire)
    assert back.mode == "energy"
    # the oracle's message from the GPU's own coefficients, byte for byte
    ref = O.Message(n, chunk, float(np.float32(0.8)), "energy", False, lat_of(q), [])
    pos = 0
    for L in O.chunk_lengths(n, chunk):
        b = L // 2 + 1
        _, ch = O.encode_spectrum(spec[pos:pos + b], L, 0.8, "energy", lat_of(q))
        ref.chunks.append(ch)
        pos += b
    assert wire == O.to_wire(ref)
    got = F.decompress(msg)
    assert rel_l2(got, O.decompress(ref)) <= 1e-5


@pytest.mark.parametrize("n", [8, 9, 1000, 1001, 65536, 100_003])
@pytest.mark.parametrize("theta", [0.0, 0.5, 0.9, 1.0])
def test_truncate_energy_mode_complex128(n, theta, energy_path):
    """spectral.truncate with mode "energy" on complex128 coefficients: the
    GPU drop set equals the oracle's (Parseval weights by n's parity)."""
    rng = np.random.default_rng(n)
    b = n // 2 + 1
    c = rng.standard_normal(b) + 1j * rng.standard_normal(b)
    c[rng.integers(0, b, size=max(1, b // 10))] = 0.25 + 0.5j         # ties
    out, mask = F.truncate(F.Spectrum(c, n), F.SparsificationSpec(theta, "energy"))
    mag = np.abs(c)
    dropped = O.drop_set(mag, O.parseval_weights(n) * mag ** 2, theta, "energy")
    ref = np.ones(b, dtype=bool)
    ref[dropped] = False
    np.testing.assert_array_equal(mask, ref)
    np.testing.assert_array_equal(out.coefficients, np.where(mask, c, 0))


# ---------------------------------------------------------------- fused-path inputs

def test_fused_input_flags():
    """The fused load raises the reference's errors (codec.py:213-226) for
    65536-sample chunks too: non-finite input, binary16 overflow."""
    rng = np.random.default_rng(21)
    g = (rng.standard_normal(2 * 65536) * 1e-2).astype(np.float32)
    q = F.tune_eps(-200.0, 200.0, 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
    bad = g.copy()
    bad[70000] = np.nan
    with pytest.raises(ValueError):
        F.compress(bad, cfg)
    big = g.copy()
    big[123] = 1e6                                   # > binary16 max: overflows the half pass
    with pytest.raises(ValueError, match="binary16"):
        F.compress(big, F.CodecConfig(F.SparsificationSpec(0.9), q, half_precision_pass=True))


def test_fused_half_pass_and_float64_input():
    """half_precision_pass (spectral.py:189-196) and float64 gradients through
    the fused kernels: the message equals the oracle's message built from the
    GPU's own coefficients, and float64 input matches its float32 rounding."""
    rng = np.random.default_rng(22)
    n = 3 * 65536 + 1000
    g64 = rng.standard_normal(n) * 1e-2
    q = F.calibrate([g64], 8, 3)
    hcfg = F.CodecConfig(F.SparsificationSpec(0.9), q, half_precision_pass=True)
    msg = F.compress(g64, hcfg)
    om = _oracle_message_from_gpu_coeffs(g64, hcfg, n, 65536, 0.9, q)
    assert F.serialize(msg)[36:] == O.to_wire(om)[36:]    # payloads; the header carries the half flag
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
    m64 = F.compress(g64, cfg)
    m32 = F.compress(g64.astype(np.float32), cfg)
    assert F.serialize(m64) == F.serialize(m32)


# ---------------------------------------------------------------- randomized parity sweep

@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("FGC_SWEEP", "16"))))
def test_random_configs_match_oracle(seed):
    """Random lengths, chunk sizes (powers of two, odd, mixed-radix and prime
    tails), keep ratios, lattices and modes: the message built from the GPU's
    own coefficients is byte-identical to the oracle's, and decompression
    matches the oracle's to 1e-5."""
    rng = np.random.default_rng(1000 + seed)
    chunk = int(rng.choice([16, 17, 100, 1024, 4096, 5000, 65536]))
    n = int(rng.integers(1, 4)) * chunk + int(rng.integers(0, chunk))
    theta = float(rng.choice([0.0, 0.25, 0.5, 0.9, 0.97, 1.0]))
    nm = [(8, 3), (4, 2), (6, 2), (16, 9), None][int(rng.integers(0, 5))]
    mode = "energy" if rng.random() < 0.3 else "count"
    g = (rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 1)).astype(np.float32)
    q = None if nm is None else F.calibrate([g], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q, chunk_size=chunk)
    spec = debug.forward_spectrum(g, cfg)
    msg = F.compress(g, cfg)
    chunks, pos = [], 0
    for L in O.chunk_lengths(n, chunk):
        b = L // 2 + 1
        chunks.append(O.encode_spectrum(spec[pos:pos + b], L, theta, mode, lat_of(q))[1])
        pos += b
    om = O.Message(n, chunk, float(np.float32(theta)), mode, False, lat_of(q), chunks)
    assert F.serialize(msg) == O.to_wire(om), (n, chunk, theta, nm, mode)
    ref = O.decompress(om)
    got = F.decompress(msg)
    scale = max(np.abs(ref).max(), 1e-30)
    assert np.abs(got - ref).max() <= 1e-5 * scale, (n, chunk, theta, nm, mode)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("FGC_SWEEP", "16"))))
def test_random_averaging_step_matches_codec(seed):
    """The one-rank averaging step (fused decode overlapped with the fused
    compress, tail chunks on the side stream) gives the bits of compress then
    decompress, over random sizes, keep ratios, lattices, dtypes and chunk
    contents that hit every selection mode (zero, tiny, tie-heavy)."""
    from paper_1811_08596_b200.comm import GradientAverager
    rng = np.random.default_rng(5000 + seed)
    L = 65536
    nch = int(rng.integers(1, 160))
    n = nch * L + int(rng.integers(0, L)) * int(rng.integers(0, 2))
    theta = float(rng.choice([0.0, 0.5, 0.9, 0.97, 1.0]))
    nm = [(8, 3), (4, 2), (6, 2), (16, 9)][int(rng.integers(0, 4))]
    dt = np.float64 if rng.random() < 0.3 else np.float32
    g = rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 1)
    for _ in range(int(rng.integers(0, 4))):       # special chunks
        c = int(rng.integers(0, nch))
        kind = int(rng.integers(0, 3))
        if kind == 0:
            g[c * L:(c + 1) * L] = 0.0
        elif kind == 1:
            g[c * L:(c + 1) * L] *= 1e-32
        else:
            g[c * L:(c + 1) * L] = 0.0
            g[c * L:(c + 1) * L:int(rng.choice([1024, 4096, 8192]))] = 1.0
    g = g.astype(dt)
    q = F.calibrate([g], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
    ref = F.codec.decompress_device(F.compress(g, cfg))
    avg = GradientAverager(n, cfg, [1.0])
    t = torch.from_numpy(g).cuda()
    for _ in range(2):
        assert torch.equal(avg.step(t), ref), (n, theta, nm, dt)
    avg.check()


# ---------------------------------------------------------------- host-buffer step
@pytest.mark.parametrize("n,mode,dt", [(8 * 65536, "count", torch.float32), (20 * 65536 + 12345, "count", torch.float32),
                                       (3 * 65536 + 7, "count", torch.float64), (40000, "count", torch.float32),
                                       (5 * 65536 + 99, "energy", torch.float32)])
def test_step_host_matches_device_step(n, mode, dt):
    """fgc_average_host (PCIe copies overlapped with the codec in pieces)
    returns the same bits as the device step followed by a plain copy."""
    from paper_1811_08596_b200.comm import GradientAverager
    rng = np.random.default_rng(n)
    g = (rng.standard_normal(n) * 1e-2).astype(np.float64 if dt == torch.float64 else np.float32)
    q = F.calibrate([g], 8, 3)
    avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9, mode), q), [1.0])
    ref = avg.step(torch.from_numpy(g).cuda()).cpu()
    hin = torch.from_numpy(g).pin_memory()
    hout = torch.empty(n, dtype=torch.float32, pin_memory=True)
    for _ in range(3):
        hout.fill_(float("nan"))
        got = avg.step_host(hin, hout)
        assert torch.equal(got, ref)
    avg.check()
    want = O.decompress(O.from_wire(F.serialize(F.compress(g, avg.config))))
    assert rel_l2(ref.double().numpy(), want) <= 1e-5


@pytest.mark.parametrize("n,mode", [(12 * 65536 + 40960, "count"), (5 * 65536 + 99, "energy"), (40000, "count")])
def test_step_host_back_to_back(n, mode):
    """Consecutive host steps queued without waiting (wait=False) overlap:
    step e+1's host->device copy of a piece starts once step e's compress has
    read that piece, while step e's results are still copied out.  Every
    step must still see its own input and produce its own output."""
    from paper_1811_08596_b200.comm import GradientAverager
    rng = np.random.default_rng(n + 5)
    K = 5
    gs = [(rng.standard_normal(n) * 1e-2 * (1 + k)).astype(np.float32) for k in range(K)]
    q = F.calibrate([gs[-1]], 8, 3)
    avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9, mode), q), [1.0])
    refs = [avg.step(torch.from_numpy(g).cuda()).cpu() for g in gs]
    hins = [torch.from_numpy(g).pin_memory() for g in gs]
    houts = [torch.full((n,), float("nan"), dtype=torch.float32).pin_memory() for _ in gs]
    for rep in range(2):
        for k in range(K):
            avg.step_host(hins[k], houts[k], wait=False)
        torch.cuda.synchronize()
        for k in range(K):
            assert torch.equal(houts[k], refs[k]), (rep, k)
            houts[k].fill_(float("nan"))
    avg.check()


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_unaligned_views_are_realigned(dt):
    """A tensor view starting off the kernels' two-sample alignment is copied
    by the Python layer; the C ABI rejects such a pointer instead of faulting."""
    from paper_1811_08596_b200 import _lib
    n = 65536 + 333
    base = (torch.randn(n + 1, dtype=torch.float64, device="cuda") * 1e-2).to(dt)
    view = base[1:]
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), F.calibrate([view.cpu().numpy()], 8, 3))
    got = F.reconstruct(view, cfg)
    ref = F.reconstruct(view.clone(), cfg)
    np.testing.assert_array_equal(got, ref)
    plan = F.codec.get_plan(n, cfg.chunk_size, 0.9, "count", False, cfg.quantizer)
    msg = plan.new_message()
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    code = _lib.DTYPE_F64 if dt == torch.float64 else _lib.DTYPE_F32
    st = _lib.lib.fgc_compress(plan.handle, view.data_ptr(), code,
                               msg.data_ptr(), fl.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert st != 0 and "aligned" in _lib.lib.fgc_last_error().decode()


def test_h1_cabs_formula_on_this_host():
    """SURVEY 8c hazard H1 on the GPU box's own host: numpy's complex128 abs
    (the reference's selection key, spectral.py:147) equals the cabs formula
    the device key follows (fgc_device.cuh cabs_key); an SSE-only numpy
    dispatch would break parity of the reference itself."""
    rng = np.random.default_rng(11)
    re = rng.standard_normal(20000) * np.exp2(rng.integers(-40, 40, 20000))
    im = re * np.exp2(rng.integers(-30, 30, 20000)) * rng.choice([-1, 1], 20000)
    im[:100] = 0.0
    got = np.abs(re + 1j * im)
    want = np.array([O.magnitude_exact(a, b) for a, b in zip(re, im)])
    assert np.array_equal(got, want)


def test_runtime_theta_one_plan():
    """theta is a per-step argument (simulator.py:333-341, 522-528): one
    averager, sized for capacity_theta, gives at every step exactly what a
    plan built for that step's theta gives, and rejects a theta its messages
    cannot hold."""
    from paper_1811_08596_b200.comm import GradientAverager
    rng = np.random.default_rng(21)
    n = 3 * 65536 + 5402
    g = torch.from_numpy((rng.standard_normal(n) * 1e-2).astype(np.float32)).cuda()
    q = F.calibrate([g.cpu().numpy()], 8, 3)
    avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0], capacity_theta=0.5)
    for theta in (0.9, 0.99, 0.5, 0.7071067811865476, 0.999, 0.9):
        got = avg.step(g, theta=theta).double().cpu().numpy()
        avg.check()
        want = F.reconstruct(g, F.CodecConfig(F.SparsificationSpec(theta), q))
        np.testing.assert_array_equal(got, want)
    with pytest.raises(ValueError):
        avg.step(g, theta=0.4)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        avg.step(g, out=out)
    with pytest.raises(ValueError):
        avg.step(g, out=torch.empty(n - 1, device="cuda"))
    avg.close()


@pytest.mark.parametrize("n,chunk,theta,mode", [(3000, 512, 0.9, "count"), (70_001, 65536, 0.7, "count"),
                                                (5000, 1024, 0.5, "energy")])
def test_reconstruct_rows_matches_rows(n, chunk, theta, mode):
    """codec.py:292-337: the batched rows call equals reconstruct() row by
    row bit for bit (test_codec.py:138-152 asserts the same of the
    reference), and the oracle within the decode tolerance."""
    rng = np.random.default_rng(n)
    rows = rng.standard_normal((3, n)) * 1e-2
    q = F.calibrate([rows[0]], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q, chunk_size=chunk)
    got = F.reconstruct_rows(rows, cfg)
    assert got.shape == rows.shape and got.dtype == np.float64
    for i in range(rows.shape[0]):
        np.testing.assert_array_equal(got[i], F.reconstruct(rows[i], cfg))
    ref = O.reconstruct_rows(rows, theta, mode, lat_of(q), False, chunk)
    assert rel_l2(got, ref) <= 1e-5


def test_pack_unpack_dtypes():
    """packer.py:49-70 through the device scatter / gather kernels."""
    rng = np.random.default_rng(5)
    for dt in (np.float64, np.float32, np.uint32, np.int16, np.uint8):
        v = (rng.integers(0, 3, 10_001) * rng.integers(1, 100, 10_001)).astype(dt)
        p = F.pack(v)
        np.testing.assert_array_equal(p.bitmap, v != 0)
        np.testing.assert_array_equal(p.dense, v[v != 0])
        assert p.dense.dtype == v.dtype
        np.testing.assert_array_equal(F.unpack(p), v)


@pytest.mark.parametrize("n,theta,mode,nm", [(3 * 65536 + 40960, 0.9, "count", (8, 3)), (5001, 0.5, "count", (6, 2)),
                                             (70_000, 0.7, "energy", (8, 3))])
def test_spectrum_error_parseval(n, theta, mode, nm):
    """fgc_spectrum_error: the sender-side Parseval error equals the
    time-domain ||x - decompress(compress(x))||^2 and ||x||^2 (float64)."""
    from paper_1811_08596_b200 import _lib, _device as D
    rng = np.random.default_rng(n)
    g = rng.standard_normal(n) * 1e-2
    q = F.calibrate([g], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q)
    msg = F.compress(g, cfg)
    plan, dm = msg.device_message()
    spec = torch.from_numpy(debug.forward_spectrum(g, cfg).view(np.float32).reshape(-1, 2).copy()).cuda()
    en = torch.empty((plan.n_chunks, 2), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib.fgc_spectrum_error(plan.handle, spec.data_ptr(), dm.data_ptr(), en.data_ptr(), D.stream()))
    err, nrm = en.sum(dim=0).cpu().numpy()
    rec = F.decompress(msg)
    assert err == pytest.approx(float(np.sum((g - rec) ** 2)), rel=1e-5)
    assert nrm == pytest.approx(float(np.sum(g * g)), rel=1e-5)


@pytest.mark.parametrize("W", [2, 5, 8])
def test_average_precision_fp32_weights_and_accumulation(W):
    """The fused average rounds each weight to float32 and accumulates the W
    weighted spectra in float32 in worker order; the reference forms
    shard_weights @ recon in float64 (simulator.py:547).  Quantified here on
    non-dyadic weights through the averaging entry point itself: rel-L2 vs the
    float64 average of the oracle's decodes of the very same messages."""
    from paper_1811_08596_b200 import _lib, _device as D
    rng = np.random.default_rng(40 + W)
    n = 4 * 65536 + 5402
    rows = (rng.standard_normal((W, n)) * 1e-2).astype(np.float32)
    q = F.calibrate([rows[0]], 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
    w = F.shard_weights(7 * W + 3, W)                       # e.g. 4/17, 3/17, ... (not dyadic)
    msgs = [F.compress(r, cfg) for r in rows]
    plan = msgs[0].device_message()[0]
    stacked = torch.cat([m.device_message()[1] for m in msgs])
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    wt = np.ascontiguousarray(w, dtype=np.float64)
    _lib.check(_lib.lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes, wt.ctypes.data,
                                           out.data_ptr(), D.stream()))
    got = out.double().cpu().numpy()
    ref = sum(wi * O.decompress(O.from_wire(F.serialize(m))) for wi, m in zip(w, msgs))
    rel = rel_l2(got, ref)
    print(f"W={W}: fused average vs float64 average of the same messages: rel-L2 {rel:.2e}")
    assert rel <= 1e-6


def test_tail_chain_matches_kernel_chain():
    """The single-CTA tail chain (FGC_TAIL_CHAIN=1, opt-in) runs the same
    device code in the same order as the multi-kernel chain, so messages and
    averages must be bit-identical to it (Pow2 and Mixed tails, f32 / f64
    input, W = 1 / 3)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    probe = Path(__file__).resolve().parent / "_tail_chain_probe.py"
    digests = []
    for flag in ("0", "1"):
        env = dict(os.environ, FGC_TAIL_CHAIN=flag)
        r = subprocess.run([sys.executable, str(probe)], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1], digests
