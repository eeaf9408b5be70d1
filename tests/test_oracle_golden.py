"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The vectors come from the reference itself (tests/golden/make_golden.py) and
include the reference's own wire fixtures (pkg/tests/fixtures/expected.json),
so a green run here means the oracle reproduces the reference bit-for-bit.
"""

import hashlib
import json
import math

import numpy as np
import pytest

import oracle as O

REF_EXPECTED = {  # pkg/tests/fixtures/expected.json (sizes + output digests)
    "passthrough_theta0": (90, [12], "dcf38ffa89a44514f13ff093614acb36d6b4647f7360c43db91b604eccb36f22"),
    "count_n8": (66, [17], "c6ae0d25e47943c015cd32707bd4229e7342985b3c697ebf778119802829be35"),
    "energy_half_chunked": (71, [7, 7, 3], "ce3e6901c5242e79953a3d8bb39f3703f06bcd6a2eb67753e67fe8313ce35840"),
}


def lat_of(q):
    if q is None:
        return None
    return O.lattice(q["min"], q["max"], q["n_bits"], q["mantissa_bits"], q["eps"])


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_fixtures_match_reference_expected(golden):
    meta, _ = golden
    for rec in meta["fixtures"]:
        size, kept, digest = REF_EXPECTED[rec["name"]]
        assert rec["bytes"] == size
        assert rec["kept_per_chunk"] == kept
        assert rec["decompressed_sha256"] == digest


def test_oracle_reproduces_wire_fixtures(golden):
    meta, arr = golden
    for rec in meta["fixtures"]:
        v = arr[f"fix_{rec['name']}_input"]
        msg = O.compress(v, rec["theta"], rec["mode"], lat_of(rec["quantizer"]),
                         rec["half"], rec["chunk_size"])
        blob = O.to_wire(msg)
        assert blob.hex() == rec["hex"], rec["name"]
        back = O.from_wire(blob)
        assert O.to_wire(back) == blob
        assert sha(O.decompress(back)) == rec["decompressed_sha256"]


def test_tune_eps_known_answers(golden):
    meta, _ = golden
    for rec in meta["tune_eps"]:
        lo, hi, n, m, e = rec["args"]
        if "error" in rec:
            with pytest.raises(ValueError):
                O.search_eps(lo, hi, n, m, e)
            continue
        lat = O.search_eps(lo, hi, n, m, e)
        q = rec["q"]
        assert (lat.lo, lat.hi, lat.eps, lat.pbase, lat.npos) == (
            q["min"], q["max"], q["eps"], q["pbase"], q["pos_count"]), rec["args"]
        assert lat.floor == q["actual_min"] and lat.ceil == q["actual_max"]


def test_encode_decode_known_answers(golden):
    meta, arr = golden
    for rec in meta["encode"]:
        lat = lat_of(rec["q"])
        np.testing.assert_array_equal(O.quantize(lat, arr[rec["key"] + "_x"]), arr[rec["key"] + "_codes"])
        np.testing.assert_array_equal(O.dequantize(lat, np.arange(2 ** lat.n_bits)),
                                      arr[rec["key"] + "_decoded"])


def test_stage_injection_known_answers(golden):
    meta, arr = golden
    for rec in meta["injection"]:
        c = arr[rec["key"] + "_coeffs"]
        kept, ch = O.encode_spectrum(c, rec["length"], rec["theta"], "count", lat_of(rec["quantizer"]))
        width = 32 if rec["quantizer"] is None else rec["quantizer"]["n_bits"]
        np.testing.assert_array_equal(kept, arr[rec["key"] + "_mask"])
        assert ch.codes.size == rec["kept"]
        assert O.flags_to_bytes(ch.bitmap).hex() == rec["bitmap_hex"]
        assert O.codes_to_bytes(ch.codes, width).hex() == rec["codes_hex"]


def test_end_to_end_codec(golden):
    meta, arr = golden
    for rec in meta["e2e"]:
        g = arr[rec["key"] + "_g"]
        msg = O.compress(g, rec["theta"], "count", lat_of(rec["quantizer"]), rec["half"], rec["chunk"])
        blob = O.to_wire(msg)
        assert len(blob) == rec["wire_bytes"]
        assert hashlib.sha256(blob).hexdigest() == rec["wire_sha256"]
        assert sha(O.decompress(msg)) == rec["out_sha256"]


def test_average_step(golden):
    meta, arr = golden
    for rec in meta["average"]:
        rows = arr[rec["key"] + "_rows"]
        got = O.average(rows, rec["weights"], rec["theta"], "count", lat_of(rec["quantizer"]),
                        False, rec["chunk"])
        np.testing.assert_array_equal(got, arr[rec["key"] + "_vhat"])


def test_calibrate(golden):
    meta, arr = golden
    for rec in meta["calibrate"]:
        lat = O.calibrate([arr[rec["key"] + "_g"]], *rec["nm"])
        assert (lat.lo, lat.hi, lat.eps, lat.npos) == (
            rec["q"]["min"], rec["q"]["max"], rec["q"]["eps"], rec["q"]["pos_count"])


def test_numpy_cabs_is_the_fma_formula():
    """Hazard H1: the selection key is numpy's SIMD cabs,
    sqrt(fma(s/b, s/b, 1)) * b.  If this host's numpy dispatch differs, the
    oracle (and the reference) would select different bins."""
    rng = np.random.default_rng(0)
    re = rng.standard_normal(4000) * np.exp2(rng.integers(-60, 60, 4000))
    im = re * np.exp2(rng.uniform(-30, 30, 4000)) * rng.choice([-1, 1], 4000)
    re[:50] = 0.0
    im[50:100] = 0.0
    c = (re + 1j * im).astype(np.complex64).astype(np.complex128)
    got = O.magnitude(c)
    want = np.array([O.magnitude_exact(z.real, z.imag) for z in c])
    np.testing.assert_array_equal(got, want)


def test_wire_errors():
    lat = O.search_eps(-1.0, 1.0, 8, 3)
    blob = O.to_wire(O.compress(np.ones(20), 0.0, "count", lat))
    for bad, kind in ((b"NOPE" + bytes(40), "header"), (blob[:10], "truncated"),
                      (blob[:-3], "truncated"), (blob + b"\x00", "format")):
        with pytest.raises(O.WireError) as e:
            O.from_wire(bad)
        assert e.value.kind == kind
    b = bytearray(blob)
    b[36] ^= 1
    with pytest.raises(O.WireError) as e:
        O.from_wire(bytes(b))
    assert e.value.kind == "bitmap"


def test_device_layout_holds_wire_bytes():
    rng = np.random.default_rng(5)
    g = rng.standard_normal(5000)
    for theta, lat in ((0.9, O.calibrate([g], 8, 3)), (0.0, None), (0.5, O.calibrate([g], 6, 2))):
        msg = O.compress(g, theta, "count", lat, False, 1024)
        dev = O.device_segments(msg, theta)
        layout, total = O.device_layout(5000, 1024, theta, msg.width)
        assert len(dev) == total
        wire = O.to_wire(msg)[36:]
        pos = 0
        for (off, bmo, co, cap), ch in zip(layout, msg.chunks):
            nnz = int.from_bytes(dev[off:off + 4], "little")
            assert nnz == ch.codes.size
            bmb = (ch.bitmap.size + 7) // 8
            cb = (nnz * msg.width + 7) // 8
            assert wire[pos:pos + 4 + bmb + cb] == dev[off:off + 4] + dev[off + bmo:off + bmo + bmb] + dev[off + co:off + co + cb]
            pos += 4 + bmb + cb
