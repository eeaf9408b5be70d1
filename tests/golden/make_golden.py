"""Regenerate the golden vectors under tests/golden/ from the REFERENCE.

Run in the build container (the reference is only present there):

    python tests/golden/make_golden.py

It imports the reference package ``fgc`` from ``$FGC_REF_PATH`` (default
``/root/reference/pkg/src/fgc``) under the alias ``fgc_ref`` and records its
outputs; the GPU box never reads the reference, only these committed files.

Outputs
  golden.json  -- wire fixtures (pkg/tests/fixtures/make_fixtures.py:45-63
                  replayed), tune_eps / encode / calibrate known answers,
                  stage-injection and end-to-end codec vectors (hex bytes +
                  sha256 of float64 outputs)
  golden.npz   -- the array inputs / float outputs those records refer to
"""

from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import struct
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def load_reference():
    path = Path(os.environ.get("FGC_REF_PATH", "/root/reference/pkg/src/fgc"))
    spec = importlib.util.spec_from_file_location(
        "fgc_ref", path / "__init__.py", submodule_search_locations=[str(path)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["fgc_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def qdict(q):
    if q is None:
        return None
    return {"min": q.min, "max": q.max, "n_bits": q.n_bits, "mantissa_bits": q.mantissa_bits,
            "eps": q.eps, "pbase": q.pbase, "pos_count": q.pos_count,
            "actual_min": q.actual_min, "actual_max": q.actual_max}


def main():
    ref = load_reference()
    codec, quant, spectral, packer = ref.codec, ref.quantizer, ref.spectral, ref.packer
    arrays: dict[str, np.ndarray] = {}
    out: dict = {"numpy": np.__version__}

    # 1. the reference's own wire fixtures (make_fixtures.py:45-63)
    rng = np.random.default_rng(20240817)
    fixtures = []
    v1 = rng.standard_normal(12)
    c1 = codec.CodecConfig(spectral.SparsificationSpec(0.0, "count"), None, chunk_size=16)
    v2 = np.tanh(rng.standard_normal(64))
    q2 = quant.tune_eps(-1.0, 1.0, 8, 3, 0.002)
    c2 = codec.CodecConfig(spectral.SparsificationSpec(0.7, "count"), q2)
    v3 = 0.25 * rng.standard_normal(40)
    q3 = quant.tune_eps(-2.0, 2.0, 6, 2, 0.002)
    c3 = codec.CodecConfig(spectral.SparsificationSpec(0.5, "energy"), q3,
                           half_precision_pass=True, chunk_size=16)
    for name, v, cfg in (("passthrough_theta0", v1, c1), ("count_n8", v2, c2),
                         ("energy_half_chunked", v3, c3)):
        msg = codec.compress(v, cfg)
        blob = codec.serialize(msg)
        rec = codec.decompress(msg)
        arrays[f"fix_{name}_input"] = v
        arrays[f"fix_{name}_output"] = rec
        fixtures.append({
            "name": name, "hex": blob.hex(), "bytes": len(blob),
            "theta": cfg.sparsification.theta, "mode": cfg.sparsification.mode,
            "half": cfg.half_precision_pass, "chunk_size": cfg.chunk_size,
            "quantizer": qdict(cfg.quantizer),
            "kept_per_chunk": [int(c.codes.size) for c in msg.chunks],
            "decompressed_sha256": sha(rec),
        })
    out["fixtures"] = fixtures

    # 2. tune_eps known answers (quantizer.py:154-214)
    tune = []
    trng = np.random.default_rng(1)
    cases = [(-1.0, 1.0, 8, 3, 0.002), (-2.0, 2.0, 6, 2, 0.002), (-194.7, 194.7, 8, 3, 0.002),
             (-1.0, 1.0, 16, 1, 0.002), (-1.0, 1.0, 16, 3, 0.002), (-1.0, 1.0, 16, 9, 0.002),
             (-8.0, 8.0, 8, 3, 0.002), (-0.5, 3.0, 4, 2, 0.002), (-1e-3, 1e-3, 8, 3, 0.002),
             (-1e30, 1e30, 12, 6, 0.002), (-3.0, 3.0, 10, 4, 1.0), (-3.0, 3.0, 8, 5, 1e-30)]
    for _ in range(300):
        n = int(trng.integers(2, 17))
        m = int(trng.integers(1, n))
        lo = -float(np.exp(trng.uniform(-20, 20)))
        hi = float(np.exp(trng.uniform(-20, 20))) if trng.random() < 0.3 else -lo
        cases.append((lo, hi, n, m, float(np.exp(trng.uniform(-30, 2)))))
    for lo, hi, n, m, e in cases:
        try:
            q = quant.tune_eps(lo, hi, n, m, e)
            tune.append({"args": [lo, hi, n, m, e], "q": qdict(q)})
        except ValueError as exc:
            tune.append({"args": [lo, hi, n, m, e], "error": str(exc)})
    out["tune_eps"] = tune

    # 3. encode / decode known answers for the sweep lattices
    enc = []
    erng = np.random.default_rng(2)
    for (lo, hi, n, m) in ((-1.0, 1.0, 8, 3), (-194.7, 194.7, 8, 3), (-2.0, 2.0, 6, 2),
                           (-5.0, 5.0, 4, 2), (-50.0, 50.0, 16, 9), (-0.5, 3.0, 8, 3)):
        q = quant.tune_eps(lo, hi, n, m, 0.002)
        x = np.concatenate([
            erng.standard_normal(2000) * hi,
            np.exp(erng.uniform(np.log(q.eps) - 2, np.log(hi) + 1, 2000)) * erng.choice([-1, 1], 2000),
            [0.0, -0.0, q.eps, -q.eps, q.eps * 0.49, q.max, 2 * q.max, q.min, 2 * q.min,
             q.actual_min, q.actual_max, np.inf, -np.inf, 1e-40, -1e-40]]).astype(np.float32)
        key = f"enc_{len(enc)}"
        arrays[key + "_x"] = x
        codes = quant.encode_array(q, x)
        arrays[key + "_codes"] = codes
        arrays[key + "_decoded"] = quant.decode_array(q, np.arange(2 ** n))
        enc.append({"key": key, "q": qdict(q)})
    out["encode"] = enc

    # 4. stage injection: given float32 coefficients, the reference's
    #    truncate -> interleave -> quantize -> pack -> wire bytes
    inj = []
    srng = np.random.default_rng(3)

    def add_injection(coeffs, length, theta, q):
        spec_ = spectral.SparsificationSpec(theta, "count")
        trunc, mask = spectral.truncate(spectral.Spectrum(coeffs.astype(np.complex128), length), spec_)
        codes = codec._quantize_parts(codec._interleave(trunc.coefficients), q)
        packed = packer.pack(codes)
        n_bits = 32 if q is None else q.n_bits
        key = f"inj_{len(inj)}"
        arrays[key + "_coeffs"] = coeffs.astype(np.complex64)
        arrays[key + "_mask"] = mask
        inj.append({"key": key, "length": length, "theta": theta, "quantizer": qdict(q),
                    "kept": int(packed.dense.size),
                    "bitmap_hex": packer.bitmap_to_bytes(packed.bitmap).hex(),
                    "codes_hex": quant.pack_codes(packed.dense, n_bits).hex()})

    for length in (16, 17, 64, 100, 1000, 4096):
        bins = length // 2 + 1
        g = (srng.standard_normal(length) * 1e-2).astype(np.float32)
        c = np.fft.rfft(g.astype(np.float64)).astype(np.complex64)
        qq = codec.calibrate([g], 8, 3)
        for theta in (0.0, 0.3, 0.7, 0.9, 0.99, 1.0):
            add_injection(c, length, theta, qq)
        add_injection(c, length, 0.6, None)
        for n, m in ((4, 2), (6, 2), (16, 9)):
            add_injection(c, length, 0.5, codec.calibrate([g], n, m))
        # ties: repeated magnitudes, zeros, sign/conjugate twins
        t = c.copy()
        t[1::3] = t[1]
        t[2::5] = 0
        t[3::7] = np.conj(t[3])
        add_injection(t, length, 0.5, qq)
        add_injection(np.zeros(bins, dtype=np.complex64), length, 0.5, qq)
    out["injection"] = inj

    # 5. end-to-end codec vectors (compress -> serialize, decompress)
    e2e = []
    crng = np.random.default_rng(4)
    for n, chunk, theta, nm, half in ((1000, 256, 0.9, (8, 3), False), (5000, 1024, 0.7, (4, 2), False),
                                      (777, 64, 0.5, (6, 2), True), (3000, 512, 0.0, None, False),
                                      (4096, 4096, 0.99, (16, 9), False), (300, 100, 0.4, None, True),
                                      (65536 + 1234, 65536, 0.9, (8, 3), False)):
        g = (crng.standard_normal(n) * 1e-2).astype(np.float32).astype(np.float64)
        q = None if nm is None else codec.calibrate([g], *nm)
        cfg = codec.CodecConfig(spectral.SparsificationSpec(theta, "count"), q,
                                half_precision_pass=half, chunk_size=chunk)
        msg = codec.compress(g, cfg)
        blob = codec.serialize(msg)
        rec = codec.decompress(msg)
        key = f"e2e_{len(e2e)}"
        arrays[key + "_g"] = g
        arrays[key + "_out"] = rec
        e2e.append({"key": key, "n": n, "chunk": chunk, "theta": theta, "half": half,
                    "quantizer": qdict(q), "wire_sha256": hashlib.sha256(blob).hexdigest(),
                    "wire_bytes": len(blob), "out_sha256": sha(rec)})
    out["e2e"] = e2e

    # 6. averaging step (simulator.py:520-547) on 4 workers
    avg = []
    for theta, nm in ((0.9, (8, 3)), (0.5, None), (0.0, None)):
        rows = (crng.standard_normal((4, 3000)) * 1e-2)
        sizes = np.array([len(s) for s in np.array_split(np.arange(10), 4)])
        weights = sizes / 10
        q = None if nm is None else codec.calibrate([rows[0]], *nm)
        cfg = codec.CodecConfig(spectral.SparsificationSpec(theta, "count"), q, chunk_size=1024)
        if theta > 0 or q is not None:
            rec = codec.reconstruct_rows(rows, cfg)
        else:
            rec = rows
        v_hat = weights @ rec
        key = f"avg_{len(avg)}"
        arrays[key + "_rows"] = rows
        arrays[key + "_vhat"] = v_hat
        avg.append({"key": key, "theta": theta, "quantizer": qdict(q), "weights": weights.tolist(),
                    "chunk": 1024})
    out["average"] = avg

    # 7. calibrate (codec.py:444-470)
    cal = []
    for n, nm in ((1000, (8, 3)), (4097, (4, 2)), (200, (16, 9))):
        g = crng.standard_normal(n) * 1e-2
        key = f"cal_{len(cal)}"
        arrays[key + "_g"] = g
        cal.append({"key": key, "nm": list(nm), "q": qdict(codec.calibrate([g], *nm))})
    out["calibrate"] = cal

    (HERE / "golden.json").write_text(json.dumps(out, indent=1) + "\n")
    np.savez_compressed(HERE / "golden.npz", **arrays)
    print(f"wrote {len(arrays)} arrays, {sum(a.nbytes for a in arrays.values())} bytes")


if __name__ == "__main__":
    main()
