"""CPU-only checks of the C-ABI library: it loads, exports every symbol the
public header declares, and its host-side logic (quantizer configuration,
message layout, wire-header / framing validation) matches the reference's
golden vectors and the oracle.  No kernel is launched here."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
from paper_1811_08596_b200.comm import message_layout, shard_weights

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "fgc_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fgc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= set(names)


def test_tune_eps_matches_reference_vectors(golden):
    meta, _ = golden
    for rec in meta["tune_eps"]:
        lo, hi, n, m, e = rec["args"]
        if "error" in rec:
            with pytest.raises(ValueError):
                F.tune_eps(lo, hi, n, m, e)
            continue
        q = F.tune_eps(lo, hi, n, m, e)
        r = rec["q"]
        assert (q.min, q.max, q.eps, q.pbase, q.pos_count) == (r["min"], r["max"], r["eps"], r["pbase"],
                                                               r["pos_count"]), rec["args"]
        assert q.actual_min == r["actual_min"] and q.actual_max == r["actual_max"]


def test_infeasible_format_message():
    with pytest.raises(ValueError, match="no valid configuration"):
        F.tune_eps(-1.0, 1.0, 16, 1, 0.002)


def test_quantizer_validation_errors():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    for kw in ({"n_bits": 17}, {"mantissa_bits": 8}, {"min": 0.5}, {"eps": 2.0},
               {"pbase": q.pbase + 1}, {"pos_count": 0}, {"pos_count": 255}):
        args = dict(min=q.min, max=q.max, n_bits=q.n_bits, mantissa_bits=q.mantissa_bits, eps=q.eps,
                    pbase=q.pbase, pos_count=q.pos_count)
        args.update(kw)
        with pytest.raises(ValueError):
            F.QuantizerConfig(**args)
    assert F.QuantizerConfig.from_params(-1.0, 1.0, 8, 3, q.eps) == q


@pytest.mark.parametrize("n,chunk,theta,nm", [(25_600_000, 65536, 0.9, (8, 3)), (1_000_000, 65536, 0.9, (8, 3)),
                                               (138_000_000, 65536, 0.9, (4, 2)), (5000, 1024, 0.5, (6, 2)),
                                               (777, 64, 0.0, None), (17, 16, 1.0, (16, 9))])
def test_layout_matches_oracle(n, chunk, theta, nm):
    q = None if nm is None else F.tune_eps(-3.0, 3.0, *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q, chunk_size=chunk)
    nc, nbytes, offs = message_layout(n, cfg)
    layout, total = O.device_layout(n, chunk, theta, 32 if q is None else q.n_bits)
    assert nc == len(layout) and nbytes == total
    assert [int(o) for o in offs[:-1]] == [l[0] for l in layout]


def test_shard_weights():
    np.testing.assert_array_equal(shard_weights(10, 4), np.array([3, 3, 2, 2]) / 10)


def _parse(blob):
    d = _lib.CodecDesc()
    st = _lib.lib.fgc_parse_header(blob, len(blob), C.byref(d))
    return st, d


def test_wire_header_and_framing_on_fixtures(golden):
    meta, _ = golden
    for rec in meta["fixtures"]:
        blob = bytes.fromhex(rec["hex"])
        st, d = _parse(blob)
        assert st == 0
        assert d.n == len(O.from_wire(blob).chunks[0].bitmap) // 2 * 0 + O.from_wire(blob).n
        n_chunks = len(O.chunk_lengths(d.n, d.chunk_size))
        offs = np.zeros(n_chunks, dtype=np.uint64)
        nnz = np.zeros(n_chunks, dtype=np.uint32)
        nv = C.c_uint32()
        st = _lib.lib.fgc_wire_index(blob, len(blob), C.byref(d), offs.ctypes.data, nnz.ctypes.data, C.byref(nv))
        assert st == 0 and nv.value == n_chunks
        assert list(nnz) == rec["kept_per_chunk"]


def test_wire_error_taxonomy_host_side(golden):
    meta, _ = golden
    blob = bytes.fromhex(meta["fixtures"][1]["hex"])
    assert _parse(b"NOPE" + bytes(40))[0] == _lib.ERR_HEADER
    bad = bytearray(blob); bad[4] = 9
    assert _parse(bytes(bad))[0] == _lib.ERR_HEADER
    bad = bytearray(blob); bad[5] |= 0x80
    assert _parse(bytes(bad))[0] == _lib.ERR_HEADER
    assert _parse(blob[:10])[0] == _lib.ERR_TRUNCATED
    st, d = _parse(blob)
    offs = np.zeros(1, dtype=np.uint64)
    nnz = np.zeros(1, dtype=np.uint32)
    nv = C.c_uint32()
    assert _lib.lib.fgc_wire_index(blob[:-3], len(blob) - 3, C.byref(d), offs.ctypes.data, nnz.ctypes.data,
                                   C.byref(nv)) == _lib.ERR_TRUNCATED
    assert _lib.lib.fgc_wire_index(blob + b"\0", len(blob) + 1, C.byref(d), offs.ctypes.data, nnz.ctypes.data,
                                   C.byref(nv)) == _lib.ERR_FORMAT


@pytest.mark.parametrize("delta", [1, -1, 7])
def test_wire_kept_field_tampered(golden, delta):
    """Raising or lowering a chunk's `kept` field: the reference compares the
    bitmap popcount with `kept` before it looks at the code bytes
    (codec.py:424-433), so the error class is the bitmap mismatch even when
    the inflated code length also runs past the buffer."""
    meta, _ = golden
    kinds = {_lib.ERR_BITMAP: "bitmap", _lib.ERR_TRUNCATED: "truncated", _lib.ERR_FORMAT: "format"}
    for rec in meta["fixtures"]:
        blob = bytearray(bytes.fromhex(rec["hex"]))
        kept = int.from_bytes(blob[36:40], "little")
        if kept + delta < 0:
            continue
        blob[36:40] = (kept + delta).to_bytes(4, "little")
        with pytest.raises(O.WireError) as exc:
            O.from_wire(bytes(blob))
        st, d = _parse(bytes(blob))
        assert st == 0
        n_chunks = len(O.chunk_lengths(d.n, d.chunk_size))
        offs = np.zeros(n_chunks, dtype=np.uint64)
        nnz = np.zeros(n_chunks, dtype=np.uint32)
        nv = C.c_uint32()
        st = _lib.lib.fgc_wire_index(bytes(blob), len(blob), C.byref(d), offs.ctypes.data, nnz.ctypes.data,
                                     C.byref(nv))
        # The host index checks the framing and, where chunk c's codes overrun
        # the buffer, chunk c's bitmap; the popcounts of the chunks it could
        # frame are the device deserializer's (tests/test_gpu_codec.py::
        # test_wire_errors), which runs before a framing error is raised.
        if st in (_lib.ERR_TRUNCATED, _lib.ERR_BITMAP):
            assert kinds[st] == exc.value.kind, (st, exc.value.kind)
        if exc.value.kind == "bitmap" and nv.value == 0:
            assert st == _lib.ERR_BITMAP


def test_compression_ratio_paper_setting():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    cfg = F.CodecConfig(F.SparsificationSpec(0.7), q)
    assert F.compression_ratio(cfg, 1 << 16) == pytest.approx(13.3333, abs=1e-3)
    assert F.compression_ratio(cfg, 1 << 16, include_bitmap=True) == pytest.approx(9.4, abs=0.1)


def test_config_validation():
    q = F.tune_eps(-1.0, 1.0, 8, 3)
    with pytest.raises(ValueError):
        F.CodecConfig(F.SparsificationSpec(0.5), q, chunk_size=8)
    with pytest.raises(ValueError):
        F.CodecConfig(F.SparsificationSpec(0.5, "count", "time"), q)
    with pytest.raises(ValueError):
        F.SparsificationSpec(1.5)
