"""The codec command line (reference cli.py:87-211, 350-392; its tests
pkg/tests/test_cli.py): usage errors and the analytic ratio run on CPU; the
data subcommands run the GPU codec and are checked against the oracle and
the reference's golden .fgc fixtures."""

import json

import numpy as np
import pytest

import oracle as O
from paper_1811_08596_b200 import cli


def run(capsys, *argv):
    code = cli.run(list(argv))
    out, err = capsys.readouterr()
    summary = json.loads(out.strip().splitlines()[-1]) if out.strip() else None
    return code, summary, err


def test_tensor_file_round_trip_and_length_check(tmp_path):
    v = np.arange(5, dtype=np.float64) * 0.5
    p = tmp_path / "t.bin"
    cli.write_tensor(str(p), v)
    np.testing.assert_array_equal(cli.read_tensor(str(p)), v)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(ValueError):
        cli.read_tensor(str(p))


@pytest.mark.parametrize("argv", [[], ["compress", "--bogus"], ["explode"]])
def test_usage_errors_exit_1(capsys, argv):
    code, _, _ = run(capsys, *argv)
    assert code == 1


def test_ratio_paper_numbers(capsys):
    code, s, _ = run(capsys, "ratio", "--theta", "0.7", "--nbits", "8")
    assert code == 0
    assert s["ratio_display"] == "13.33"
    assert s["exclude_bitmap_ratio"] == pytest.approx(13.3333, abs=1e-3)
    assert s["include_bitmap_ratio"] == pytest.approx(9.4, abs=0.1)
    code, s, _ = run(capsys, "ratio", "--theta", "0", "--nbits", "32")
    assert code == 0 and s["exclude_bitmap_ratio"] == 1.0


@pytest.mark.gpu
def test_compress_decompress_files(capsys, tmp_path):
    rng = np.random.default_rng(0)
    g = rng.standard_normal(3 * 65536 + 512)
    src, msg, out = tmp_path / "g.bin", tmp_path / "g.fgc", tmp_path / "r.bin"
    cli.write_tensor(str(src), g)
    code, s, _ = run(capsys, "compress", "--input", str(src), "--out", str(msg), "--theta", "0.6")
    assert code == 0 and s["measured_ratio"] > 1.0
    assert msg.stat().st_size == s["message_bytes"]
    code, s, _ = run(capsys, "decompress", "--input", str(msg), "--out", str(out))
    assert code == 0 and s["original_len"] == g.size
    ref = O.decompress(O.from_wire(msg.read_bytes()))
    got = cli.read_tensor(str(out))
    np.testing.assert_allclose(got, ref.astype(np.float32), rtol=0, atol=1e-5 * np.abs(ref).max())


@pytest.mark.gpu
def test_decompress_reference_fixtures(capsys, tmp_path, golden):
    meta, arr = golden
    for rec in meta["fixtures"]:
        f = tmp_path / (rec["name"] + ".fgc")
        f.write_bytes(bytes.fromhex(rec["hex"]))
        out = tmp_path / (rec["name"] + ".bin")
        code, _, _ = run(capsys, "decompress", "--input", str(f), "--out", str(out))
        assert code == 0
        ref = arr[f"fix_{rec['name']}_output"]
        got = cli.read_tensor(str(out))
        assert np.abs(got - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), rec["name"]


@pytest.mark.gpu
def test_data_errors_exit_2(capsys, tmp_path):
    bad = tmp_path / "bad.fgc"
    bad.write_bytes(b"NOPE" + bytes(64))
    code, s, err = run(capsys, "decompress", "--input", str(bad), "--out", str(tmp_path / "x.bin"))
    assert code == 2 and s["status"] == "error" and "magic" in err
    code, _, _ = run(capsys, "decompress", "--input", str(tmp_path / "nope.fgc"), "--out", str(tmp_path / "x.bin"))
    assert code == 2


@pytest.mark.gpu
def test_inspect_and_quantizer_dump(capsys, tmp_path):
    src = tmp_path / "sig.bin"
    cli.write_tensor(str(src), np.ones(16))
    out = tmp_path / "spec.csv"
    code, _, _ = run(capsys, "inspect", "--input", str(src), "--spectrum", "--out", str(out))
    lines = out.read_text().splitlines()
    assert code == 0 and lines[0] == "bin,magnitude" and len(lines) == 10
    assert float(lines[1].split(",")[1]) == pytest.approx(16.0)
    q = tmp_path / "codes.csv"
    code, s, _ = run(capsys, "quantizer-dump", "--nbits", "8", "--mantissa", "3", "--out", str(q))
    lines = q.read_text().splitlines()
    assert code == 0 and lines[0] == "code,value" and len(lines) == 257 and lines[1] == "0,0.0"
    lat = O.lattice(s["min"], s["max"], 8, 3, s["eps"])
    vals = np.array([float(x.split(",")[1]) for x in lines[1:]])
    np.testing.assert_array_equal(vals, O.dequantize(lat, np.arange(256)))


# ---------------------------------------------------------------- simulate (cli.py:268-345)
import hashlib  # noqa: E402
from pathlib import Path  # noqa: E402

SIM_CLI = json.loads((Path(__file__).resolve().parent / "golden" / "sim_golden.json").read_text())["cli"]


def _simulate(capsys, tmp_path, rec):
    out = tmp_path / "trace.csv"
    code, s, _ = run(capsys, *rec["argv"], "--out", str(out))
    s.pop("out")
    return code, s, out.read_bytes()


def test_simulate_bypass_matches_reference_bytes(capsys, tmp_path):
    rec = SIM_CLI[0]                    # theta 0, passthrough: plain SGD, no codec
    code, s, csv_bytes = _simulate(capsys, tmp_path, rec)
    assert code == rec["code"] and s == rec["summary"]
    assert hashlib.sha256(csv_bytes).hexdigest() == rec["csv_sha256"]


def test_simulate_config_file_and_errors(capsys, tmp_path, monkeypatch):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"iters": 5, "theta0": 0.0, "bogus": 1}))
    code, s, _ = run(capsys, "simulate", "--config", str(cfg))
    assert code == 2 and s["status"] == "error" and "bogus" in s["error"]
    cfg.write_text(json.dumps({"iters": 5, "theta0": 0.0}))
    monkeypatch.setenv("FGC_SEED", "17")
    code, s, _ = run(capsys, "simulate", "--config", str(cfg))
    assert code == 0 and s["iterations"] == 5 and s["seed"] == 17
    code, _, _ = run(capsys, "simulate", "--channel", "pigeon")
    assert code == 1


@pytest.mark.gpu
@pytest.mark.parametrize("i", [1, 2])
def test_simulate_compressed_follows_reference(capsys, tmp_path, i):
    rec = SIM_CLI[i]
    code, s, csv_bytes = _simulate(capsys, tmp_path, rec)
    assert code == rec["code"] and s["iterations"] == rec["summary"]["iterations"]
    loss = [float(r.split(b",")[1]) for r in csv_bytes.splitlines()[1:]]
    np.testing.assert_allclose(loss, rec["loss"], rtol=1e-6, atol=0)
    assert s["final_loss"] == pytest.approx(rec["summary"]["final_loss"], rel=1e-6)
