"""The compressed BSP-SGD simulator (reference simulator.py:470-601 and its
tests pkg/tests/test_simulator.py) replayed against the reference's own
traces (tests/golden/sim_golden.json, made by make_sim_golden.py).

CPU: problems, Lipschitz constants, schedules, random batch stream and the
bypass trace (theta = 0, passthrough: plain SGD) are bit-identical, CSV bytes
included.  GPU: the compressed runs through the "wire" / "memory" / "gpu"
channels follow the reference trajectory within the stated tolerances (the
GPU codec transforms in float32; the measured drift stays below 1.4e-7
relative over 60 iterations)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import simulator as S
CASES = json.loads((Path(__file__).resolve().parent / "golden" / "sim_golden.json").read_text())["cases"]
BY_NAME = {c["name"]: c for c in CASES}

# trajectory tolerances for the compressed (GPU codec) runs; measured on a
# B200: loss <= 2.6e-8 relative, grad_sq_norm <= 1.4e-7, err_ratio <= 6e-8
LOSS_RTOL = 1e-6
GRAD_RTOL = 1e-5
ERR_ATOL = 1e-6


def build(case, channel=None):
    kind, pkw = case["problem"]
    problem = S.make_problem(kind, **pkw)
    kw = dict(case["config"])
    kw["lr"] = S.LrSchedule(**kw["lr"])
    kw["theta"] = S.ThetaSchedule(**kw["theta"])
    if channel:
        kw["channel"] = channel
    q = case["quantizer"]
    quant = None if q is None else F.QuantizerConfig.from_params(q["min"], q["max"], q["n_bits"],
                                                                 q["mantissa_bits"], q["eps"])
    return problem, S.TrainConfig(quantizer=quant, **kw)


@pytest.mark.parametrize("name", [c["name"] for c in CASES])
def test_problem_and_schedules_match_reference(name):
    case = BY_NAME[name]
    problem, cfg = build(case)
    meta = case["meta"]
    assert problem.dim == meta["dim"] and problem.n_examples == meta["n_examples"]
    # bit-equal here; BLAS kernels on another host CPU may round the Gram matrix differently
    assert problem.lipschitz == pytest.approx(meta["lipschitz"], rel=1e-12)
    T = len(case["eta"])
    eta = [cfg.lr.rate(t) for t in range(T)]
    theta = [cfg.theta.value(t, eta[t], meta["lipschitz"], cfg.iterations) for t in range(T)]
    assert eta == case["eta"] and theta == case["theta"]
    assert problem.loss(problem.x0) == pytest.approx(case["loss"][0], rel=1e-12)    # every run starts at x0


def test_bypass_trace_bit_identical():
    case = BY_NAME["quad_bypass"]
    problem, cfg = build(case)
    tr = S.run(problem, cfg)
    assert tr.loss.tolist() == case["loss"]
    assert tr.grad_sq_norm.tolist() == case["grad_sq_norm"]
    assert tr.err_ratio.tolist() == case["err_ratio"]
    assert hashlib.sha256(tr.to_csv_bytes()).hexdigest() == case["csv_sha256"]
    m = dict(tr.meta)
    assert m == case["meta"]


def test_config_validation():
    lr, th = S.LrSchedule(0.1), S.ThetaSchedule()
    for bad in ({"workers": 0}, {"workers": 4, "batch_size": 2}, {"iterations": 0}, {"mode": "topk"},
                {"channel": "carrier-pigeon"}, {"clip_c1": 0.0}):
        with pytest.raises(ValueError):
            S.TrainConfig(lr, th, **bad)
    S.TrainConfig(lr, th, channel="gpu")
    with pytest.raises(ValueError):
        S.LrSchedule(0.0)
    with pytest.raises(ValueError):
        S.LrSchedule(0.1, "diminishing", tau=0.0)
    with pytest.raises(ValueError):
        S.ThetaSchedule("fixed", theta0=1.5)
    with pytest.raises(ValueError):
        S.ThetaSchedule("cosine")
    with pytest.raises(ValueError):
        S.make_problem("resnet")
    with pytest.raises(ValueError):
        S.MlpProblem.synthesize(hidden=65)
    p = S.make_problem("quadratic")
    with pytest.raises(ValueError):
        S.TrainConfig(S.LrSchedule(1.0), th, enforce_theorem_bounds=True).validate_theorem_bounds(p.lipschitz)
    with pytest.raises(ValueError):
        S.sub_gradient(p, p.x0, [])
    with pytest.raises(FloatingPointError):
        S.step(np.zeros(2), np.array([np.inf, 0.0]), 0.1)


def _check_trace(tr, case):
    ref_loss = np.array(case["loss"])
    assert tr.iterations == ref_loss.size and tr.diverged == case["diverged"]
    np.testing.assert_allclose(tr.theta, case["theta"], rtol=1e-12, atol=0)
    np.testing.assert_array_equal(tr.eta, case["eta"])
    np.testing.assert_allclose(tr.loss, ref_loss, rtol=LOSS_RTOL, atol=0)
    np.testing.assert_allclose(tr.grad_sq_norm, case["grad_sq_norm"], rtol=GRAD_RTOL, atol=0)
    np.testing.assert_allclose(tr.err_ratio, case["err_ratio"], rtol=0, atol=ERR_ATOL)
    for h, r in zip(tr.histograms, case["hist"]):
        assert h.iteration == r["iteration"]
        assert h.mean == pytest.approx(r["mean"], rel=1e-5, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("channel", ["wire", "memory", "gpu"])
@pytest.mark.parametrize("name", [c["name"] for c in CASES if c["name"] != "quad_bypass"])
def test_compressed_trace_follows_reference(name, channel):
    case = BY_NAME[name]
    problem, cfg = build(case, channel)
    tr = S.run(problem, cfg)
    _check_trace(tr, case)
    assert tr.meta["channel"] == channel


@pytest.mark.gpu
def test_wire_and_memory_channels_identical():
    """The reference asserts the wire and memory paths are bit-identical
    (test_codec.py:129-152); so are this package's."""
    case = BY_NAME["mlp_stepwise"]
    a = S.run(*build(case, "wire"))
    b = S.run(*build(case, "memory"))
    np.testing.assert_array_equal(a.loss, b.loss)
    np.testing.assert_array_equal(a.err_ratio, b.err_ratio)
