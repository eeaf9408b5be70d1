"""Regenerate tests/golden/sim_golden.json from the REFERENCE simulator
(pkg/src/fgc/simulator.py:470-601): convergence traces of small compressed
BSP-SGD runs that tests/test_simulator.py replays through this package.

    python tests/golden/make_sim_golden.py

Each case records the problem recipe, the TrainConfig fields (quantizer as
its from_params arguments) and the reference's trace columns, meta and
histogram summaries; the bypass case (theta = 0, passthrough) also records the
sha256 of its CSV bytes, which must match bit for bit.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import load_reference, qdict  # noqa: E402

CASES = [
    # name, problem kind + kwargs, config kwargs (lr / theta as dicts), quantizer (min, max, N, m) or None
    ("quad_bypass", ("quadratic", {"seed": 1}), {"lr": {"eta0": 0.02}, "theta": {"kind": "fixed"},
                                                 "workers": 4, "batch_size": 8, "iterations": 60, "seed": 3}, None),
    ("quad_fixed_wire", ("quadratic", {"seed": 2}), {"lr": {"eta0": 0.02}, "theta": {"kind": "fixed", "theta0": 0.5},
                                                     "workers": 4, "batch_size": 8, "iterations": 60, "seed": 4},
     None),
    ("logistic_diminishing", ("logistic", {"seed": 3}),
     {"lr": {"eta0": 0.5, "kind": "diminishing", "tau": 20.0, "power": 1.0},
      "theta": {"kind": "diminishing", "cap": 0.9}, "workers": 2, "batch_size": 16, "iterations": 60, "seed": 5,
      "channel": "memory"}, (-4.0, 4.0, 8, 3)),
    ("mlp_stepwise", ("mlp", {"seed": 4}),
     {"lr": {"eta0": 0.05}, "theta": {"kind": "stepwise", "theta0": 0.5, "theta1": 0.0, "switch_at": 30},
      "workers": 4, "batch_size": 8, "iterations": 60, "seed": 6, "hist_interval": 10}, (-8.0, 8.0, 8, 3)),
    ("quad_energy_chunks", ("quadratic", {"seed": 5, "dim": 300, "feature_smoothing": 5}),
     {"lr": {"eta0": 0.002}, "theta": {"kind": "fixed", "theta0": 0.3}, "workers": 3, "batch_size": 9,
      "iterations": 40, "seed": 7, "mode": "energy", "chunk_size": 64}, None),
    ("mlp_polynomial_clip", ("mlp", {"seed": 6, "in_dim": 12, "hidden": 32}),
     {"lr": {"eta0": 0.05}, "theta": {"kind": "polynomial", "theta0": 0.8, "power": 2.0}, "workers": 2,
      "batch_size": 6, "iterations": 40, "seed": 8, "clip_c1": 0.5}, (-1.0, 1.0, 6, 2)),
    # fused 65536-sample chunk + generic tail: dim = 64 * (1100 + 2) + 1 = 70529
    ("mlp_fused_chunk", ("mlp", {"seed": 7, "in_dim": 1100, "hidden": 64}),
     {"lr": {"eta0": 0.02}, "theta": {"kind": "fixed", "theta0": 0.9}, "workers": 4, "batch_size": 8,
      "iterations": 12, "seed": 9}, (-2.0, 2.0, 8, 3)),
]


def main():
    ref = load_reference()
    sim, quant = ref.simulator, ref.quantizer
    out = {"numpy": np.__version__, "cases": []}
    for name, (kind, pkw), ckw, q in CASES:
        problem = sim.make_problem(kind, **pkw)
        kw = dict(ckw)
        kw["lr"] = sim.LrSchedule(**kw["lr"])
        kw["theta"] = sim.ThetaSchedule(**kw["theta"])
        qc = None if q is None else quant.tune_eps(q[0], q[1], q[2], q[3])
        tr = sim.run(problem, sim.TrainConfig(quantizer=qc, **kw))
        case = {"name": name, "problem": [kind, pkw], "config": ckw, "quantizer": qdict(qc),
                "loss": tr.loss.tolist(), "grad_sq_norm": tr.grad_sq_norm.tolist(),
                "err_ratio": tr.err_ratio.tolist(), "theta": tr.theta.tolist(), "eta": tr.eta.tolist(),
                "diverged": tr.diverged, "meta": tr.meta,
                "hist": [{"iteration": h.iteration, "mean": h.mean, "std": h.std, "lo": h.lo, "hi": h.hi,
                          "counts": h.counts.tolist()} for h in tr.histograms],
                "csv_sha256": hashlib.sha256(tr.to_csv_bytes()).hexdigest()}
        out["cases"].append(case)
        print(name, "final loss", tr.loss[-1], "max err_ratio", float(tr.err_ratio.max()))
    # the `simulate` subcommand (cli.py:268-345, 407-435): summary line + CSV bytes
    import contextlib
    import io
    import os
    import tempfile
    import importlib
    ref_cli = importlib.import_module("fgc_ref.cli")
    out["cli"] = []
    for argv in (["simulate", "--theta0", "0", "--iters", "50", "--workers", "2"],
                 ["simulate", "--problem", "logistic", "--nbits", "8", "--iters", "40", "--theta-schedule",
                  "diminishing", "--lr-schedule", "diminishing", "--lr-tau", "10"],
                 ["simulate", "--problem", "mlp", "--nbits", "6", "--mantissa", "2", "--iters", "30",
                  "--theta0", "0.7", "--seed", "11"]):
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "trace.csv")
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                code = ref_cli.dispatch(argv + ["--out", path])
            csv_bytes = open(path, "rb").read()
        summary = json.loads(buf.getvalue().strip().splitlines()[-1])
        summary.pop("out")
        out["cli"].append({"argv": argv, "code": code, "summary": summary,
                           "csv_sha256": hashlib.sha256(csv_bytes).hexdigest(),
                           "loss": [float(r.split(b",")[1]) for r in csv_bytes.splitlines()[1:]]})
    (HERE / "sim_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
