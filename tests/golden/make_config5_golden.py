"""Regenerate tests/golden/config5_golden.json: BASELINE.json config 5 -- a
ResNet-32-shaped (464,154-parameter) data-parallel SGD run with compressed
gradient averaging and the diminishing theta schedule theta_t =
min(0.99, sqrt(L eta_t)) (simulator.py:333-341) -- driven through the
REFERENCE simulator.run (pkg/src/fgc/simulator.py:470-601, channel "memory",
i.e. reconstruct_rows) with the duck-typed problem
paper_1811_08596_b200.simulator.ResNet32ShapeProblem (pure numpy; the
reference's own problems cannot reach this size).

    python tests/golden/make_config5_golden.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))
from make_golden import load_reference, qdict  # noqa: E402

PROBLEM = {"seed": 5}
CONFIG = {"lr": {"eta0": 0.5, "kind": "diminishing", "tau": 10.0, "power": 1.0},
          "theta": {"kind": "diminishing", "cap": 0.99}, "workers": 4, "batch_size": 16, "iterations": 24,
          "seed": 11, "channel": "memory"}
NM = (8, 3)


def main():
    ref = load_reference()
    sim, quant, codec = ref.simulator, ref.quantizer, ref.codec
    from paper_1811_08596_b200.simulator import ResNet32ShapeProblem
    problem = ResNet32ShapeProblem(**PROBLEM)
    # the range is fixed once from a full-batch gradient at x0 (TrainConfig.quantizer, simulator.py:354)
    g0 = problem.example_grads(np.arange(problem.n_examples), problem.x0).mean(axis=0)
    q = codec.calibrate([g0], *NM)
    kw = dict(CONFIG)
    kw["lr"] = sim.LrSchedule(**kw["lr"])
    kw["theta"] = sim.ThetaSchedule(**kw["theta"])
    t0 = time.time()
    tr = sim.run(problem, sim.TrainConfig(quantizer=q, **kw))
    print(f"reference run: {time.time() - t0:.1f}s, loss {tr.loss[0]:.6g} -> {tr.loss[-1]:.6g}, "
          f"theta {tr.theta[0]:.4f} -> {tr.theta[-1]:.4f}, max err_ratio {tr.err_ratio.max():.4f}")
    out = {"numpy": np.__version__, "problem": PROBLEM, "config": CONFIG, "quantizer": qdict(q),
           "loss": tr.loss.tolist(), "grad_sq_norm": tr.grad_sq_norm.tolist(), "err_ratio": tr.err_ratio.tolist(),
           "theta": tr.theta.tolist(), "eta": tr.eta.tolist(), "diverged": tr.diverged, "meta": tr.meta}
    (HERE / "config5_golden.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
