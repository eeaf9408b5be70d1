"""BASELINE.json config 5 against the reference: a ResNet-32-shaped
(464,154-parameter) data-parallel SGD loop with compressed gradient
averaging and the diminishing theta schedule (simulator.py:333-341), run
through the reference simulator.run in the build container
(tests/golden/make_config5_golden.py, channel "memory") and replayed here on
the GPU: the "gpu" channel (one plan for the whole run, theta set every step
at run time, W messages averaged by one frequency-domain decode) and the
"memory" channel (reconstruct_rows on the device).

Tolerance: the GPU codec transforms in float32; the trajectory follows the
reference's float64 one within the stated relative bounds below (loss and
gradient norm), theta / eta are bit-identical (the schedules are host
arithmetic)."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import simulator as S

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

G = json.loads((Path(__file__).resolve().parent / "golden" / "config5_golden.json").read_text())
LOSS_RTOL = 1e-5
GRAD_RTOL = 1e-4
ERR_ATOL = 1e-4


@pytest.mark.parametrize("channel", ["gpu", "memory"])
def test_config5_resnet32_shape_follows_reference(channel):
    problem = S.ResNet32ShapeProblem(**G["problem"])
    kw = dict(G["config"])
    kw["lr"] = S.LrSchedule(**kw["lr"])
    kw["theta"] = S.ThetaSchedule(**kw["theta"])
    kw["channel"] = channel
    q = G["quantizer"]
    quant = F.QuantizerConfig.from_params(q["min"], q["max"], q["n_bits"], q["mantissa_bits"], q["eps"])
    tr = S.run(problem, S.TrainConfig(quantizer=quant, **kw))
    assert not tr.diverged and not G["diverged"]
    assert tr.theta.tolist() == G["theta"] and tr.eta.tolist() == G["eta"]
    assert len(set(G["theta"])) == len(G["theta"])          # theta moved every step: one plan served them all
    loss_rel = np.abs(tr.loss - G["loss"]) / np.abs(G["loss"])
    grad_rel = np.abs(tr.grad_sq_norm - G["grad_sq_norm"]) / np.abs(G["grad_sq_norm"])
    err_abs = np.abs(tr.err_ratio - G["err_ratio"])
    print(f"config 5 [{channel}]: max rel loss {loss_rel.max():.2e}, grad_sq {grad_rel.max():.2e}, "
          f"err_ratio abs {err_abs.max():.2e}")
    assert loss_rel.max() <= LOSS_RTOL
    assert grad_rel.max() <= GRAD_RTOL
    assert err_abs.max() <= ERR_ATOL
