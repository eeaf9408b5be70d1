"""Deviation of the GPU simulator traces from the reference's golden traces."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_1811_08596_b200 import simulator as S
import importlib.util
_spec = importlib.util.spec_from_file_location("sim_tests", Path(__file__).resolve().parents[1] / "tests" / "test_simulator.py")
T = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(T)
CASES, build = T.CASES, T.build

for case in CASES:
    for ch in ("wire", "memory", "gpu"):
        tr = S.run(*build(case, ch))
        rl = np.abs(tr.loss - case["loss"]) / np.abs(case["loss"])
        rg = np.abs(tr.grad_sq_norm - case["grad_sq_norm"]) / np.abs(case["grad_sq_norm"])
        de = np.abs(tr.err_ratio - case["err_ratio"])
        print(f"{case['name']:22s} {ch:6s} loss_rel {rl.max():.2e} grad_rel {rg.max():.2e} err_abs {de.max():.2e} "
              f"iters {tr.iterations}/{len(case['loss'])}", flush=True)
