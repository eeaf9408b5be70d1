"""Small driver for ncu captures: compress + decode of an n-float gradient."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25_600_000)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--theta", type=float, default=0.9)
ap.add_argument("--mode", default="count", choices=["count", "energy"])
a = ap.parse_args()
torch.cuda.set_device(0)
g = torch.randn(a.n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(a.theta, a.mode), q)
avg = GradientAverager(a.n, cfg, [1.0])
for _ in range(a.iters):
    avg.step(g)
torch.cuda.synchronize()
print("ok", float(avg.out[:4].sum()))
