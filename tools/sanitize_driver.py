"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the hot path once -- fused compress + decode (two
65536-sample chunks and a mixed-radix tail), the overlapped one-rank
averaging step (programmatic dependent decode + done tags), energy mode,
the wire format and calibrate.  Run one sanitizer tool per process."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
n = 2 * 65536 + 40960
g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
q = F.calibrate([g], 8, 3)
for theta, mode in ((0.9, "count"), (0.7, "energy")):
    cfg = F.CodecConfig(F.SparsificationSpec(theta, mode), q)
    m = F.compress(g, cfg)
    out = F.decompress(m)
    wire = F.serialize(m)
    m2 = F.deserialize(wire)
    assert F.serialize(m2) == wire
    print(mode, "round trip ok", len(wire), float(np.abs(out).max()))
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0], capacity_theta=0.5)
gt = torch.from_numpy(g).cuda()
for theta in (0.9, 0.95, 0.9):
    avg.step(gt, theta=theta)
avg.check()
h = torch.from_numpy(g).pin_memory()
avg.step_host(h)
torch.cuda.synchronize()
print("averaging ok")
