"""Host-buffer averaging step: back-to-back steps (wait=False, as bench.py's
e2e loop) with cross-step overlap against FGC_HOST_SERIAL=1, alternated in
one process.  argv: n steps reps"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
hin = torch.randn(n).mul_(1e-2).pin_memory()
hout = torch.empty(n, pin_memory=True)
q = F.calibrate([hin[:1 << 20].numpy()], 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
res = {"overlap": [], "serial": []}
for r in range(reps):
    for mode in ("overlap", "serial"):
        if mode == "serial":
            os.environ["FGC_HOST_SERIAL"] = "1"
        else:
            os.environ.pop("FGC_HOST_SERIAL", None)
        for _ in range(2):
            avg.step_host(hin, hout, wait=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            avg.step_host(hin, hout, wait=False)
        e1.record()
        torch.cuda.synchronize()
        res[mode].append(e0.elapsed_time(e1) / steps)
for k, v in res.items():
    print(f"{k:8s} ms/step: " + " ".join(f"{x:.3f}" for x in v) + f"   median {np.median(v):.3f}")
