"""Host-buffer averaging step time against its piece count (FGC_HOST_PIECES)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, numpy as np
import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager
n = 25_600_000
hin = torch.randn(n).mul_(1e-2).pin_memory(); hout = torch.empty(n, pin_memory=True)
q = F.calibrate([hin[:1 << 20].numpy()], 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
def timed(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for rep in range(2):
  for P in [6, 8, 10]:
    os.environ["FGC_HOST_PIECES"] = str(P)
    print(P, round(timed(lambda: avg.step_host(hin, hout, wait=False)), 3), flush=True)
