"""Host-buffer averaging step time for ramp / piece variants (env set per process)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager
n = 25_600_000
hin = torch.randn(n).mul_(1e-2).pin_memory(); hout = torch.empty(n, pin_memory=True)
q = F.calibrate([hin[:1 << 20].numpy()], 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
for _ in range(3): avg.step_host(hin, hout, wait=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): avg.step_host(hin, hout, wait=False)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("FGC_HOST_PIECES", "8"), os.environ.get("FGC_HOST_TAIL", "2"), round(e0.elapsed_time(e1) / 20, 3))
