"""Phase times of the single-CTA tail chains (FGC_TAIL_CHAIN=1) at 25.6M floats."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os
os.environ.setdefault("FGC_TAIL_CHAIN", "1")
import numpy as np, torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
from paper_1811_08596_b200.comm import GradientAverager
n = 25_600_000
g = torch.randn(n, device="cuda") * 1e-2
q = F.tune_eps(-200., 200., 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
for _ in range(3): avg.step(g)
torch.cuda.synchronize()
ts = np.zeros(32, dtype=np.uint64)
_lib.lib.fgc_debug_tail_timestamps(ts.ctypes.data)
t = ts.astype(np.int64)
print("forward us:", [(t[i+1]-t[i])/1e3 for i in range(5)], "total", (t[5]-t[0])/1e3)
print("inverse us:", [(t[i+1]-t[i])/1e3 for i in range(10,15)], "total", (t[15]-t[10])/1e3)
print("fwd start -> inv start", (t[10]-t[0])/1e3)
