"""Driver for an ncu capture of the fused decode at W messages (one warm call + one captured)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.codec import _compress_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
torch.cuda.set_device(0)
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
msgs = []
for w in range(W):
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(w)) * 1e-2
    plan, m, _ = _compress_device(g, _lib.DTYPE_F32, cfg)
    msgs.append(m)
stacked = torch.stack(msgs)
out = torch.empty(n, dtype=torch.float32, device="cuda")
wt = np.full(W, 1.0 / W)
for _ in range(2):
    _lib.check(_lib.lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes, wt.ctypes.data,
                                           out.data_ptr(), D.stream()))
torch.cuda.synchronize()
print("ok")
