"""Per-phase timing of the fused compress kernel (globaltimer stamps, knob 128)."""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
theta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
torch.cuda.set_device(0)
g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
F.compress(g, cfg)
_lib.lib.fgc_debug_set_fused_knobs.argtypes = [ctypes.c_uint32]
_lib.lib.fgc_debug_set_fused_knobs(128 | (int(sys.argv[3]) if len(sys.argv) > 3 else 0))
F.compress(g, cfg)
torch.cuda.synchronize()
ts = np.zeros(2048 * 16, dtype=np.uint64)
_lib.lib.fgc_debug_fused_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
_lib.lib.fgc_debug_fused_timestamps(ts.ctypes.data, ts.size)
nct = 2 * (n // 65536)
t = ts[: nct * 16].reshape(nct, 16).astype(np.int64)
order = [(0, 1, "load"), (1, 2, "pass12"), (2, 3, "pass3+r2c"), (3, 7, "hist1 local"), (7, 8, "A+bucket+hist2"),
         (8, 9, "B+bucket2+collect"), (9, 10, "C+resolve"), (10, 4, "D"), (4, 11, "emit codes"), (11, 5, "E"),
         (5, 6, "pack+write")]
dur = (t[:, 6] - t[:, 0]) / 1e3
print("CTA duration us: mean %.1f  min %.1f max %.1f" % (dur.mean(), dur.min(), dur.max()))
for a, b, nm in order:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{nm:18s} mean {d.mean():7.2f} us  p90 {np.percentile(d, 90):7.2f}  (CTA0 {d[0::2].mean():6.2f} CTA1 {d[1::2].mean():6.2f})")
t0 = t[:, 0].min()
print("kernel span us", (t[:, 6].max() - t0) / 1e3)
