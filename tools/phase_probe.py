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
torch.cuda.set_device(0)
g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
F.compress(g, cfg)
_lib.lib.fgc_debug_set_fused_knobs.argtypes = [ctypes.c_uint32]
_lib.lib.fgc_debug_set_fused_knobs(128)
F.compress(g, cfg)
torch.cuda.synchronize()
ts = np.zeros(2048 * 8, dtype=np.uint64)
_lib.lib.fgc_debug_fused_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
_lib.lib.fgc_debug_fused_timestamps(ts.ctypes.data, ts.size)
nct = 2 * (n // 65536)
t = ts[: nct * 8].reshape(nct, 8).astype(np.int64)
t0 = t[:, 0].min()
d = np.diff(t, axis=1) / 1000.0
names = ["load", "pass12", "pass3+r2c", "select", "codes", "pack+write"]
t = t[:, :7]
d = np.diff(t, axis=1) / 1000.0
dur = (t[:, 6] - t[:, 0]) / 1e3
print("CTA duration us: mean %.1f  min %.1f max %.1f" % (dur.mean(), dur.min(), dur.max()))
for i, nm in enumerate(names):
    print(f"{nm:10s} mean {d[:, i].mean():7.2f} us  p90 {np.percentile(d[:, i], 90):7.2f}")
print("kernel span us", (t[:, 6].max() - t0) / 1e3)
starts = np.sort((t[:, 0] - t0) / 1e3)
print("start times (us) at CTA 0,148,296,444,592,740:", [round(starts[i], 1) for i in (0, 148, 296, 444, 592, 740) if i < len(starts)])
