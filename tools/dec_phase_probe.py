"""Per-phase timing of the fused decode kernel (globaltimer stamps, knob 128).  argv: n W"""
import ctypes
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, _device as D
from paper_1811_08596_b200.codec import _compress_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
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
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
lib = _lib.lib
lib.fgc_debug_set_fused_knobs.argtypes = [ctypes.c_uint32]
lib.fgc_debug_fused_timestamps.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
dec = lambda: _lib.check(lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes,
                                                wt.ctypes.data, out.data_ptr(), D.stream()))
dec()
flush.fill_(1.0)
lib.fgc_debug_set_fused_knobs(128 | (int(sys.argv[3]) if len(sys.argv) > 3 else 0))
dec()
torch.cuda.synchronize()
lib.fgc_debug_set_fused_knobs(0)
ts = np.zeros(2048 * 16, dtype=np.uint64)
lib.fgc_debug_fused_timestamps(ts.ctypes.data, ts.size)
nct = min(2048, 2 * (n // 65536))
t = ts[: nct * 16].reshape(nct, 16).astype(np.int64)
order = [(0, 7, "msg0 loads+scan"), (7, 8, "msg0-3 codes"), (8, 1, "rest msgs"), (1, 2, "cluster sync 1"),
         (2, 3, "Y gather+twiddle"), (3, 4, "cluster sync 2"), (4, 9, "Y store+sync 3"), (9, 5, "ifft pass12"),
         (5, 6, "pass3+store")]
print(f"W={W} CTA span (TS0->TS6) mean {((t[:, 6] - t[:, 0]) / 1e3).mean():.1f} us")
for a, b, nm in order:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{nm:18s} mean {d.mean():7.2f} us  p90 {np.percentile(d, 90):7.2f}")
print("kernel span us", (t[:, 6].max() - t[:, 0].min()) / 1e3)
