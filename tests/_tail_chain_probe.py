"""Helper for test_gpu_codec.py::test_tail_chain_matches_kernel_chain (and
tools/): prints
a digest of compress messages and averaged outputs (W = 1 and 3) for plans
with a fused class and a tail, under whatever FGC_TAIL_CHAIN the caller sets."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib, debug
from paper_1811_08596_b200.codec import _compress_device

out = hashlib.sha256()
for n, theta, nm, dt in [(3 * 65536 + 40960, 0.9, (8, 3), np.float32), (2 * 65536 + 4096, 0.5, (4, 2), np.float32),
                         (65536 + 16960, 0.97, (16, 9), np.float64), (4 * 65536 + 46720, 0.9, (8, 3), np.float32),
                         (65536 + 2, 0.0, (8, 3), np.float32)]:
    rng = np.random.default_rng(n)
    gs = [(rng.standard_normal(n) * 1e-2).astype(dt) for _ in range(3)]
    q = F.calibrate([gs[0]], *nm)
    cfg = F.CodecConfig(F.SparsificationSpec(theta), q)
    msgs = []
    for g in gs:
        plan, m, _ = _compress_device(torch.from_numpy(g).cuda(), _lib.DTYPE_F64 if dt == np.float64 else _lib.DTYPE_F32,
                                      cfg)
        msgs.append(m)
        out.update(m.cpu().numpy().tobytes())
    stacked = torch.stack(msgs)
    for W in (1, 3):
        w = np.arange(1, W + 1, dtype=np.float64)
        w /= w.sum()
        res = torch.empty(n, dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib.fgc_decode_average(plan.handle, stacked.data_ptr(), W, plan.message_bytes, w.ctypes.data,
                                               res.data_ptr(), 0))
        torch.cuda.synchronize()
        out.update(res.cpu().numpy().tobytes())
print(out.hexdigest())
