"""PCIe copy rates (H2D alone, D2H alone, both at once) for the e2e workload
size, and the host-buffer averaging step against its piece count."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager

n = 25_600_000
dev = torch.device("cuda")
hin = torch.randn(n).mul_(1e-2).pin_memory()
hout = torch.empty(n, pin_memory=True)
d1 = torch.empty(n, device=dev)
d2 = torch.empty(n, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


res = {"h2d_ms": timed(lambda: d1.copy_(hin, non_blocking=True)),
       "d2h_ms": timed(lambda: hout.copy_(d2, non_blocking=True)),
       "both_ms": timed(both)}
def copy_pipeline(P, compute=None):
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    b = [n * i // P for i in range(P + 1)]
    ev = []
    for i in range(P):
        with torch.cuda.stream(s1):
            d1[b[i]:b[i + 1]].copy_(hin[b[i]:b[i + 1]], non_blocking=True)
            e = torch.cuda.Event()
            e.record(s1)
        cur.wait_event(e)
        if compute:
            compute(b[i], b[i + 1])
        e2 = torch.cuda.Event()
        e2.record(cur)
        ev.append(e2)
    for i in range(P):
        s2.wait_event(ev[i])
        with torch.cuda.stream(s2):
            hout[b[i]:b[i + 1]].copy_(d1[b[i]:b[i + 1]], non_blocking=True)
    cur.wait_stream(s2)


for P in [8, 32]:
    res[f"copy_pipeline_P{P}_ms"] = timed(lambda: copy_pipeline(P))
    res[f"copy_pipeline_scale_P{P}_ms"] = timed(lambda: copy_pipeline(P, lambda lo, hi: d1[lo:hi].mul_(1.0)))
q = F.calibrate([hin[:1 << 20].numpy()], 8, 3)
avg = GradientAverager(n, F.CodecConfig(F.SparsificationSpec(0.9), q), [1.0])
res["device_step_ms"] = timed(lambda: avg.step(d1))
for P in [8, 12, 16, 32]:
    os.environ["FGC_HOST_NO_RAMP"] = "1"
    os.environ["FGC_HOST_PIECES"] = str(P)
    res[f"host_step_noramp_P{P}_ms"] = timed(lambda: avg.step_host(hin, hout, wait=False))
os.environ.pop("FGC_HOST_NO_RAMP")
for P in [1, 2, 4, 6, 8, 10, 12, 16, 24, 32]:
    os.environ["FGC_HOST_PIECES"] = str(P)
    res[f"host_step_P{P}_ms"] = timed(lambda: avg.step_host(hin, hout, wait=False))
print(json.dumps(res, indent=1))
