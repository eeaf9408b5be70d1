"""Time compress / decode_average for a few sizes (tail-chunk cost in isolation)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1811_08596_b200 as F
from paper_1811_08596_b200.comm import GradientAverager

torch.cuda.set_device(0)
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9), q)
sizes = [int(x) for x in sys.argv[1:]] or [40960, 65536, 390 * 65536, 25_600_000]
for n in sizes:
    g = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
    avg = GradientAverager(n, cfg, [1.0])
    for _ in range(3):
        avg.step(g)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(20):
        avg.step(g)
    e[1].record()
    torch.cuda.synchronize()
    st = getattr(avg, "last_stage_ms", None)
    print(f"n={n:>10d} step {e[0].elapsed_time(e[1]) / 20 * 1e3:8.1f} us", st if st else "")
