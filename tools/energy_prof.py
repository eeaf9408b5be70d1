"""Energy-mode compress + decode of a 25.6M-float gradient (ncu launch-list driver)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1811_08596_b200 as F
g = torch.randn(25_600_000, device="cuda", generator=torch.Generator("cuda").manual_seed(0)) * 1e-2
q = F.tune_eps(-200.0, 200.0, 8, 3)
cfg = F.CodecConfig(F.SparsificationSpec(0.9, "energy"), q)
for _ in range(2):
    m = F.compress(g, cfg)
    out = F.codec.decompress_device(m)
torch.cuda.synchronize()
print("ok")
