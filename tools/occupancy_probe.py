"""2-CTA clusters of the fused compress / decode resident at once (the fused grids' wave size)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch, paper_1811_08596_b200 as F
from paper_1811_08596_b200 import _lib
g = torch.randn(1000000, device="cuda")
q = F.tune_eps(-200., 200., 8, 3)
F.compress(g, F.CodecConfig(F.SparsificationSpec(0.9), q))
torch.cuda.synchronize()
print("compress clusters", _lib.lib.fgc_debug_fused_max_clusters(0), "decode clusters",
      _lib.lib.fgc_debug_fused_max_clusters(1), "SMs", torch.cuda.get_device_properties(0).multi_processor_count)
