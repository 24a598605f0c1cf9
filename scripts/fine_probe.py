"""Times the compress phases on the cfg2 field (CUDA events, median of 5); decode errors ignored
(diagnostic builds)."""
import json, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import paper_2401_05994_b200 as mg
from bench import multisine_torch
u = multisine_torch((513, 513, 513), "cuda").to(torch.float32)
spec = mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel)
grid = mg.make_grid(tuple(u.shape))
dst = torch.empty(u.numel() * 9 + (1 << 20), dtype=torch.uint8, device="cuda")
mg.set_profiling(True)
ts = []
for _ in range(7):
    try:
        mg.compress_to(u, dst, grid, spec)
    except mg.MgrcError:
        pass
    ts.append({k: ms for k, ms, _ in mg.last_profile()})
import os
ph = os.environ.get("PHASE", "fine")
val = sorted(t.get(ph, 0.0) for t in ts)[3]
print(json.dumps({"tag": sys.argv[1] if len(sys.argv) > 1 else "", ph + "_ms": round(val, 4)}))
