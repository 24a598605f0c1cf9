"""Times the transfer-function decoder's phases on the cfg2 field and one cfg5 slab (CUDA events)."""
import os, subprocess, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
if len(sys.argv) > 1:
    import torch
    import numpy as np
    import paper_2401_05994_b200 as mg
    from bench import multisine_torch, multisine_rows
    if sys.argv[1] == "cfg2":
        u = multisine_torch((513, 513, 513), "cuda").to(torch.float32)
        spec = mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel)
    else:
        u = multisine_rows((2049, 2049, 2049), 0, 257, "cuda").to(torch.float32).contiguous()
        spec = mg.ErrorSpec(4.68e-4, mg.Norm.inf, 0.0, mg.Mode.abs)
    grid = mg.make_grid(tuple(u.shape))
    n = mg.compress_to(u, None, grid, spec)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    mg.compress_to(u, dst, grid, spec)
    out = torch.empty_like(u)
    mg.set_profiling(True)
    ts = []
    for _ in range(5):
        try:
            mg.decompress_into(dst, out)
        except mg.MgrcError:
            pass
        ts.append({k: round(ms, 4) for k, ms, _ in mg.last_profile() if k.startswith("huff")})
    print(json.dumps({"wl": sys.argv[1], "phases_ms": ts[2], "decode_ms": round(sum(ts[2].values()), 4)}))
else:
    for wl in ("cfg2", "cfg5slab"):
        subprocess.run([sys.executable, __file__, wl])
