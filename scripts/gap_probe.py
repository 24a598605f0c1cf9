"""Host-side time of one compress / decompress call on the cfg2 field (device buffers) against the sum of
its kernel phases (CUDA events) — the difference is launch gaps, syncs and host work."""
import json, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import paper_2401_05994_b200 as mg
from bench import multisine_torch
u = multisine_torch((513, 513, 513), "cuda").to(torch.float32)
spec = mg.ErrorSpec(1e-4, mg.Norm.inf, 0.0, mg.Mode.rel)
grid = mg.make_grid(tuple(u.shape))
n = mg.compress_to(u, None, grid, spec)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
out = torch.empty_like(u)
for prof in (False, True):
    mg.set_profiling(prof)
    res = {"profiling": prof}
    for name, fn in (("compress", lambda: mg.compress_to(u, dst, grid, spec)), ("decompress", lambda: mg.decompress_into(dst, out))):
        ws = []
        for _ in range(7):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ws.append((time.perf_counter() - t0) * 1e3)
        res[name + "_wall_ms"] = round(sorted(ws)[3], 4)
        if prof:
            ph = mg.last_profile()
            res[name + "_phases_ms"] = round(sum(ms for _, ms, _ in ph), 4)
            res[name + "_phases"] = {k: round(ms, 4) for k, ms, _ in ph}
    print(json.dumps(res))
