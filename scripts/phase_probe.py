"""Per-phase CUDA-event times of one compress + decompress of a cfg5 slab
(rows [0, R) of the 2049^3 multisine field, f32, INF ABS 4e-4 ~ the global REL 1e-4)."""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import torch

import paper_2401_05994_b200 as mg
from bench import multisine_rows

R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
shape = (2049, 2049, 2049)
u = multisine_rows(shape, 0, R, "cuda").to(torch.float32).contiguous()
spec = mg.ErrorSpec(4e-4, mg.Norm.inf, 0.0, mg.Mode.abs)
g = mg.make_grid(tuple(u.shape))
dst = torch.empty(u.numel() * 8, dtype=torch.uint8, device="cuda")
out = torch.empty_like(u)
for _ in range(2):
    n = mg.compress_to(u, dst, g, spec)
    mg.decompress_into(dst[:n], out)
torch.cuda.synchronize()
mg.set_profiling(True)
for name, fn in (("compress", lambda: mg.compress_to(u, dst, g, spec)), ("decompress", lambda: mg.decompress_into(dst[:n], out))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(name, f"{ms:.2f} ms {u.numel() * 4 / ms / 1e6:.1f} GB/s", [(a, round(b, 3)) for a, b, c in mg.last_profile()])
print("container", n, "ratio", u.numel() * 4 / n)
