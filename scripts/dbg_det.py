import sys; sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2401_05994_b200 as mg
from bench import multisine_torch
for shape, dt, tol in [((257,257,257), torch.float64, 1e-5), ((513,513,513), torch.float64, 1e-5), ((1025,1025,1025), torch.float64, 1e-5)]:
    u = multisine_torch(shape, 'cuda').to(dt)
    spec = mg.ErrorSpec(tol, mg.Norm.inf, 0.0, mg.Mode.rel)
    g = mg.make_grid(shape)
    ns = [mg.compress_to(u, None, g, spec) for _ in range(3)]
    mg.set_profiling(True)
    n = mg.compress_to(u, None, g, spec)
    print(shape, ns, n, [(a, round(b,3)) for a, b, c in mg.last_profile()], flush=True)
    mg.set_profiling(False)
    del u
    torch.cuda.empty_cache()
