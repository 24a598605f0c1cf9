import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2401_05994_b200 as mg
from bench import multisine_rows
shape = (2049, 2049, 2049)
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 257
u = multisine_rows(shape, 0, rows, 'cuda').to(torch.float32).contiguous()
bs = (rows, 2049, 2049)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); mg.set_stream(st.cuda_stream)
g = mg.make_grid(bs)
spec = mg.ErrorSpec(1e-4 * 4.0, mg.Norm.inf, 0.0, mg.Mode.abs)
dst = torch.empty(u.numel() * 8, dtype=torch.uint8, device='cuda')
out = torch.empty_like(u)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    mg.set_profiling(True)
    n = mg.compress_to(u, dst, g, spec, mg.Codec.huffman)
    pc = mg.last_profile()
    mg.decompress_into(dst[:n], out)
    pd = mg.last_profile()
    mg.set_profiling(False)
print('rows', rows, 'container', n, 'ratio', u.numel() * 4 / n)
print('compress', [(a, round(b, 3)) for a, b, c in pc])
print('decompress', [(a, round(b, 3)) for a, b, c in pd])
