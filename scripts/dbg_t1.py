import sys; sys.path.insert(0,'/root/repo')
import numpy as np
import paper_2401_05994_b200 as mg
from oracle import binding
o=binding.get('restatement')
for shape in [(14,33,17),(13,33,17)]:
    u=o.multisine_noisy(shape,42,0.05).astype(np.float32)
    coords=[np.arange(s,dtype=np.float64)+(7 if a==0 else 0) for a,s in enumerate(shape)]
    g=mg.make_grid(shape, coords)
    b=mg.compress(u,g,mg.ErrorSpec(1e-4,mg.Norm.inf,0.0,mg.Mode.abs))
    print(shape, len(b), b==o.compress(u,1e-4,0,0.0,0,2,coords=coords), flush=True)
u=o.multisine_noisy((40,33,17),42,0.05).astype(np.float32)
print(len(mg.compress_chunked(u, mg.ErrorSpec(1e-4,mg.Norm.inf,0.0,mg.Mode.rel), mg.Codec.huffman, chunk_mem=17*33*17*4)))
