import sys, time, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2401_05994_b200 as mg
from paper_2401_05994_b200 import mdr, _lib
n=257
x=np.linspace(0,1,n); X,Y,Z=np.meshgrid(x,x,x,indexing='ij')
u=np.sin(6.1*X)*np.cos(4.3*Y)+0.5*np.sin(9.7*Z+X)+0.1*X*Y
import torch
du=torch.from_numpy(u).cuda()
L=_lib.lib()
for src,name in ((u,'host'),(du,'device')):
    for _ in range(2):
        mg.set_profiling(True)
        ptr, shape, keep = mdr._f64_ptr(src, "u")
        gshape, coords, ck = mdr._grid_args(mg.make_grid(shape))
        h=C.c_void_p()
        torch.cuda.synchronize(); t0=time.perf_counter()
        L.mgrc_gpu_mdr_refactor(ptr, len(gshape), gshape.ctypes.data, coords, 32, C.byref(h))
        t1=time.perf_counter()
        ph=mg.last_profile()
    print(name, 'refactor call', round((t1-t0)*1e3,2),'ms', [(k,round(ms,3)) for k,ms,_ in ph][:12])
    t0=time.perf_counter(); store=mdr.refactor(src, planes=32); t1=time.perf_counter()
    print(name, 'python refactor total', round((t1-t0)*1e3,2), 'ms')
