import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, warnings
warnings.simplefilter("ignore")
from hmgen.build import CONFIGS, make_mesh, rwg_basis, plane_wave_dirs
from paper_2109_04129_b200 import farfield
cfg = CONFIGS["C4"]; m = make_mesh(cfg); bs = rwg_basis(m)
_, khat, _ = plane_wave_dirs(cfg)
g = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (m.nodes, m.tris, bs.tp, bs.tm, bs.vp, bs.vm)]
print([ (x.dtype, x.shape) for x in g])
X = torch.randn(360, bs.N, dtype=torch.complex128, device="cuda").T
rh = torch.from_numpy(-np.asarray(khat)).cuda()
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    F, s = farfield(*g, cfg.k, 120*np.pi, X, rh, mono=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("mono call", (t1-t0)*1e3, "ms", flush=True)
