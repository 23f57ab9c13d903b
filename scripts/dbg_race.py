import sys, os, warnings, numpy as np
sys.path.insert(0, os.getcwd())
warnings.simplefilter("ignore")
import torch, ctypes
from hmgen.build import load_or_generate
from hmgen.synth import random_rhs
from paper_2109_04129_b200 import PsHandle, PS_OP_RT
from oracle import read_hm, compute_scaling, apply_Rt
keep = []
for name in ["T1", "C1", "T2", "C1", "C1"]:
    meta = load_or_generate(name)
    h = PsHandle(meta["hm"]); h.setup()
    H = read_hm(meta["hm"]); S = compute_scaling(H)
    B = random_rhs(h.N, 3, 0)
    Bd = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(B).T)).cuda().T
    Y = torch.empty_like(Bd)
    h.apply(PS_OP_RT, Bd, Y)
    y = Y.T.cpu().numpy().T[S.e2rwg]
    ref = apply_Rt(S, B[S.e2rwg])
    # pointers: d_op vs d_T via ps_info? print error
    print(name, "RT rel err", np.linalg.norm(y - ref) / np.linalg.norm(ref))
    keep.append(h)
