# GPU debugging aid (not collected by pytest): dump T per pass for the rank-3 breakdown case
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W, oracle as O
from paper_2405_18966_b200 import svdsc as S
rng = np.random.default_rng(3)
D = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 40))
v0 = rng.standard_normal(40)
A = W.dense_matrix(D)
r_or = O.svds(A, 5, v0, t=15, maxit=20)
print("oracle", r_or.status, r_or.passes, r_or.breakdowns, r_or.S)
H = S.Handle()
M = S.Matrix.from_host(H, A)
path = "gpurun_out/T_dump.bin"
if os.path.exists(path): os.remove(path)
os.environ["SVDSC_DEBUG_DUMP"] = path
for fp in range(1, r_or.passes + 1):
    try:
        r = S.svds_c(M, 5, t=15, maxit=20, v0=torch.from_numpy(v0).cuda(), fixed_passes=fp)
        print(fp, r.info, r.S.cpu().numpy())
    except Exception as e:
        print(fp, "ERR", e)
        break
T = np.fromfile(path).reshape(-1, 16, 16)
np.set_printoptions(linewidth=250, precision=3)
print(len(T), "dumps; finite:", [bool(np.isfinite(x).all()) for x in T][-10:])
np.save("gpurun_out/T_last.npy", T[-1])
print(T[-1].T)
