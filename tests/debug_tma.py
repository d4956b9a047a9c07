import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_2405_18966_b200 import svdsc as S
os.environ["SVDSC_OPCGS_FUSED"] = "1t"
os.environ["SVDSC_FORCE_STREAM"] = "1"
H = S.Handle()
for N, c in [(4096, 129), (4096, 200)]:
    rng = np.random.default_rng(5)
    Q = np.linalg.qr(rng.standard_normal((N, c)))[0]
    w = rng.standard_normal(N)
    ld = -(-N // 32) * 32
    Qd = torch.zeros((c + 1, ld), dtype=torch.float64, device="cuda")
    Qd[:c, :N] = torch.from_numpy(np.ascontiguousarray(Q.T)).cuda()
    wd = torch.from_numpy(w).cuda()
    for var in ("2", "0"):
        os.environ["SVDSC_STREAM_VARIANT"] = var
        wg, nrm = S.cgs2(H, Qd.t()[:N, :c], wd)
        wg = wg.cpu().numpy()
        w_or = O.cgs2(Q, w)
        nor = np.linalg.norm(w_or)
        err = np.abs(wg - w_or / nor)
        print(N, c, "variant", var, "nrm", nrm.item(), nor, "maxerr", err.max())
        # project the error onto Q columns: which columns leak?
        leak = Q.T @ (wg * nor - w_or)
        big = np.argsort(-np.abs(leak))[:8]
        print("   leak cols", big, np.abs(leak[big]))
