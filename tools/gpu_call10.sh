cd $GRAFT_REPO_ROOT
cp paper_2405_18966_b200/libsvdsc_gdbg.so paper_2405_18966_b200/libsvdsc.so
python - <<'PY' 2>&1 | tail -30
import sys; sys.path.insert(0, '.')
import torch, workloads as W
from paper_2405_18966_b200 import svdsc as S
wl = W.config(1)
H = S.Handle(); M = S.Matrix.from_host(H, wl.A)
def solve(): return S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=torch.from_numpy(wl.v0).cuda(), fixed_passes=4)
solve(); print("plain ok", flush=True)
H.profile(True)
try:
    solve(); print("prof ok", H.profile_read(), flush=True)
except Exception as e: print("ERR", e, flush=True)
PY
