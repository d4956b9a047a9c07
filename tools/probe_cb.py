"""Column-blocked SpMV timing probe: back-to-back launches of one product."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402

H = S.Handle()
wl = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
M = S.Matrix.from_host(H, wl.A)
x = torch.randn(wl.A.n, device="cuda", dtype=torch.float64)
for reps in (1, 10):
    S.matvec(M, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        S.matvec(M, x)
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('SVDSC_LIB_VARIANT', 'libsvdsc.so')} reps {reps}: {e0.elapsed_time(e1) * 1e3 / reps:.1f} us per A v")
