"""Where the end-to-end (host-buffer) solve spends its time (tuning aid).

    python tools/probe_e2e.py [cid] [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    wl = W.config(cid)
    A = wl.A
    H = S.Handle()
    Ah = W.Matrix("csr", A.m, A.n, row_ptr=torch.from_numpy(A.row_ptr).pin_memory().numpy(),
                  col_idx=torch.from_numpy(A.col_idx).pin_memory().numpy(),
                  values=torch.from_numpy(A.values).pin_memory().numpy())
    v0 = torch.from_numpy(wl.v0).pin_memory().numpy()
    if os.environ.get("PROBE_DEVICE_FIRST"):  # the bench's order: device-buffer solves first
        M0 = S.Matrix.from_host(H, A)
        ws = torch.empty(S.workspace_size(M0, wl.k, t=wl.t), dtype=torch.uint8, device="cuda")
        x0 = torch.from_numpy(wl.v0).cuda()
        H.profile(True)
        S.svds_c(M0, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=x0, workspace=ws)
        H.profile(True, families=("cgs2_fused",))
        for _ in range(int(os.environ["PROBE_DEVICE_FIRST"])):
            S.svds_c(M0, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=x0, workspace=ws)
        torch.cuda.synchronize()
        H.profile(False)
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = S.svds_c_host(H, Ah, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=v0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        info = out[5]
        print(f"wall {1e3 * (t1 - t0):.1f} ms  solve(host clock) {1e3 * info['seconds_total']:.1f} ms  "
              f"passes {info['passes']} steps {info['steps']}", flush=True)
    M = S.Matrix.from_host(H, A)
    t0 = time.perf_counter()
    M2 = S.Matrix.from_host(H, A)
    torch.cuda.synchronize()
    print(f"Matrix.from_host (H2D + analysis): {1e3 * (time.perf_counter() - t0):.1f} ms")
    x = torch.from_numpy(wl.v0).cuda()
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = S.svds_c(M, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=x)
        torch.cuda.synchronize()
        print(f"device-buffer solve wall {1e3 * (time.perf_counter() - t0):.1f} ms  (host clock "
              f"{1e3 * r.info['seconds_total']:.1f} ms)", flush=True)


if __name__ == "__main__":
    main()
