"""Time the two products of one BASELINE config through the C ABI (tuning aid).

    python tools/probe_spmv.py [cid] [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def med(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    H = S.Handle()
    wl = W.config(cid)
    M = S.Matrix.from_host(H, wl.A)
    x_n = torch.randn(wl.A.n, device="cuda", dtype=torch.float64)
    x_m = torch.randn(wl.A.m, device="cuda", dtype=torch.float64)
    b = wl.A.bytes_one_pass()
    av = med(lambda: S.matvec(M, x_n), reps)
    at = med(lambda: S.matvec(M, x_m, trans=True), reps)
    print(f"{os.environ.get('SVDSC_LIB_VARIANT', 'libsvdsc.so')} cfg{cid}: Av {av:.1f} us ({b / av / 1e3:.0f} GB/s)  "
          f"ATu {at:.1f} us ({b / at / 1e3:.0f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
