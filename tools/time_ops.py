"""Per-op device timings through the C ABI (profiling aid, not a test).

    python tools/time_ops.py [--cid 3]

Times (CUDA events, median of repeats, inputs resident) the step-level entry
points at BASELINE config shapes: A v / A^T u (svdsc_op_matvec), CGS2 at
several basis widths (svdsc_op_cgs2), the small SVD (svdsc_op_small_svd) on a
Lanczos T, and the recombination (svdsc_op_recombine).  Prints one JSON object.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def timeit(fn, reps=10):
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


def bidiag_arrow(p, rng):
    k = p // 3
    T = np.zeros((p, p))
    T[np.arange(k), np.arange(k)] = np.sort(np.exp(-np.arange(k) / 40.0))[::-1] * 3
    T[:k, k] = rng.uniform(-0.01, 0.01, k)
    d = np.exp(-np.arange(k, p) / 40.0)
    T[np.arange(k, p), np.arange(k, p)] = d
    T[np.arange(k, p - 1), np.arange(k + 1, p)] = 0.5 * d[:-1]
    return T


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cid", type=int, default=3)
    args = ap.parse_args()
    out = {}
    H = S.Handle()
    wl = W.config(args.cid)
    M = S.Matrix.from_host(H, wl.A)
    x_n = torch.randn(wl.A.n, device="cuda", dtype=torch.float64)
    x_m = torch.randn(wl.A.m, device="cuda", dtype=torch.float64)
    bA = wl.A.bytes_one_pass()
    us = timeit(lambda: S.matvec(M, x_n))
    out["Av_us"] = us
    out["Av_GBs"] = bA / us / 1e3
    us = timeit(lambda: S.matvec(M, x_m, trans=True))
    out["ATu_us"] = us
    out["ATu_GBs"] = bA / us / 1e3
    for N in sorted({wl.A.m, wl.A.n}):
        ld = -(-N // 32) * 32
        Q = torch.zeros((wl.t + 1, ld), device="cuda", dtype=torch.float64)
        Qc = torch.randn(N, wl.t + 1, device="cuda", dtype=torch.float64)
        Qc, _ = torch.linalg.qr(Qc)
        Q[:, :N] = Qc.t()
        Qm = Q.t()
        w = torch.randn(N, device="cuda", dtype=torch.float64)
        # the solver's fused CGS2 kernels (SVDSC_OPCGS_FUSED test hook): Q-resident
        # when it fits, else streaming variant 0 (TMA), 2 (register-blocked cp.async)
        os.environ["SVDSC_OPCGS_FUSED"] = "1t"
        for var in ("0", "2"):
            os.environ["SVDSC_STREAM_VARIANT"] = var
            for c in (wl.k, (wl.k + wl.t) // 2, wl.t):
                us = timeit(lambda: S.cgs2(H, Qm[:N, :c], w))
                out[f"cgs2v{var}_N{N}_c{c}_us"] = us
                out[f"cgs2v{var}_N{N}_c{c}_GBs"] = 3 * 8 * N * c / us / 1e3
        del os.environ["SVDSC_OPCGS_FUSED"]
        Wm = S.colmajor(wl.t, wl.t)
        Wm.copy_(torch.randn(wl.t, wl.t, device="cuda", dtype=torch.float64))
        us = timeit(lambda: S.recombine(H, Qm[:N, :], Wm, wl.k, out=Qm[:N, :]))
        out[f"recombine_N{N}_us"] = us
        out[f"recombine_N{N}_TFs"] = 2 * N * wl.t * wl.k / us / 1e6
        del Q, Qc, Qm
    rng = np.random.default_rng(0)
    for p in (wl.t,):
        T = bidiag_arrow(p, rng)
        Td = S.colmajor(p, p)
        Td.copy_(torch.from_numpy(np.asfortranarray(T)).cuda())
        for hmax in (None, 20, 10, 6):  # half-block width of the cluster Jacobi
            if hmax:
                os.environ["SVDSC_JACOBI_H"] = str(hmax)
            sw = []
            us = timeit(lambda: sw.append(S.small_svd(H, Td)[3]), reps=3)
            tag = f"h{hmax}" if hmax else "default"
            out[f"small_svd_p{p}_{tag}_us"] = us
            out[f"small_svd_p{p}_{tag}_sweeps"] = sw[-1]
            os.environ.pop("SVDSC_JACOBI_H", None)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
