"""Per-kernel timing of the hot-path ops at a BASELINE config (CUDA events),
small enough to run under `ncu --set full -k regex:...`.

    python tools/profile_ops.py --workload 4 [--reps 5] [--cgs-cols 200]

Prints one JSON line: microseconds and algorithmic GB/s of A v (a5), A^T u
(a1) and the fused CGS2 half-step (a2-a4 / a6) on the U side (N = m) and the
V side (N = n) with i = --cgs-cols basis columns.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=4)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cgs-cols", type=int, default=200)
    ap.add_argument("--skip-cgs", action="store_true")
    ap.add_argument("--spmv", default=None, help="SpMV schedule (svdsc_set_policy): auto, bins, merge, seg")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    wl = W.config(a.workload, scale=a.scale)
    tgen = time.time() - t0
    H = S.Handle(torch.cuda.current_stream())
    if a.spmv:
        H.set_policy(spmv=a.spmv)
    t0 = time.time()
    M = S.Matrix.from_host(H, wl.A)
    torch.cuda.synchronize()
    tana = time.time() - t0
    m, n = wl.A.m, wl.A.n
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, device="cuda", dtype=torch.float64, generator=g)
    u = torch.randn(m, device="cuda", dtype=torch.float64, generator=g)
    out = {"tag": a.tag, "spmv": a.spmv, "workload": wl.name, "m": m, "n": n, "nnz": wl.A.nnz, "gen_s": round(tgen, 1),
           "analysis_s": round(tana, 2)}
    bA = wl.A.bytes_one_pass() if wl.A.kind == "dense" else 12 * wl.A.nnz + 4 * (m + 1)
    bAt = wl.A.bytes_one_pass() if wl.A.kind == "dense" else 12 * wl.A.nnz + 4 * (n + 1)
    us = timed(lambda: S.matvec(M, x), a.reps)
    out["Av_us"], out["Av_GBs"] = round(us, 1), round(bA / us / 1e3, 1)
    us = timed(lambda: S.matvec(M, u, trans=True), a.reps)
    out["ATu_us"], out["ATu_GBs"] = round(us, 1), round(bAt / us / 1e3, 1)
    if not a.skip_cgs:
        c = a.cgs_cols
        for side, N in (("U", m), ("V", n)):
            ld = -(-N // 32) * 32
            Qs = torch.randn(c, ld, device="cuda", dtype=torch.float64, generator=g)
            Qs[:, N:] = 0
            # orthonormal columns (reduced QR on device: a test basis, not the product path)
            q, _ = torch.linalg.qr(Qs[:, :N].t())
            Qs[:, :N] = q.t()
            del q
            Q = Qs.t()[:N, :]
            w0 = torch.randn(N, device="cuda", dtype=torch.float64, generator=g)
            us = timed(lambda: S.cgs2(H, Q, w0), a.reps)
            byt = 8 * N * (3 * c + 5)
            out[f"cgs2_{side}_us"], out[f"cgs2_{side}_GBs"] = round(us, 1), round(byt / us / 1e3, 1)
            del Qs, Q
            torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
