"""A/B timing of kernel-schedule policies on whole solves (tuning aid).

    python tools/ab_policy.py --workload 4 --solves 2 "spmv=seg" "spmv=bins"

Each argument is a comma-separated list of svdsc_set_policy settings; prints
ms per solve, passes and the per-family breakdown of one profiled solve.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=4)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--solves", type=int, default=2)
    ap.add_argument("policies", nargs="+")
    a = ap.parse_args()
    wl = W.config(a.workload, scale=a.scale)
    for pol in a.policies:
        kw = dict(x.split("=") for x in pol.split(",") if x)
        H = S.Handle(torch.cuda.current_stream())
        H.set_policy(**kw)
        M = S.Matrix.from_host(H, wl.A)
        v0 = torch.from_numpy(wl.v0).cuda()

        def solve():
            return S.svds_c(M, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=v0)

        r = solve()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.solves):
            r = solve()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.solves
        H.profile(True)
        solve()
        prof = {k: round(v[0], 1) for k, v in H.profile_read().items() if v[1]}
        H.profile(False)
        print(json.dumps({"policy": pol, "workload": wl.name, "ms_per_solve": round(ms, 1),
                          "passes": r.info["passes"], "steps": r.info["steps"],
                          "steps_per_s": round(r.info["steps"] / ms * 1e3, 1), "sigma1": float(r.S[0]),
                          "breakdown_ms": prof}), flush=True)
        M.close()
        H.close()


if __name__ == "__main__":
    main()
