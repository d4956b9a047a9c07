"""Kernel timeline of one solve via the CUPTI activity trace (torch.profiler):
per-kernel device time and the idle gaps between consecutive kernels, grouped
by (previous kernel -> next kernel).  Profiling aid, not a test.

    python tools/timeline.py [--workload 3] [--out gpurun_out/timeline.json]
"""
import argparse
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def short(name):
    name = name.replace("void ", "").replace("svdsc::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    args = ap.parse_args()
    wl = W.config(args.workload)
    H = S.Handle()
    M = S.Matrix.from_host(H, wl.A)
    v0 = torch.from_numpy(wl.v0).cuda()
    ws = torch.empty(S.workspace_size(M, wl.k, t=wl.t), dtype=torch.uint8, device="cuda")
    solve = lambda: S.svds_c(M, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=v0, workspace=ws)  # noqa: E731
    solve()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = solve()
        torch.cuda.synchronize()
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
            evs.append((e.time_range.start, e.time_range.end, short(e.name)))
    evs.sort()
    busy = collections.defaultdict(float)
    cnt = collections.Counter()
    gaps = collections.defaultdict(float)
    gcnt = collections.Counter()
    for i, (s, e, n) in enumerate(evs):
        busy[n] += e - s
        cnt[n] += 1
        if i:
            g = s - evs[i - 1][1]
            key = f"{evs[i - 1][2]} -> {n}"
            gaps[key] += max(g, 0)
            gcnt[key] += 1
    span = evs[-1][1] - evs[0][0]
    out = {"span_ms": span / 1e3, "kernels_ms": sum(busy.values()) / 1e3, "gaps_ms": sum(gaps.values()) / 1e3,
           "launches": len(evs), "steps": r.info["steps"],
           "busy": {k: [round(v / 1e3, 3), cnt[k], round(v / cnt[k], 2)] for k, v in
                    sorted(busy.items(), key=lambda kv: -kv[1])},
           "gaps": {k: [round(v / 1e3, 3), gcnt[k], round(v / gcnt[k], 2)] for k, v in
                    sorted(gaps.items(), key=lambda kv: -kv[1])[:15]}}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("span_ms", "kernels_ms", "gaps_ms", "launches", "steps")}))
    for k, v in list(out["busy"].items())[:8]:
        print(f"  busy {k:40s} {v}")
    for k, v in list(out["gaps"].items())[:8]:
        print(f"  gap  {k:60s} {v}")


if __name__ == "__main__":
    main()
