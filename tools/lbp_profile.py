"""One first LBP pass (svdsc_op_lbp) of a BASELINE config: the solver's own
kernel sequence, including the deferred CGS2 update, small enough to run under
`ncu --set full -k regex:k_cgs2_stream2 -s <skip> -c 2` (tuning aid).

    python tools/lbp_profile.py --workload 4 --t 200
"""
import argparse
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
    ap.add_argument("--t", type=int, default=200)
    a = ap.parse_args()
    wl = W.config(a.workload)
    H = S.Handle(torch.cuda.current_stream())
    M = S.Matrix.from_host(H, wl.A)
    U, V, T, info = S.lbp(M, a.t, torch.from_numpy(wl.v0).cuda())
    torch.cuda.synchronize()
    print({"steps": info["steps"], "bytes_reorth": info["bytes_reorth"]})


if __name__ == "__main__":
    main()
