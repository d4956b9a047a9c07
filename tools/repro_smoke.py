"""Repro of __graft_entry__.smoke()'s solve with a bitwise fingerprint.

Prints one line: sigma error vs the oracle and a hash of S/U/V, so runs under
ncu / compute-sanitizer / env perturbations can be compared bit for bit.
    python tools/repro_smoke.py [--scale 2] [--no-oracle]
"""
import argparse
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18966_b200 import svdsc as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--passes", type=int, default=9)
    ap.add_argument("--tag", default="")
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = W.config(a.config, scale=a.scale)
    H = S.Handle()
    M = S.Matrix.from_host(H, wl.A)
    r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit,
                 v0=torch.from_numpy(wl.v0).cuda(), fixed_passes=a.passes)
    torch.cuda.synchronize()
    s = r.S.cpu().numpy()
    h = hashlib.sha256()
    for x in (r.S, r.U, r.V):
        h.update(x.contiguous().cpu().numpy().tobytes())
    ref = os.path.join(ROOT, "gpurun_out", f"ref_sigma_c{a.config}_s{a.scale}_p{a.passes}.npy")
    err = float("nan")
    if a.no_oracle:
        pass
    elif os.path.exists(ref):
        so = np.load(ref)
        err = float(np.abs(s - so).max() / so[0])
    else:
        import oracle as O
        r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit, fixed_passes=a.passes)
        os.makedirs(os.path.dirname(ref), exist_ok=True)
        np.save(ref, r_or.S)
        err = float(np.abs(s - r_or.S).max() / r_or.S[0])
    print(f"REPRO {a.tag} err={err:.3e} hash={h.hexdigest()[:16]} passes={r.info['passes']} "
          f"launches={r.info['launches']} breakdowns={r.info['breakdowns']}", flush=True)


if __name__ == "__main__":
    main()
