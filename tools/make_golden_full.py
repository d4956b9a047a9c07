"""Write full-size oracle goldens (SURVEY.md 8(c) pins for configs 3 and 4).

Calls only oracle/ and workloads/ (the GPU test compares against the files):
  tests/golden/oracle_config3.json  -- the CPU oracle's full restarted solve
      (Alg. 2) of BASELINE config 3 (200,000 x 100,000,
      10M nnz, k = 100, t = 300): sigma_1..sigma_100, Eq. (4) residuals,
      passes, steps (about 10-20 min single-threaded).
  tests/golden/oracle_config4_lbp20.json -- SURVEY 8(c) pin (ii): the first
      20 Lanczos steps (Alg. 1, full CGS2 PAPER.md:121) of
      the FULL config 4 instance (4M x 2M power law, ~150M nnz): alpha_1..21,
      beta_1..20.

    python tools/make_golden_full.py [3] [4]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def config3():
    wl = W.config(3)
    t0 = time.time()
    r = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    doc = {"_doc": "oracle (oracle/oracle.c) full solve of workloads.config(3) (BASELINE config 3); "
                   "written by tools/make_golden_full.py (calls only oracle/ and workloads/)",
           "workload": wl.name, "m": wl.A.m, "n": wl.A.n, "nnz": int(wl.A.nnz), "k": wl.k, "t": wl.t,
           "tol": wl.tol, "maxit": wl.maxit, "passes": r.passes, "converged": bool(r.converged),
           "steps": r.steps, "matvecs": r.matvecs, "oracle_seconds": round(time.time() - t0, 1),
           "S": [float(x) for x in r.S], "resid": [float(x) for x in r.resid]}
    out = os.path.join(ROOT, "tests", "golden", "oracle_config3.json")
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(out, r.passes, r.converged, doc["oracle_seconds"], flush=True)


def config4(steps=20):
    wl = W.config(4)
    t0 = time.time()
    U, V, T, info = O.lbp(wl.A, steps, wl.v0)
    alpha = [float(T[i, i]) for i in range(steps + 1)]
    beta = [float(T[i, i + 1]) for i in range(steps)]
    doc = {"_doc": "oracle (oracle/oracle.c or_lbp) first pass LBP(A, t+1) with t = %d on the full "
                   "workloads.config(4) instance (BASELINE config 4): T's diagonal alpha_1..alpha_{t+1} "
                   "and superdiagonal beta_1..beta_t; written by tools/make_golden_full.py" % steps,
           "workload": wl.name, "m": wl.A.m, "n": wl.A.n, "nnz": int(wl.A.nnz), "t": steps,
           "oracle_seconds": round(time.time() - t0, 1), "alpha": alpha, "beta": beta,
           "v_last_sample": [float(x) for x in V[:: max(1, wl.A.n // 64), steps]]}
    out = os.path.join(ROOT, "tests", "golden", "oracle_config4_lbp20.json")
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(out, doc["oracle_seconds"], flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["4", "3"]
    if "4" in which:
        config4()
    if "3" in which:
        config3()
