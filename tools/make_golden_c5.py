"""Write tests/golden/oracle_config5_div2000.json: the CPU ORACLE's result on
BASELINE config 5 (banded 30M x 5M, k = 200, t = 600) scaled by 1/2000
(15,000 x 2,500; same per-row band structure).  Calls only oracle/ and
workloads/ (the oracle run takes ~100 s, too slow to repeat inside the GPU
test); the GPU parity test compares against this file.

    python tools/make_golden_c5.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def main():
    wl = W.config(5, scale=2000)
    r = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    doc = {"_doc": "oracle (oracle/oracle.c) result on workloads.config(5, scale=2000); written by "
                   "tools/make_golden_c5.py (calls only oracle/ and workloads/)",
           "workload": wl.name, "m": wl.A.m, "n": wl.A.n, "nnz": int(wl.A.nnz), "k": wl.k, "t": wl.t,
           "tol": wl.tol, "maxit": wl.maxit, "passes": r.passes, "converged": bool(r.converged),
           "steps": r.steps, "S": [float(x) for x in r.S], "resid": [float(x) for x in r.resid]}
    out = os.path.join(ROOT, "tests", "golden", "oracle_config5_div2000.json")
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(out, r.passes, r.converged)


if __name__ == "__main__":
    main()
