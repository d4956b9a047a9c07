"""The C-ABI library loads and exports every symbol include/svdsc.h declares
(no compute calls; runs without a GPU).  Also: the product package never
imports the oracle, and the host-only partitioner."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDRS = [os.path.join(ROOT, "include", f) for f in ("svdsc.h", "svdsc_paper.h")]
SO = os.path.join(ROOT, "paper_2405_18966_b200", "libsvdsc.so")


def declared():
    out = set()
    for hdr in HDRS:
        src = open(hdr).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        out |= set(re.findall(r"\b(svdsc_[a-z_0-9]+|svds_C[a-z_]*)\s*\(", src))
    return sorted(out)


@pytest.fixture(scope="module")
def so():
    from paper_2405_18966_b200 import build
    build.build()
    return SO


def test_exports_match_header(so):
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = set(re.findall(r" T (svdsc_\w+|svds_C\w*)", out))
    decl = declared()
    assert len(decl) >= 20
    missing = [d for d in decl if d not in exported]
    assert not missing, missing
    extra = sorted(e for e in exported if e not in decl)
    assert not extra, extra


def test_ctypes_load(so):
    from paper_2405_18966_b200 import svdsc
    L = svdsc.lib()
    for name in declared():
        assert hasattr(L, name)
    assert L.svdsc_version().decode().startswith("svdsc")


def test_product_does_not_use_oracle():
    pkg = os.path.join(ROOT, "paper_2405_18966_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f


def test_partitioner_host_only(so):
    from paper_2405_18966_b200 import svdsc
    import workloads as W
    A = W.sparse_powerlaw(20000, 10000, 300000, cap=5000, seed=1)
    for P in (1, 2, 3, 8):
        b = svdsc.partition_rows(A.row_ptr, 200, P)
        assert b[0] == 0 and b[-1] == A.m and np.all(np.diff(b) >= 0)
        cost = 24 * np.diff(A.row_ptr) + 24 * 200
        part = np.array([cost[b[q]:b[q + 1]].sum() for q in range(P)])
        # balanced up to one row's cost
        assert part.max() - part.min() <= 2 * cost.max() + 1
