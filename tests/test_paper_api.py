"""The paper's interface (include/svdsc_paper.h) and Matrix
Market I/O: host-only layout conversion and parsing run
without a GPU; svds_C / svds_C_dense and the CLI run on the GPU against the
CPU oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import workloads as W
from paper_2405_18966_b200 import build as B
from paper_2405_18966_b200 import svdsc as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2405_18966_b200", "svdsc-cli")


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


# ---------------------------------------------------------------- layout (host)
def test_paper_layout_identity():
    # pointerB=[1,2], pointerE=[2,3], cols=[1,2] -> row_ptr [0,1,2], cols [0,1]
    A = S.paper_csr(2, 2, [1.0, 1.0], [1, 2], [1, 2], [2, 3])
    rp, ci, va = S.paper_csr_to_csr(A)
    assert rp.tolist() == [0, 1, 2] and ci.tolist() == [0, 1] and va.tolist() == [1.0, 1.0]


def test_paper_layout_empty_row_and_gaps():
    # row 1 empty (pointerB == pointerE); a gap between pointerE[0] and pointerB[2]
    # (entries 3..4 of cols belong to no row) is dropped
    vals = [1.0, 2.0, 99.0, 98.0, 3.0]
    cols = [1, 3, 2, 2, 2]
    A = S.paper_csr(3, 3, vals, cols, [1, 3, 5], [3, 3, 6])
    rp, ci, va = S.paper_csr_to_csr(A)
    assert rp.tolist() == [0, 2, 2, 3]
    assert ci.tolist() == [0, 2, 1] and va.tolist() == [1.0, 2.0, 3.0]


@pytest.mark.parametrize("pB,pE,cols", [([2, 1], [1, 2], [1, 1]),   # pointerE < pointerB
                                         ([1, 2], [2, 9], [1, 1]),   # past nnz + 1
                                         ([1, 2], [2, 3], [1, 7])])  # column outside 1..ncols
def test_paper_layout_errors(pB, pE, cols):
    A = S.paper_csr(2, 2, [1.0, 1.0], cols, pB, pE)
    with pytest.raises(S.PaperError):
        S.paper_csr_to_csr(A)


# ---------------------------------------------------------------- Matrix Market (host)
def test_mm_identity_duplicates_symmetric(tmp_path):
    p = write(tmp_path, "id.mtx", "%%MatrixMarket matrix coordinate real general\n% c\n2 2 2\n1 1 1\n2 2 1\n")
    kind, d = S.read_mm(p)
    assert kind == "csr" and d["pointerB"].tolist() == [1, 2] and d["pointerE"].tolist() == [2, 3]
    assert d["cols"].tolist() == [1, 2] and d["values"].tolist() == [1.0, 1.0]
    p = write(tmp_path, "dup.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.5\n1 1 0.5\n")
    _, d = S.read_mm(p)
    assert d["values"].tolist() == [1.0] and d["pointerE"].tolist() == [2, 2]
    p = write(tmp_path, "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 4\n3 3 5\n")
    _, d = S.read_mm(p)
    assert len(d["values"]) == 3  # off-diagonal expanded to both triangles
    rp, ci, va = S.paper_csr_to_csr(S.paper_csr(3, 3, d["values"], d["cols"], d["pointerB"], d["pointerE"]))
    D = np.zeros((3, 3))
    for i in range(3):
        D[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    assert np.array_equal(D, [[0, 4, 0], [4, 0, 0], [0, 0, 5]])


def test_mm_array_and_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    A = rng.standard_normal((5, 3))
    p = tmp_path / "a.mtx"
    S.write_mm(p, dense=A)
    kind, D = S.read_mm(p)
    assert kind == "dense" and np.array_equal(D, A)  # 17 significant digits: lossless
    Sp = W.sparse_uniform_cells(40, 30, 200, seed=2)
    pB = (Sp.row_ptr[:-1] + 1).astype(np.int32)
    pE = (Sp.row_ptr[1:] + 1).astype(np.int32)
    csr = {"nrows": 40, "ncols": 30, "values": Sp.values, "cols": Sp.col_idx + 1, "pointerB": pB, "pointerE": pE}
    q = tmp_path / "s.mtx"
    S.write_mm(q, csr=csr)
    kind, d = S.read_mm(q)
    assert kind == "csr"
    assert np.array_equal(d["values"], Sp.values) and np.array_equal(d["cols"] - 1, Sp.col_idx)
    assert np.array_equal(d["pointerB"], pB) and np.array_equal(d["pointerE"], pE)


@pytest.mark.parametrize("text,where", [
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", ":1:"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", ":3:"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "fewer entries"),
    ("hello\n", ":1:")])
def test_mm_errors_name_the_line(tmp_path, text, where):
    p = write(tmp_path, "bad.mtx", text)
    with pytest.raises(S.PaperError) as e:
        S.read_mm(p)
    assert where in str(e.value)


def test_cli_usage_errors():
    assert subprocess.run([CLI, "decompose", "--k", "0", "--input", "x.mtx"], capture_output=True).returncode == 1
    assert subprocess.run([CLI, "frobnicate"], capture_output=True).returncode == 1


# ---------------------------------------------------------------- on the GPU
@pytest.mark.gpu
def test_svds_C_sparse_and_dense_vs_oracle(tmp_path):
    wl = W.config(1, scale=2)
    A = wl.A
    Pc = S.paper_csr(A.m, A.n, A.values, A.col_idx + 1, A.row_ptr[:-1] + 1, A.row_ptr[1:] + 1)
    U, s, V, st = S.svds_C(Pc, 5)  # paper defaults: tol 1e-10, t = max(15, 3k), r = 10
    assert U.shape == (A.m, 5) and V.shape == (A.n, 5) and st in (0, 1)
    D = np.zeros((A.m, A.n))
    for i in range(A.m):
        D[i, A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.values[A.row_ptr[i]:A.row_ptr[i + 1]]
    assert np.linalg.norm(D @ V - U * s, axis=0).max() <= 1e-9 * s[0]
    # the paper's interface has no start-vector argument (the library draws it,
    # reading Q8), so the oracle cannot share it; with enough restarts to
    # converge, both must reach the exact top sigma (library SVD of the dense
    # expansion) to the tolerance-limited accuracy -- asserted unconditionally
    U, s, V, st = S.svds_C(Pc, 5, tol=1e-10, t=15, r=200)
    assert st == 0
    r_or = O.svds(A, 5, np.random.default_rng(0).standard_normal(A.n), tol=1e-10, t=15, maxit=200)
    assert r_or.converged
    s_np = np.linalg.svd(D, compute_uv=False)[:5]
    assert np.abs(s - s_np).max() <= 1e-8 * s_np[0]
    assert np.abs(r_or.S - s_np).max() <= 1e-8 * s_np[0]
    assert np.abs(s - r_or.S).max() <= 1e-8 * s_np[0]
    # dense entry point, options given explicitly
    Dd = W.dense_with_spectrum(300, 200, W.spectrum("decay2", 200), seed=4)
    U2, s2, V2, st2 = S.svds_C(Dd.dense, 8, tol=1e-10, t=40, r=20)
    assert st2 == 0
    assert np.abs(s2 - W.spectrum("decay2", 8)).max() <= 1e-10


@pytest.mark.gpu
def test_cli_decompose(tmp_path):
    Dd = W.dense_with_spectrum(200, 150, W.spectrum("decay2", 150), seed=7)
    p = tmp_path / "decay2.mtx"
    S.write_mm(p, dense=Dd.dense)
    out = tmp_path / "r.json"
    pr = subprocess.run([CLI, "decompose", "--input", str(p), "--k", "6", "--tol", "1e-10", "--restarts", "10",
                         "--output", str(out)], capture_output=True, text=True)
    assert pr.returncode == 0, pr.stderr
    doc = json.loads(out.read_text())
    assert doc["converged"] and doc["m"] == 200 and len(doc["singular_values"]) == 6
    assert np.abs(np.array(doc["singular_values"]) - W.spectrum("decay2", 6)).max() <= 1e-10
    assert max(doc["residuals"]) < 1e-10
    pr = subprocess.run([CLI, "decompose", "--input", str(p), "--k", "3", "--output", str(tmp_path / "r.csv")],
                        capture_output=True, text=True)
    assert pr.returncode == 0
    lines = (tmp_path / "r.csv").read_text().strip().splitlines()
    assert lines[0] == "index,sigma,residual" and len(lines) == 4
