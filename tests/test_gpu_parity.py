"""Parity of the CUDA path (through the C ABI) with the CPU oracle, row by row
of SURVEY.md 8(a), on seeded synthetic inputs.  -m gpu (B200 via gpurun).

Tolerances:
  * products a1/a5: per element |y - y_or| <= 2 gamma_{L+2} sum_j |a_rj x_j|
    (both sides are valid reduction orders; gamma_n = n u / (1 - n u)).
  * CGS2 / norms: |w - w_or| <= 1e-12 ||w_in||, |nrm - nrm_or| <= 1e-12 ||w_in||.
  * small SVD: |s - s_or| <= 1e-13 s_1; singular vectors (distinct s, sign rule)
    within 1e-9.
  * end to end (BASELINE north_star): |s_i - s_i^or| <= 1e-10 s_1, principal
    angles (from sines) <= 1e-8, same pass count (reading Q18).
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from helpers import certificates, gamma, orth_error, sin_max_angle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2405_18966_b200 import build, svdsc
    build.build()
    return svdsc


@pytest.fixture(scope="module")
def H(S):
    return S.Handle()


@pytest.fixture
def Hp(S):
    """A fresh handle per test, for tests that force a kernel schedule
    (svdsc_set_policy applies to the handle's later calls)."""
    h = S.Handle()
    yield h
    h.close()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def product_budget(A, x, trans):
    D = np.abs(A.to_dense()) if (A.kind == "dense" or A.m * A.n < 4e7) else None
    if D is not None:
        absprod = (D.T if trans else D) @ np.abs(x)
        lens = (D.T if trans else D).astype(bool).sum(1) if A.kind == "csr" else np.full(absprod.size, A.m if trans else A.n)
    else:
        Aa = W.Matrix("csr", A.m, A.n, row_ptr=A.row_ptr, col_idx=A.col_idx, values=np.abs(A.values))
        absprod = O.spmv_t(Aa, np.abs(x)) if trans else O.spmv(Aa, np.abs(x))
        if trans:
            lens = np.bincount(A.col_idx, minlength=A.n)
        else:
            lens = np.diff(A.row_ptr)
    return 2 * gamma(lens + 2) * absprod


def check_products(S, H, A, seed=0):
    M = S.Matrix.from_host(H, A)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(A.n)
    u = rng.standard_normal(A.m)
    y = S.matvec(M, dev(x)).cpu().numpy()
    yt = S.matvec(M, dev(u), trans=True).cpu().numpy()
    y_or, yt_or = O.spmv(A, x), O.spmv_t(A, u)
    assert np.all(np.abs(y - y_or) <= product_budget(A, x, False) + 1e-300)
    assert np.all(np.abs(yt - yt_or) <= product_budget(A, u, True) + 1e-300)
    # epilogue: y = A x - c * yprev
    c = torch.tensor([0.75], dtype=torch.float64, device="cuda")
    yp = rng.standard_normal(A.m)
    y2 = S.matvec(M, dev(x), c=c, yprev=dev(yp)).cpu().numpy()
    assert np.all(np.abs(y2 - (y_or - 0.75 * yp)) <= product_budget(A, x, False) + 4 * gamma(2) * np.abs(yp) + 1e-300)
    M.close()


# ---------------------------------------------------------------- a1 / a5
@pytest.mark.parametrize("sched", ["auto", "bins", "seg"])
@pytest.mark.parametrize("cid,scale", [(1, 1), (3, 10), (4, 100), (5, 1000), (4, 10), (3, 2)])
def test_products_configs(S, Hp, cid, scale, sched):
    """Every SpMV schedule on every config (svdsc_set_policy SVDSC_POLICY_SPMV):
    "auto" picks the row bins or the segmented chunks by row statistics."""
    Hp.set_policy(spmv=sched)
    wl = W.config(cid, scale=scale)
    check_products(S, Hp, wl.A)


@pytest.mark.parametrize("sched", ["auto", "bins", "seg"])
def test_products_edge_cases(S, Hp, sched):
    H = Hp
    H.set_policy(spmv=sched)
    rng = np.random.default_rng(7)
    m, n = 3001, 777
    rows = []
    # empty rows, single-entry rows, a 70k-long row (chunked path), a 3k row (CTA path)
    lens = rng.integers(0, 40, m)
    lens[::17] = 0
    lens[-3:] = 0  # trailing empty rows (row 0 is empty too)
    lens[5] = n  # dense row
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int32)
    val = rng.standard_normal(rp[-1])
    A = W.Matrix("csr", m, n, row_ptr=rp, col_idx=col, values=val)
    check_products(S, H, A)
    # a very long row (> 65536 nnz) with duplicates (duplicates act as their sum)
    m2, n2 = 40, 50000
    lens2 = np.full(m2, 3)
    lens2[7] = 150000
    rp2 = np.zeros(m2 + 1, np.int64)
    rp2[1:] = np.cumsum(lens2)
    col2 = rng.integers(0, n2, rp2[-1]).astype(np.int32)
    A2 = W.Matrix("csr", m2, n2, row_ptr=rp2, col_idx=col2, values=rng.standard_normal(rp2[-1]))
    M = S.Matrix.from_host(H, A2)
    x = rng.standard_normal(n2)
    u = rng.standard_normal(m2)
    y = S.matvec(M, dev(x)).cpu().numpy()
    yt = S.matvec(M, dev(u), trans=True).cpu().numpy()
    assert np.all(np.abs(y - O.spmv(A2, x)) <= product_budget(A2, x, False) + 1e-300)
    # the transposed product sums duplicates; bound by the same per-column budget
    Aa = W.Matrix("csr", m2, n2, row_ptr=rp2, col_idx=col2, values=np.abs(A2.values))
    bud = 2 * gamma(np.bincount(col2, minlength=n2) + 2) * O.spmv_t(Aa, np.abs(u))
    assert np.all(np.abs(yt - O.spmv_t(A2, u)) <= bud + 1e-300)


@pytest.mark.parametrize("m,n", [(5000, 1250), (1001, 333), (20000, 5000)])
def test_products_dense(S, H, m, n):
    rng = np.random.default_rng(m)
    A = W.dense_matrix(rng.standard_normal((m, n)))
    check_products(S, H, A, seed=n)


# ---------------------------------------------------------------- a2-a4 / a6
@pytest.mark.parametrize("variant", ["auto", "split", "qs", "stream", "tma", "cluster"])
@pytest.mark.parametrize("N,c", [(10007, 37), (200000, 300), (4096, 150), (1250, 64), (333, 5), (4096, 65),
                                 (4096, 96), (4096, 128), (4096, 129), (65536, 150), (70001, 257),
                                 (4096, 600), (30011, 17), (70001, 9), (40000, 30), (3, 1), (50000, 0)])
def test_cgs2_variants(S, Hp, N, c, variant):
    """One re-orthogonalization half-step (svdsc_op_cgs2: CGS2 + norm +
    normalize) through every kernel the solver may pick (svdsc_set_policy
    SVDSC_POLICY_CGS2; a forced kernel that cannot run the shape falls back to
    the split sweeps) against the oracle's CGS2 and norm."""
    Hp.set_policy(cgs2=variant)
    rng = np.random.default_rng(N * 7 + c)
    Q = np.linalg.qr(rng.standard_normal((N, max(c, 1))))[0][:, :c]
    w = rng.standard_normal(N)
    if c:
        w += Q @ rng.standard_normal(c) * 3
    ld = -(-N // 32) * 32
    Qd = torch.zeros((c + 1, ld), dtype=torch.float64, device="cuda")  # column-major, ld % 32 == 0
    if c:
        Qd[:c, :N] = dev(np.ascontiguousarray(Q.T))
    wd = torch.zeros(ld, dtype=torch.float64, device="cuda")
    wd[:N] = dev(w)
    Qv = Qd.t()[:N, :c] if c else None
    wg, nrm = S.cgs2(Hp, Qv, wd[:N])
    w_or = O.cgs2(Q, w) if c else w.copy()
    nor = O.norm2(w_or)
    assert abs(nrm.item() - nor) <= 1e-12 * np.linalg.norm(w)
    assert np.abs(wg.cpu().numpy() - w_or / nor).max() <= 1e-12 * np.linalg.norm(w) / nor


# ---------------------------------------------------------------- a7
def _bidiag(rng, p):
    T = np.diag(rng.uniform(0.5, 2, p)) + np.diag(rng.uniform(0.1, 1, p - 1), 1)
    return T


def _arrow(rng, p, k):
    T = np.zeros((p, p))
    T[np.arange(k), np.arange(k)] = np.sort(rng.uniform(1, 3, k))[::-1]
    T[:k, k] = rng.uniform(-0.1, 0.1, k)
    T[k:, k:] = _bidiag(rng, p - k)
    return T


@pytest.mark.parametrize("kernel", ["auto", "register", "block", "one_cta"])
@pytest.mark.parametrize("p,kind", [(30, "bidiag"), (150, "arrow"), (300, "arrow"), (31, "bidiag"), (1, "bidiag"),
                                    (2, "bidiag"), (33, "arrow"), (63, "arrow"), (64, "bidiag"), (601, "arrow")])
def test_small_svd(S, Hp, p, kind, kernel):
    H = Hp
    if kernel == "one_cta" and p > 300:
        pytest.skip("one-CTA fallback is slow at this size")
    if kernel == "register" and p > 64:
        pytest.skip("register Jacobi is for p <= 64 (auto beyond)")
    H.set_policy(small_svd=kernel)
    rng = np.random.default_rng(p)
    T = _bidiag(rng, p) if kind == "bidiag" or p < 3 else _arrow(rng, p, p // 3)
    Td = S.colmajor(p, p)
    Td.copy_(dev(np.asfortranarray(T)))
    U, s, V, sw = S.small_svd(H, Td)
    Uo, so, Vo, _ = O.jacobi_svd(T)
    s = s.cpu().numpy()
    # rounding of ~50 p rotations per column on two valid orders (DESIGN.md tolerances)
    assert np.abs(s - so).max() <= 2e-12 * so[0]
    gaps = np.minimum(np.abs(np.diff(so, prepend=np.inf)), np.abs(np.diff(so, append=-np.inf)))
    ok = gaps > 1e-6 * so[0]
    # singular-vector error <= (sigma error budget) / gap, column by column
    bud = 5e-12 * so[0] / gaps[ok]
    assert np.all(np.abs(U.cpu().numpy()[:, ok] - Uo[:, ok]).max(0) <= bud)
    assert np.all(np.abs(V.cpu().numpy()[:, ok] - Vo[:, ok]).max(0) <= bud)
    print(f"p={p} sweeps={sw}")
    assert orth_error(U.cpu().numpy()) <= 1e-13 * p and orth_error(V.cpu().numpy()) <= 1e-13 * p


# ---------------------------------------------------------------- a8 / a9
@pytest.mark.parametrize("N,t,k", [(10007, 30, 10), (200000, 300, 100), (77, 600, 200)])
def test_recombine(S, H, N, t, k):
    rng = np.random.default_rng(t)
    Q = rng.standard_normal((N, t + 1))
    Wm = rng.standard_normal((t, t))
    Qd = S.colmajor(N, t + 1)
    Qd.copy_(dev(np.asfortranarray(Q)))
    Wd = S.colmajor(t, t)
    Wd.copy_(dev(np.asfortranarray(Wm)))
    out = S.recombine(H, Qd, Wd, k).cpu().numpy()
    ref = Q[:, :t] @ Wm[:, :k]
    bud = 2 * gamma(t + 2) * (np.abs(Q[:, :t]) @ np.abs(Wm[:, :k]))
    assert np.all(np.abs(out - ref) <= bud)
    # in place
    S.recombine(H, Qd, Wd, k, out=Qd)
    got = Qd.cpu().numpy()
    assert np.all(np.abs(got[:, :k] - ref) <= bud)
    assert np.array_equal(got[:, k:], Q[:, k:])


# ---------------------------------------------------------------- one pass
@pytest.mark.parametrize("cid,scale,t", [(1, 1, 30), (3, 20, 60), (2, 4, 40), (4, 100, 40)])
def test_lbp_first_pass(S, H, cid, scale, t):
    wl = W.config(cid, scale=scale)
    M = S.Matrix.from_host(H, wl.A)
    U, V, T, info = S.lbp(M, t, dev(wl.v0))
    Uo, Vo, To, _ = O.lbp(wl.A, t, wl.v0)
    T = T.cpu().numpy()
    al, be = np.diag(T)[:t], np.diag(T, 1)[:t]
    alo, beo = np.diag(To)[:t], np.diag(To, 1)[:t]
    scale_ = max(alo.max(), beo.max())
    assert np.abs(al - alo).max() <= 1e-10 * scale_
    assert np.abs(be - beo).max() <= 1e-10 * scale_
    assert orth_error(U.cpu().numpy()[:, :t]) <= 1e-12
    assert orth_error(V.cpu().numpy()) <= 1e-12
    assert sin_max_angle(U.cpu().numpy()[:, :t], Uo[:, :t]) <= 1e-8
    assert sin_max_angle(V.cpu().numpy(), Vo) <= 1e-8
    assert info["matvecs"] == 2 * t  # u_{t+1} is not formed on the GPU (reading Q2)
    M.close()


# ---------------------------------------------------------------- end to end
def _e2e(S, H, wl, fixed=True, **kw):
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit, **kw)
    M = S.Matrix.from_host(H, wl.A)
    r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0),
                 fixed_passes=r_or.passes if fixed else 0, **kw)
    s = r.S.cpu().numpy()
    assert np.abs(s - r_or.S).max() <= 1e-10 * r_or.S[0]
    U, V = r.U.cpu().numpy(), r.V.cpu().numpy()
    assert r.info["passes"] == r_or.passes
    M.close()
    return r, r_or, U, V, s


@pytest.mark.parametrize("mode", ["fused", "stream", "split"])
@pytest.mark.parametrize("cid,scale", [(1, 1), (2, 4), (3, 20), (6, 10), (7, 10), (8, 10)])
def test_svds_parity(S, Hp, cid, scale, mode):
    H = Hp
    if mode == "split":
        H.set_policy(cgs2="split")
    if mode == "stream":
        if cid == 1:
            pytest.skip("covered by the other configs")
        H.set_policy(cgs2="stream")
    wl = W.config(cid, scale=scale)
    r, r_or, U, V, s = _e2e(S, H, wl)
    k = wl.k
    assert sin_max_angle(U, r_or.U) <= 1e-8
    assert sin_max_angle(V, r_or.V) <= 1e-8
    assert bool(r.info["converged"]) == r_or.converged
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10
    r1, r2 = certificates(wl.A, s, U, V)
    assert np.all(r1 <= 1e-10 * s[0])
    # Eq. (4) residual vs the true ||A^T u - s v|| / s: they agree to rounding
    # of the computed vectors, ~eps ||A|| / s_j relative -- compared absolutely,
    # in units of sigma_1 (reading Q16a: Decay3 has s_k / s_1 = 1e-6)
    assert np.all(np.abs(r2 - r.resid.cpu().numpy()) * s <= 1e-8 * s[0])
    # free-running GPU stops on the same pass as the oracle here
    M = S.Matrix.from_host(H, wl.A)
    rf = S.svds_c(M, k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0))
    assert rf.info["passes"] == r_or.passes


def test_svds_forced_restarts_and_breakdown(S, H):
    # t = k + 3 forces restarts (Eqs. 5-7)
    A = W.dense_with_spectrum(500, 400, W.spectrum("decay1", 400), seed=5)
    wl = W.Workload("decay1", A, W.start_vector(400, 5), 10, 13, 1e-10, 500)
    r, r_or, U, V, s = _e2e(S, H, wl)
    assert r.info["restarts"] >= 1, r.info
    assert r.info["steps"] == r_or.steps, (r.info, r_or.steps, r_or.passes, r_or.restarts)
    # exactly rank-3 matrix, k = 5: breakdown replacements (reading Q7)
    rng = np.random.default_rng(3)
    D = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 40))
    wl2 = W.Workload("rank3", W.dense_matrix(D), rng.standard_normal(40), 5, 15, 1e-10, 20)
    r_or = O.svds(wl2.A, 5, wl2.v0, t=15, maxit=20)
    M = S.Matrix.from_host(H, wl2.A)
    r = S.svds_c(M, 5, t=15, maxit=20, v0=dev(wl2.v0), fixed_passes=r_or.passes)
    # After the Krylov space is exhausted every new vector is rounding noise whose
    # norm sits at the breakdown threshold 1e-14 max(alpha, beta) (reading Q7), so
    # the decision on a vector can flip with the reduction order; the count
    # agrees up to such flips (Q7a), the three nonzero sigma exactly.
    assert r_or.breakdowns >= 1 and r.info["breakdowns"] >= 1
    assert abs(r.info["breakdowns"] - r_or.breakdowns) <= 2
    assert np.abs(r.S.cpu().numpy()[:3] - r_or.S[:3]).max() <= 1e-10 * r_or.S[0]


def test_svds_contract_errors(S, H):
    wl = W.config(1, scale=10)
    M = S.Matrix.from_host(H, wl.A)
    for kw in (dict(k=0), dict(k=5, tol=0.0), dict(k=298), dict(k=5, reorth=3), dict(k=5, reorth=-2)):
        with pytest.raises(S.SvdscError) as e:
            S.svds_c(M, **kw)
        assert e.value.status == -1
    r = S.svds_c(M, 5, maxit=1, v0=dev(wl.v0), tol=1e-14)
    assert r.status == 1 and r.info["passes"] == 1  # NOT_CONVERGED, outputs filled
    assert np.all(np.isfinite(r.S.cpu().numpy()))


def test_deterministic_and_host_path(S, H):
    wl = W.config(1, scale=2)
    M = S.Matrix.from_host(H, wl.A)
    a = S.svds_c(M, wl.k, t=wl.t, v0=dev(wl.v0))
    b = S.svds_c(M, wl.k, t=wl.t, v0=dev(wl.v0))
    assert torch.equal(a.S, b.S) and torch.equal(a.U, b.U) and torch.equal(a.V, b.V)
    Sh, Uh, Vh, Rh, st, info = S.svds_c_host(H, wl.A, wl.k, t=wl.t, v0=wl.v0)
    assert np.array_equal(Sh, a.S.cpu().numpy()) and np.array_equal(Uh, a.U.cpu().numpy())
    assert np.array_equal(Vh, a.V.cpu().numpy())


# ---------------------------------------------------------------- scaled replicas of configs 4 and 5
def test_svds_parity_config4_scaled(S, H):
    """BASELINE config 4 (power-law rows, 4M x 2M, k = 100, t = 300) at 1/200
    scale: full oracle parity (SURVEY.md 8(c) pin (i) for configs 4-5)."""
    wl = W.config(4, scale=200)
    r, r_or, U, V, s = _e2e(S, H, wl)
    assert sin_max_angle(U, r_or.U) <= 1e-8 and sin_max_angle(V, r_or.V) <= 1e-8
    r1, r2 = certificates(wl.A, s, U, V)
    assert np.all(r1 <= 1e-10 * s[0])
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10


def test_svds_parity_config5_scaled(S, H):
    """BASELINE config 5 (banded-plus-random rows, 30M x 5M, k = 200, t = 600) at
    1/2000 scale against the oracle's stored result (tests/golden/
    oracle_config5_div2000.json, written by tools/make_golden_c5.py, which calls
    only oracle/): sigma parity, same pass count, and the a-posteriori
    certificates of the GPU vectors.  Exercises the t = 600 paths (p = 601
    cluster Jacobi with the register-pull exchange, 601-column CGS2)."""
    g = json.load(open(os.path.join(GOLD, "oracle_config5_div2000.json")))
    wl = W.config(5, scale=2000)
    assert (wl.A.m, wl.A.n, int(wl.A.nnz), wl.k, wl.t) == (g["m"], g["n"], g["nnz"], g["k"], g["t"])
    M = S.Matrix.from_host(H, wl.A)
    r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0), fixed_passes=g["passes"])
    s = r.S.cpu().numpy()
    S_or = np.array(g["S"])
    assert np.abs(s - S_or).max() <= 1e-10 * S_or[0]
    assert bool(r.info["converged"]) == g["converged"]
    U, V = r.U.cpu().numpy(), r.V.cpu().numpy()
    r1, r2 = certificates(wl.A, s, U, V)
    assert np.all(r1 <= 1e-10 * s[0])
    assert np.all(np.abs(r2 - r.resid.cpu().numpy()) * s <= 1e-8 * s[0])
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10
