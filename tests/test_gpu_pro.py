"""Parity of the partial re-orthogonalization path (opts.reorth = 1, SURVEY.md
8(f4), reading Q20) with the oracle's, through the C ABI.  -m gpu.

The decisions are integers taken from floating point: both sides compute the
omega rows with the same operation order (pro.cu mirrors oracle.c), but the
norms and T entries they start from differ by rounding, so the tests compare
what decides the outcome: the alpha/beta sequences to 1e-10 (a single flipped
decision would move them by ~sqrt(eps) relative), the number of
re-orthogonalized half-steps (the oracle also decides for u_{t+1}, which the
GPU does not form, reading Q2: it may count up to one more per pass), the
singular values to the end-to-end bar, and the semi-orthogonality the method
promises.  The sizes cover every fused CGS2 variant the gate sits in
(cluster, Q-resident, streaming).
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from helpers import certificates, orth_error

pytestmark = pytest.mark.gpu
SQRT_EPS = 2.0 ** -26


@pytest.fixture(scope="module")
def S():
    from paper_2405_18966_b200 import build, svdsc
    build.build()
    return svdsc


@pytest.fixture(scope="module")
def H(S):
    return S.Handle()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def decay2(m=400, n=300, seed=4):
    return W.dense_with_spectrum(m, n, W.spectrum("decay2", n), seed=seed)


@pytest.mark.parametrize("case", ["c1", "decay2", "c2s4", "c3s4"])
def test_pro_lbp_first_pass(S, H, case):
    if case == "c1":
        A, t, v0 = W.config(1).A, 30, W.config(1).v0
    elif case == "decay2":
        A, t = decay2(), 120
        v0 = np.random.default_rng(1).standard_normal(A.n)
    elif case == "c2s4":
        wl = W.config(2, scale=4)
        A, t, v0 = wl.A, wl.t, wl.v0
    else:  # streaming CGS2 kernels on both sides (U: 120 MB, V: 60 MB at t = 300)
        wl = W.config(3, scale=4)
        A, t, v0 = wl.A, wl.t, wl.v0
    M = S.Matrix.from_host(H, A)
    U, V, T, info = S.lbp(M, t, dev(v0), reorth=1)
    Uo, Vo, To, io = O.lbp(A, t, v0, reorth=1)
    T = T.cpu().numpy()
    al, be = np.diag(T)[:t], np.diag(T, 1)[:t]
    alo, beo = np.diag(To)[:t], np.diag(To, 1)[:t]
    sc = max(alo.max(), beo.max())
    assert np.abs(al - alo).max() <= 1e-10 * sc
    assert np.abs(be - beo).max() <= 1e-10 * sc
    assert 0 <= io.reorths - info["reorths"] <= 1
    assert info["reorths"] < 2 * t  # it is partial
    Ug, Vg = U.cpu().numpy()[:, :t], V.cpu().numpy()
    assert orth_error(Ug) <= 10 * SQRT_EPS and orth_error(Vg) <= 10 * SQRT_EPS
    M.close()


@pytest.mark.parametrize("case", ["c1", "decay2", "c2s4"])
def test_pro_svds_vs_oracle(S, H, case):
    if case == "c1":
        wl = W.config(1)
        A, k, t, v0, maxit, tol = wl.A, wl.k, wl.t, wl.v0, 30, 1e-10
    elif case == "decay2":
        A, k, t, maxit, tol = decay2(), 8, 30, 50, 1e-10
        v0 = np.random.default_rng(5).standard_normal(A.n)
    else:
        wl = W.config(2, scale=4)
        A, k, t, v0, maxit, tol = wl.A, wl.k, wl.t, wl.v0, wl.maxit, wl.tol
    r_or = O.svds(A, k, v0, tol=tol, t=t, maxit=maxit, reorth=1)
    M = S.Matrix.from_host(H, A)
    r = S.svds_c(M, k, tol=tol, t=t, maxit=maxit, v0=dev(v0), fixed_passes=r_or.passes, reorth=1)
    s = r.S.cpu().numpy()
    assert np.abs(s - r_or.S).max() <= 1e-10 * r_or.S[0]
    assert bool(r.info["converged"]) == r_or.converged
    assert 0 <= r_or.reorths - r.info["reorths"] <= r_or.passes
    U, V = r.U.cpu().numpy(), r.V.cpu().numpy()
    assert orth_error(U) <= 1e-8 and orth_error(V) <= 1e-8
    # semi-orthogonal bases: the true residual is bounded at the sqrt(eps) level,
    # not by the Eq. (4) estimate (reading Q20; the oracle shows the same)
    r1, _ = certificates(A, s, U, V)
    assert np.all(r1 <= 10 * SQRT_EPS * s[0])
    # free-running: stops on the oracle's pass and re-orthogonalizes less than CGS2 every step
    rf = S.svds_c(M, k, tol=tol, t=t, maxit=maxit, v0=dev(v0), reorth=1)
    assert rf.info["passes"] == r_or.passes
    r2 = S.svds_c(M, k, tol=tol, t=t, maxit=maxit, v0=dev(v0), reorth=2)
    assert rf.info["reorths"] < r2.info["reorths"]
    M.close()


def test_pro_contract(S, H):
    A = W.config(1, scale=2).A
    M = S.Matrix.from_host(H, A)
    with pytest.raises(Exception):
        S.svds_c(M, 5, reorth=3)
    M.close()


def test_pro_forced_restarts_and_breakdown(S, H):
    """reorth = 1 through restarts (t = k + 3) and through breakdown repairs
    (exactly rank-3 matrix, k = 5): the decision kernels are no-ops while a
    breakdown abort is pending and the replayed half-steps decide again."""
    A = W.dense_with_spectrum(500, 400, W.spectrum("decay1", 400), seed=5)
    v0 = W.start_vector(400, 5)
    r_or = O.svds(A, 10, v0, tol=1e-10, t=13, maxit=500, reorth=1)
    M = S.Matrix.from_host(H, A)
    r = S.svds_c(M, 10, tol=1e-10, t=13, maxit=500, v0=dev(v0), fixed_passes=r_or.passes, reorth=1)
    assert r.info["restarts"] >= 1
    assert np.abs(r.S.cpu().numpy() - r_or.S).max() <= 1e-10 * r_or.S[0]
    M.close()
    rng = np.random.default_rng(3)
    D = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 40))
    A2 = W.dense_matrix(D)
    v2 = rng.standard_normal(40)
    r_or = O.svds(A2, 5, v2, t=15, maxit=20, reorth=1)
    M = S.Matrix.from_host(H, A2)
    r = S.svds_c(M, 5, t=15, maxit=20, v0=dev(v2), fixed_passes=r_or.passes, reorth=1)
    assert r_or.breakdowns >= 1 and r.info["breakdowns"] >= 1
    assert np.abs(r.S.cpu().numpy()[:3] - r_or.S[:3]).max() <= 1e-10 * r_or.S[0]
    M.close()
