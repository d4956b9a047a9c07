"""The deferred second CGS2 update of the single-GPU streaming kernel
(reading G5): a re-orthogonalization leaves w' in its basis
column with h2 and 1/beta recorded, the next product reads w'/beta, and the
next call on the same side (or the pass-end flush) forms the column
(w' - Q h2)/beta.  The automatic kernel choice only streams tall bases
(configs 3-5); SVDSC_POLICY_CGS2 = stream forces the streaming kernel -- and
with it the deferral -- on small problems, so every path (first sweep forming
a pending column, explicit-norm fallback, breakdown repair, restarts, the
pass-end flush before the recombination) is checked here against the CPU
oracle at the north_star tolerances.  -m gpu.
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from helpers import certificates, orth_error, sin_max_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2405_18966_b200 import build, svdsc
    build.build()
    return svdsc


@pytest.fixture
def Hs(S):
    h = S.Handle()
    h.set_policy(cgs2="stream")
    yield h
    h.close()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("cid,scale,t", [(1, 1, 30), (3, 20, 60), (2, 4, 40), (4, 100, 40)])
def test_deferred_lbp_first_pass(S, Hs, cid, scale, t):
    """One pass through svdsc_op_lbp: alpha / beta against the oracle, and the
    returned bases (every pending column formed by the next same-side call or
    the pass-end flush) orthonormal and spanning the oracle's subspaces."""
    wl = W.config(cid, scale=scale)
    M = S.Matrix.from_host(Hs, wl.A)
    U, V, T, info = S.lbp(M, t, dev(wl.v0))
    Uo, Vo, To, _ = O.lbp(wl.A, t, wl.v0)
    T = T.cpu().numpy()
    al, be = np.diag(T)[:t], np.diag(T, 1)[:t]
    alo, beo = np.diag(To)[:t], np.diag(To, 1)[:t]
    sc = max(alo.max(), beo.max())
    assert np.abs(al - alo).max() <= 1e-10 * sc
    assert np.abs(be - beo).max() <= 1e-10 * sc
    Un, Vn = U.cpu().numpy()[:, :t], V.cpu().numpy()
    assert orth_error(Un) <= 1e-12 and orth_error(Vn) <= 1e-12
    assert sin_max_angle(Un, Uo[:, :t]) <= 1e-8 and sin_max_angle(Vn, Vo) <= 1e-8
    # column by column: each basis vector is the oracle's to rounding
    assert np.abs(np.abs(np.sum(Un * Uo[:, :t], 0)) - 1).max() <= 1e-9
    M.close()


@pytest.mark.parametrize("cid,scale", [(1, 1), (3, 20), (4, 200)])
def test_deferred_end_to_end(S, Hs, cid, scale):
    wl = W.config(cid, scale=scale)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    M = S.Matrix.from_host(Hs, wl.A)
    r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0), fixed_passes=r_or.passes)
    s, U, V = r.S.cpu().numpy(), r.U.cpu().numpy(), r.V.cpu().numpy()
    assert np.abs(s - r_or.S).max() <= 1e-10 * r_or.S[0]
    assert sin_max_angle(U, r_or.U) <= 1e-8 and sin_max_angle(V, r_or.V) <= 1e-8
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10
    r1, _ = certificates(wl.A, s, U, V)
    assert np.all(r1 <= 1e-10 * s[0])
    # the deferred path moves fewer bytes: two basis sweeps per half-step
    # instead of three (info.bytes_reorth counts what was executed)
    h3 = S.Handle()
    h3.set_policy(cgs2="split")  # the three-sweep reference
    M3 = S.Matrix.from_host(h3, wl.A)
    r3 = S.svds_c(M3, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0), fixed_passes=r_or.passes)
    assert r.info["steps"] == r3.info["steps"]
    assert r.info["bytes_reorth"] < 0.8 * r3.info["bytes_reorth"]
    M3.close()
    h3.close()
    M.close()


def test_deferred_restarts_and_breakdown(S, Hs):
    # t = k + 3 forces restarts (Eqs. 5-7): the pass-end flush precedes the recombination
    A = W.dense_with_spectrum(500, 400, W.spectrum("decay1", 400), seed=5)
    wl = W.Workload("decay1", A, W.start_vector(400, 5), 10, 13, 1e-10, 500)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    M = S.Matrix.from_host(Hs, wl.A)
    r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0), fixed_passes=r_or.passes)
    assert r.info["restarts"] >= 1
    assert np.abs(r.S.cpu().numpy() - r_or.S).max() <= 1e-10 * r_or.S[0]
    assert sin_max_angle(r.V.cpu().numpy(), r_or.V) <= 1e-8
    M.close()
    # exactly rank-3, k = 5: breakdowns while columns are pending (repair after the flush)
    rng = np.random.default_rng(3)
    D = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 40))
    wl2 = W.Workload("rank3", W.dense_matrix(D), rng.standard_normal(40), 5, 15, 1e-10, 20)
    r_or = O.svds(wl2.A, 5, wl2.v0, t=15, maxit=20)
    M = S.Matrix.from_host(Hs, wl2.A)
    r = S.svds_c(M, 5, t=15, maxit=20, v0=dev(wl2.v0), fixed_passes=r_or.passes)
    assert r.info["breakdowns"] >= 1
    assert abs(r.info["breakdowns"] - r_or.breakdowns) <= 2
    assert np.abs(r.S.cpu().numpy()[:3] - r_or.S[:3]).max() <= 1e-10 * r_or.S[0]
    assert orth_error(r.V.cpu().numpy()[:, :3]) <= 1e-10
    M.close()


def test_deferred_deterministic(S, Hs):
    wl = W.config(3, scale=20)
    M = S.Matrix.from_host(Hs, wl.A)
    a = S.svds_c(M, wl.k, t=wl.t, v0=dev(wl.v0), fixed_passes=2)
    Hs.profile(True)  # eager launches instead of the restart-pass graph
    b = S.svds_c(M, wl.k, t=wl.t, v0=dev(wl.v0), fixed_passes=2)
    Hs.profile(False)
    assert torch.equal(a.S, b.S) and torch.equal(a.U, b.U) and torch.equal(a.V, b.V)
    M.close()


def test_defer_policy_off(S):
    """SVDSC_POLICY_DEFER = off: the literal three-sweep CGS2 of PAPER.md:121 in
    the same streaming kernel; the two agree to rounding and with the oracle."""
    wl = W.config(3, scale=20)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    out = {}
    for d in ("auto", "off"):
        h = S.Handle()
        h.set_policy(cgs2="stream", defer=d)
        M = S.Matrix.from_host(h, wl.A)
        r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=dev(wl.v0), fixed_passes=r_or.passes)
        out[d] = (r.S.cpu().numpy(), r.V.cpu().numpy(), r.info["bytes_reorth"])
        M.close()
        h.close()
    for s, V, _ in out.values():
        assert np.abs(s - r_or.S).max() <= 1e-10 * r_or.S[0]
        assert sin_max_angle(V, r_or.V) <= 1e-8
    assert np.abs(out["auto"][0] - out["off"][0]).max() <= 1e-12 * r_or.S[0]
    assert out["auto"][2] < 0.8 * out["off"][2]
