"""The library's multi-rank path (row-partitioned A, sliced V,
reduce-scatter of A^T u, all-gather of v, all-reduces of the CGS2 coefficient
vectors between the three launches of the streaming CGS2 kernel, status
agreement before compute) driven on ONE GPU: P ranks are threads of this
process, each with its own handle and stream, joined by the in-process
loopback group (svdsc_comm_init_group).  The collectives synchronize each
rank's stream and meet at a host barrier (no kernel waits on another rank).

The result must match the CPU oracle with the BASELINE.json north_star
tolerances (sigma within 1e-10 sigma_1, principal angles <= 1e-8, same pass
count: reading Q18) -- the same bar as the single-GPU path.  -m gpu.
"""
import threading

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


def local_rows(A, r0, r1):
    if A.kind == "csr":
        rp = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
        return W.Matrix("csr", r1 - r0, A.n, row_ptr=rp, col_idx=A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]],
                        values=A.values[A.row_ptr[r0]:A.row_ptr[r1]])
    return W.dense_matrix(np.ascontiguousarray(A.dense[r0:r1]))


def run_ranks(S, wl, P, bounds, opts_per_rank=None, timeout=600):
    """Solve wl on P loopback ranks; returns per-rank (status, S, U_local, V, info) or exceptions."""
    g = S.Group(P)
    out = [None] * P
    barrier = threading.Barrier(P)

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                h = S.Handle(st)
                h.comm_init_group(g, r)
                r0, r1 = int(bounds[r]), int(bounds[r + 1])
                M = S.Matrix.from_host(h, local_rows(wl.A, r0, r1), row_offset=r0, m_global=wl.A.m)
                kw = dict(k=wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit,
                          v0=torch.from_numpy(wl.v0).cuda())
                if opts_per_rank:
                    kw.update(opts_per_rank[r])
                barrier.wait()
                try:
                    res = S.svds_c(M, **kw)
                    st.synchronize()
                    out[r] = (res.status, res.S.cpu().numpy(), res.U.cpu().numpy(), res.V.cpu().numpy(), res.info)
                except S.SvdscError as e:
                    out[r] = e
                M.close()
                h.close()
        except Exception as e:  # noqa: BLE001
            out[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
        assert not t.is_alive(), "a rank hung"
    g.close()
    return out


def bounds_for(S, wl, P):
    if wl.A.kind == "csr":
        return S.partition_rows(wl.A.row_ptr, (wl.k + wl.t) // 2, P)
    return np.linspace(0, wl.A.m, P + 1).astype(np.int64)


@pytest.mark.parametrize("cid,scale,P", [(1, 2, 2), (3, 20, 2), (4, 200, 3), (2, 8, 2), (5, 2000, 2)])
def test_loopback_ranks_match_oracle(S, cid, scale, P):
    wl = W.config(cid, scale=scale)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    bounds = bounds_for(S, wl, P)
    out = run_ranks(S, wl, P, bounds, [dict(fixed_passes=r_or.passes)] * P)
    for o in out:
        assert not isinstance(o, Exception), o
    s0 = out[0][1]
    for r in range(1, P):  # S and V are replicated, bitwise (rank-ordered sums)
        assert np.array_equal(out[r][1], s0)
        assert np.array_equal(out[r][3], out[0][3])
    U = np.concatenate([out[r][2] for r in range(P)], axis=0)
    V = out[0][3]
    assert np.abs(s0 - r_or.S).max() <= 1e-10 * r_or.S[0]
    assert sin_max_angle(U, r_or.U) <= 1e-8
    assert sin_max_angle(V, r_or.V) <= 1e-8
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10
    r1, _ = certificates(wl.A, s0, U, V)
    assert np.all(r1 <= 1e-10 * s0[0])
    info = out[0][4]
    assert info["passes"] == r_or.passes
    assert info["steps"] == r_or.steps


def test_loopback_free_running_same_passes(S):
    # without fixed_passes the ranks stop on the same pass as the oracle
    wl = W.config(3, scale=20)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    out = run_ranks(S, wl, 2, bounds_for(S, wl, 2))
    for o in out:
        assert not isinstance(o, Exception), o
        assert o[4]["passes"] == r_or.passes and o[0] == 0


def test_status_agreement(S):
    """One rank's contract violation: every rank returns an error before any
    compute, none hangs in a collective (SURVEY.md 8(b) "Multi-GPU")."""
    wl = W.config(1, scale=5)
    out = run_ranks(S, wl, 2, bounds_for(S, wl, 2), [dict(), dict(k=0)], timeout=120)
    assert isinstance(out[1], S.SvdscError) and out[1].status == -1
    assert isinstance(out[0], S.SvdscError) and out[0].status == -1
    assert "another rank" in str(out[0])


def test_loopback_breakdown_and_restarts(S):
    # exactly rank-3 rows partitioned over 2 ranks (breakdown repairs are
    # agreed across ranks) and t = k + 3 (restarts) on another matrix
    rng = np.random.default_rng(3)
    D = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 40))
    wl = W.Workload("rank3", W.dense_matrix(D), rng.standard_normal(40), 5, 15, 1e-10, 20)
    r_or = O.svds(wl.A, 5, wl.v0, t=15, maxit=20)
    out = run_ranks(S, wl, 2, np.array([0, 29, 60]), [dict(fixed_passes=r_or.passes)] * 2)
    for o in out:
        assert not isinstance(o, Exception), o
    assert out[0][4]["breakdowns"] >= 1
    assert np.abs(out[0][1][:3] - r_or.S[:3]).max() <= 1e-10 * r_or.S[0]
    A = W.dense_with_spectrum(500, 400, W.spectrum("decay1", 400), seed=5)
    wl2 = W.Workload("decay1", A, W.start_vector(400, 5), 10, 13, 1e-10, 500)
    r2 = O.svds(wl2.A, 10, wl2.v0, tol=1e-10, t=13, maxit=500)
    out = run_ranks(S, wl2, 2, np.array([0, 250, 500]), [dict(fixed_passes=r2.passes)] * 2)
    for o in out:
        assert not isinstance(o, Exception), o
    assert out[0][4]["restarts"] >= 1
    assert np.abs(out[0][1] - r2.S).max() <= 1e-10 * r2.S[0]


def test_comm_check_nccl_one_rank(S):
    """The NCCL communicator code (runtime-loaded libnccl, ncclCommInitRank and
    every collective wrapper of comm.cu) on the one GPU of the box: a one-rank
    communicator passes svdsc_comm_check, and a solve on that handle (single-GPU
    path) is bitwise equal to one without a communicator."""
    uid = S.comm_unique_id()
    assert len(uid) == 128
    wl = W.config(1, scale=2)
    res = []
    for with_comm in (False, True):
        h = S.Handle()
        if with_comm:
            h.comm_init(1, 0, uid)
            h.comm_check()
        M = S.Matrix.from_host(h, wl.A)
        r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=torch.from_numpy(wl.v0).cuda(), fixed_passes=3)
        res.append((r.S.cpu().numpy(), r.U.cpu().numpy(), r.V.cpu().numpy()))
        M.close()
        h.close()
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("P", [1, 2, 3])
def test_comm_check_loopback(S, P):
    g = S.Group(P)
    errs = [None] * P

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                h = S.Handle(st)
                h.comm_init_group(g, r)
                h.comm_check()
                h.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
        assert not t.is_alive(), "a rank hung"
    g.close()
    assert errs == [None] * P, errs


def test_comm_check_without_communicator(S):
    h = S.Handle()
    with pytest.raises(S.SvdscError) as e:
        h.comm_check()
    assert e.value.status == -1
    h.close()
