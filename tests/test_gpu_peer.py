"""the multi-GPU re-orthogonalization with its all-reduces
inside the kernel (peer mailboxes: each rank pushes its column sums of
h1 = Q^T w and [h2 = Q^T w'; ||w'||^2] into every rank's mailbox).

On one GPU the P ranks are emulated as P groups of CTAs of ONE cooperative
launch (svdsc_op_cgs2_peer_emulate; separate launches that wait on one another
must never share a GPU), running the same kernel body and protocol the solver
launches once per rank over NCCL.  Checks:
  * every rank's rows of w'' / beta against the oracle's CGS2 of the whole
    vector (the same 1e-12 ||w|| bar as the single-GPU kernels),
  * beta bitwise equal on every rank (rank-ordered sums of the same slots),
  * P = 1 bitwise equal to the single-GPU streaming kernel (same sums),
  * the solver's peer path (SVDSC_POLICY_CGS2 = 6 on a one-rank NCCL
    communicator: mailbox setup, per-solve counter reset, device-resident
    sequence under CUDA-graph replay) bitwise equal to the streaming-kernel
    solve, and against the oracle at the north_star tolerances.  -m gpu.
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W
from helpers import sin_max_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2405_18966_b200 import build, svdsc
    build.build()
    return svdsc


@pytest.fixture(scope="module")
def H(S):
    h = S.Handle()
    yield h
    h.close()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def problem(N, c, seed):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((N, max(c, 1))))[0][:, :c]
    w = rng.standard_normal(N)
    if c:
        w += Q @ rng.standard_normal(c) * 3
    ld = -(-N // 32) * 32
    Qd = torch.zeros((c + 1, ld), dtype=torch.float64, device="cuda")
    if c:
        Qd[:c, :N] = dev(Q.T)
    return Q, w, Qd.t()[:N, :c] if c else None


def bounds(N, P, seed):
    """uneven even-aligned row offsets (the multi-GPU partition is by nnz)"""
    rng = np.random.default_rng(seed)
    cut = np.sort(rng.choice(np.arange(1, N // 2), P - 1, replace=False)) * 2 if P > 1 else np.array([], int)
    return np.concatenate([[0], cut, [N]]).astype(np.int64)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("N,c", [(10007 + 1, 37), (40000, 300), (4096, 64), (70000, 129), (20000, 0), (4096, 1),
                                 (333 + 1, 5), (65536, 200)])
def test_peer_cgs2_emulated(S, H, P, N, c):
    Q, w, Qv = problem(N, c, N * 31 + c)
    r0 = bounds(N, P, N + P)
    wg, betas = S.cgs2_peer_emulate(H, Qv, dev(w), r0)
    w_or = O.cgs2(Q, w) if c else w.copy()
    nor = O.norm2(w_or)
    assert np.all(betas == betas[0]), betas  # every rank formed the same sums
    assert abs(betas[0] - nor) <= 1e-12 * np.linalg.norm(w)
    assert np.abs(wg.cpu().numpy() - w_or / nor).max() <= 1e-12 * np.linalg.norm(w) / nor


@pytest.mark.parametrize("N,c", [(10008, 37), (40000, 300), (70000, 129), (20000, 0)])
def test_peer_one_rank_bitwise_equals_streaming_kernel(S, N, c):
    Q, w, Qv = problem(N, c, N + c)
    h = S.Handle()
    h.set_policy(cgs2="stream")
    ws, nrm = S.cgs2(h, Qv, dev(w))
    wp, betas = S.cgs2_peer_emulate(h, Qv, dev(w), np.array([0, N]))
    h.close()
    assert betas[0] == nrm.item()
    assert torch.equal(ws, wp)


def test_peer_breakdown_agrees(S, H):
    """w in span(Q): every rank sees beta = 0 (reading Q7) and leaves w unnormalized."""
    N, c, P = 8192, 20, 3
    rng = np.random.default_rng(5)
    Q = np.linalg.qr(rng.standard_normal((N, c)))[0]
    w = Q @ rng.standard_normal(c)
    ld = -(-N // 32) * 32
    Qd = torch.zeros((c, ld), dtype=torch.float64, device="cuda")
    Qd[:, :N] = dev(Q.T)
    _, betas = S.cgs2_peer_emulate(H, Qd.t()[:N, :], dev(w), bounds(N, P, 1))
    assert np.all(betas == 0.0)


def test_peer_emulate_rejects_bad_partition(S, H):
    Q, w, Qv = problem(1000, 4, 1)
    with pytest.raises(S.SvdscError):
        S.cgs2_peer_emulate(H, Qv, dev(w), np.array([0, 501, 1000]))  # odd offset
    with pytest.raises(S.SvdscError):
        S.cgs2_peer_emulate(H, Qv, dev(w), np.array([0, 0, 1000]))  # empty rank


@pytest.mark.parametrize("cid,scale", [(1, 1), (3, 20)])
def test_solver_peer_path_one_rank(S, cid, scale):
    """The solver's multi-GPU CGS2 path on a one-rank NCCL communicator
    (SVDSC_POLICY_CGS2 = 6: mailbox setup, per-solve reset, device-resident
    sequence under graph replay, the deferred second update of reading G5)
    bitwise equal to the same solve with the single-GPU streaming kernel (the
    one-rank exchange sums the same values in the same order), and within the
    north_star tolerances of the oracle."""
    wl = W.config(cid, scale=scale)
    r_or = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    res = []
    for pol in ("stream", "peer"):
        h = S.Handle()
        h.comm_init(1, 0, S.comm_unique_id())  # a unique id serves one communicator
        h.set_policy(cgs2=pol)
        M = S.Matrix.from_host(h, wl.A)
        for _ in range(2):  # the second solve re-uses the mailbox (per-solve reset)
            r = S.svds_c(M, wl.k, tol=wl.tol, t=wl.t, maxit=wl.maxit, v0=torch.from_numpy(wl.v0).cuda(),
                         fixed_passes=r_or.passes)
        res.append((r.S.cpu().numpy(), r.U.cpu().numpy(), r.V.cpu().numpy()))
        M.close()
        h.close()
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)
    assert np.abs(res[1][0] - r_or.S).max() <= 1e-10 * r_or.S[0]
    assert sin_max_angle(res[1][2], r_or.V) <= 1e-8
