"""World-size-2 CPU tests (gloo) of the row-partitioned multi-GPU path
(SURVEY.md 8(e)).  The NCCL kernels cannot run here, so this pins the pieces
that are host logic or pure math:

  * the C++ partitioner + rank-local slicing used by bench.py cover A exactly,
    and bench.py's rank-local generation (workloads.degrees + config(r0, r1):
    every rank generates only its rows) equals the rows of the global matrix;
  * the NCCL unique-id bootstrap broadcast (svdsc_comm_unique_id -> gloo);
  * the collective schedule the C++ driver issues per Lanczos step -- reduce-
    scatter of the partial A^T u, all-gather of v, all-reduces of the CGS2
    coefficients and squared norms, Pythagorean beta -- executed here with
    numpy + gloo collectives on 2 ranks reproduces the single-process oracle's
    alpha/beta sequence.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slices(n, P):
    n_pad = -(-n // P) * P
    ns = n_pad // P
    return n_pad, ns


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from paper_2405_18966_b200 import svdsc as S

        out = {}
        # --- bootstrap: rank 0's unique id reaches every rank unchanged
        try:
            uid = [S.comm_unique_id() if rank == 0 else None]
        except Exception:
            uid = [b"x" * 128 if rank == 0 else None]  # NCCL not loadable: still test the broadcast
        dist.broadcast_object_list(uid, src=0)
        out["uid_len"] = len(uid[0])

        # --- partition (the product's host partitioner) and rank-local rows
        wl = W.config(1, scale=2)
        A = wl.A
        b = S.partition_rows(A.row_ptr, (wl.k + wl.t) // 2, world)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        rp = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
        col = A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]]
        val = A.values[A.row_ptr[r0]:A.row_ptr[r1]]
        out["rows"] = (r0, r1)
        D = A.to_dense()
        Dl = np.zeros((r1 - r0, A.n))
        rows = np.repeat(np.arange(r1 - r0), np.diff(rp))
        np.add.at(Dl, (rows, col.astype(np.int64)), val)
        out["local_ok"] = bool(np.array_equal(Dl, D[r0:r1]))

        # --- bench.py --gpus N: rank-local generation of a power-law config
        deg = W.degrees(4, scale=100)
        rpg = np.zeros(deg.size + 1, dtype=np.int64)
        rpg[1:] = np.cumsum(deg)
        bb = S.partition_rows(rpg, 200, world)
        g0, g1 = int(bb[rank]), int(bb[rank + 1])
        loc = W.config(4, scale=100, r0=g0, r1=g1).A
        glob = W.config(4, scale=100).A
        out["gen_rows"] = (g0, g1, int(bb[-1]))
        out["gen_ok"] = bool(np.array_equal(loc.row_ptr, glob.row_ptr[g0:g1 + 1] - glob.row_ptr[g0]) and
                             np.array_equal(loc.col_idx, glob.col_idx[glob.row_ptr[g0]:glob.row_ptr[g1]]) and
                             np.array_equal(loc.values, glob.values[glob.row_ptr[g0]:glob.row_ptr[g1]]))

        # --- the per-step collective schedule of the C++ driver (P > 1)
        n, m_loc = A.n, r1 - r0
        n_pad, ns = _slices(n, world)
        v0 = np.zeros(n_pad)
        v0[:n] = wl.v0
        t = 12

        def allreduce(x):
            tt = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(tt)
            return tt.numpy()

        def allgather(x):
            parts = [torch.zeros(ns, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(x)))
            return np.concatenate([p.numpy() for p in parts])

        def reduce_scatter(y):  # gloo has no reduce_scatter: all-reduce, keep own slice
            return allreduce(y)[rank * ns:(rank + 1) * ns]

        def cgs2_norm(Q, wv):
            """h1 = AR(Q^T w); w' = w - Q h1; [h2; ||w'||^2] = AR(.); beta^2 = ||w'||^2 - ||h2||^2."""
            if Q.shape[1] == 0:
                nrm = allreduce(np.array([wv @ wv]))[0]
                return wv, np.sqrt(nrm)
            h1 = allreduce(Q.T @ wv)
            wp = wv - Q @ h1
            red = allreduce(np.concatenate([Q.T @ wp, [wp @ wp]]))
            h2, nrmp = red[:-1], red[-1]
            wpp = wp - Q @ h2
            beta2 = nrmp - h2 @ h2
            if not beta2 > 0.5 * nrmp:  # explicit norm (the pass-end repair, reading G3)
                beta2 = allreduce(np.array([wpp @ wpp]))[0]
            return wpp, np.sqrt(beta2)

        Vs = np.zeros((ns, t + 1))
        Ul = np.zeros((m_loc, t + 1))
        vs = v0[rank * ns:(rank + 1) * ns]
        nv = np.sqrt(allreduce(np.array([vs @ vs]))[0])
        Vs[:, 0] = vs / nv
        z = Dl @ allgather(Vs[:, 0])[:n]
        z, a = cgs2_norm(Ul[:, :0], z)
        Ul[:, 0] = z / a
        alphas, betas = [a], []
        for i in range(1, t + 1):
            y = np.zeros(n_pad)
            y[:n] = Dl.T @ Ul[:, i - 1]
            w = reduce_scatter(y) - alphas[-1] * Vs[:, i - 1]
            w, bta = cgs2_norm(Vs[:, :i], w)
            Vs[:, i] = w / bta
            betas.append(bta)
            if i < t:
                z = Dl @ allgather(Vs[:, i])[:n] - bta * Ul[:, i - 1]
                z, a = cgs2_norm(Ul[:, :i], z)
                Ul[:, i] = z / a
                alphas.append(a)
        out["alphas"] = alphas
        out["betas"] = betas
        q.put((rank, out))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    from paper_2405_18966_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return res


def test_bootstrap_broadcast(results):
    assert results[0]["uid_len"] == results[1]["uid_len"] == 128


def test_partition_covers_rows(results):
    import workloads as W
    wl = W.config(1, scale=2)
    (a0, a1), (b0, b1) = results[0]["rows"], results[1]["rows"]
    assert a0 == 0 and a1 == b0 and b1 == wl.A.m
    assert results[0]["local_ok"] and results[1]["local_ok"]


def test_rank_local_generation(results):
    (a0, a1, m), (b0, b1, m2) = results[0]["gen_rows"], results[1]["gen_rows"]
    assert a0 == 0 and a1 == b0 and b1 == m == m2
    assert results[0]["gen_ok"] and results[1]["gen_ok"]


def test_distributed_schedule_matches_oracle(results):
    import oracle as O
    import workloads as W
    wl = W.config(1, scale=2)
    t = 12
    _, _, T, _ = O.lbp(wl.A, t, wl.v0)
    al, be = np.diag(T)[:t], np.diag(T, 1)[:t]
    for r in (0, 1):  # every rank holds the same (all-reduced) alpha/beta
        assert np.allclose(results[r]["alphas"], al, rtol=1e-12, atol=0)
        assert np.allclose(results[r]["betas"], be, rtol=1e-12, atol=0)
    assert results[0]["alphas"] == results[1]["alphas"]
