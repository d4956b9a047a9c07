#!/usr/bin/env python
"""Benchmark of the svds-C hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C] [--impl ours|reference]

A "step" is one full svds-C solve (Alg. 2: every SURVEY.md 8(a) row -- the
Lanczos steps, the small SVD, the restarts and the final assembly) on the
workload's synthetic input, which is resident in HBM before timing starts.
  value        Lanczos steps per second of the whole job (steps of all timed
               solves / max-over-ranks device time)
  ms_per_step  time-to-k-triplets of one solve (ms)
  roofline     dominant kernel family by device time (the fused CGS2
               re-orthogonalization on sparse inputs, the A / A^T products on
               dense ones): algorithmic bytes per launch over
               its CUDA-event-timed average duration inside the timed region,
               against MEASURED_PEAKS.json hbm_gbs; `traffic` from the committed
               ncu capture (profiles/traffic.json)
  e2e          same metric through the C-ABI host-buffer entry point
               (svdsc_solve_host_*), H2D of A and v0 and D2H of S, U, V, resid
               inside the timed region
  spmv_vs_gather_ceiling  (sparse, N = 1) each product (10 back-to-back
               svdsc_op_matvec calls) against the live ceiling of a kernel
               doing only its memory operations, timed the same way right
               after (index + value streams and one random 8-byte gather per
               nonzero, tools/gather_bw.cu): random gathers are bound by L1
               wavefronts / L2 sectors, not HBM
  cpu_baseline the CPU oracle (oracle/oracle.c, 1 thread pinned to one core):
               per-step cost t(i) = a + b i fitted on two bounded samples of
               the first Lanczos steps, extrapolated to the GPU solve's step
               schedule (labelled "extrapolated")
The default workload is BASELINE.json configs[3], the largest config that fits
one GPU (power-law 4,000,000 x 2,000,000, ~150M nnz, k = 100): A is 1.8 GB per
pass, far larger than the 126 MB L2, so no flush is needed between solves.
--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL); every rank generates only its own rows.

--impl reference times the CPU oracle as it stands (the reference arm of this
tier), 1 thread on one pinned core, rank 0 only: each step is one Lanczos step
of the same workload at the restart passes' average basis size.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lanczos steps/s & time-to-k triplets; HBM GB/s vs 8 TB/s peak, 1/2/4/8 GPUs"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc, self.th = index, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=5)
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def gather_ceiling(nnz, n):
    """Memory-side ceiling of a random-column CSR SpMV of this size, measured
    live by tools/gather_bw (the index + value streams and one 8-byte x gather
    per nonzero, nothing else): the best rate over its gather
    kernels, in nonzeros per second.  None if the tool is missing."""
    exe = os.path.join(ROOT, "tools", "gather_bw")
    src = exe + ".cu"
    try:
        if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
            subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", src, "-o", exe],
                                  stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        out = subprocess.run([exe, str(int(nnz)), str(int(n))], capture_output=True, text=True, timeout=120).stdout
        rows = [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]
        best = min((r for r in rows if r["kernel"] in ("gather", "gnc")), key=lambda r: r["us"])
        return {"gnnz_per_s": best["gnnz_per_s"], "us": best["us"], "kernel": best["kernel"],
                "ctas_per_sm": best["ctas_per_sm"]}
    except Exception:
        return None


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class PinnedCore:
    """Pin this process to one core while the single-threaded oracle runs."""

    def __enter__(self):
        self.old = None
        try:
            self.old = os.sched_getaffinity(0)
            self.core = min(self.old)
            os.sched_setaffinity(0, {self.core})
        except Exception:
            self.core = None
        return self

    def __exit__(self, *a):
        if self.old is not None:
            os.sched_setaffinity(0, self.old)


def cpu_fit(wl, seconds_target=15.0):
    """Time the oracle as it stands (1 thread, one pinned core) and fit the cost
    of Lanczos step i as t(i) = a + b i:
      b: the oracle's CGS2 (or_cgs2) of one U-side and one V-side vector against
         a c-column basis block (synthetic, the workload's row counts), / c;
      a: the first s Lanczos steps of LBP on the workload (its products and
         norms), minus their CGS2 share b * s(s+1)/2, / s."""
    import numpy as np

    import oracle as O
    rng = np.random.default_rng(0)
    with PinnedCore() as pc:
        t0 = time.perf_counter()
        O.lbp(wl.A, 2, wl.v0)
        probe = max(time.perf_counter() - t0, 1e-4) / 2.0
        s = int(max(2, min(wl.t, 0.4 * seconds_target / probe)))
        t0 = time.perf_counter()
        O.lbp(wl.A, s, wl.v0)
        t_lbp = time.perf_counter() - t0
        # CGS2 per basis column, both sides (bounded: c columns of each side)
        c = max(2, min(wl.t, 64, int(2e9 // (8 * (wl.A.m + wl.A.n)))))  # <= 2 GB of host basis
        t_cgs = 0.0
        for N in (wl.A.m, wl.A.n):
            Q = np.asfortranarray(rng.standard_normal((N, c)))
            w = rng.standard_normal(N)
            t0 = time.perf_counter()
            O.cgs2(Q, w)
            t_cgs += time.perf_counter() - t0
            del Q
    b = t_cgs / c
    a = max(0.0, (t_lbp - b * s * (s + 1) / 2) / s)
    return {"a": float(a), "b": float(b), "s": s, "c": c, "t_lbp": t_lbp, "t_cgs": t_cgs,
            "core": pc.core, "sample_seconds": t_lbp + t_cgs}


def step_schedule(k, t, passes):
    """Basis sizes i of the Lanczos steps of a solve: 1..t, then k+1..t per restart."""
    return list(range(1, t + 1)) + list(range(k + 1, t + 1)) * max(0, passes - 1)


def relaunch_distributed(args_list, n):
    """--gpus N without torchrun: one process per GPU via torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + args_list
    return subprocess.call(cmd)


def workload_config(name, m, n, nnz, k, t, tol, maxit, dense, world, reorth):
    """The `config` object of the bench line: names the workload only (nothing
    measured, which goes to `run`), so both arms (this library and --impl
    reference) print the same dict for the same command line."""
    mb = (8 * m * n if dense else 12 * nnz) >> 20
    bases_mb = (8 * (m + n) * (t + 1)) >> 20
    ws_mb = (1 if dense else 2) * mb + bases_mb  # A (+ its CSC copy) and the Lanczos bases U, V at i = t
    if ws_mb > 126:
        l2 = (f"inputs larger than L2 (A = {mb} MB per pass, bases {bases_mb} MB at i = t; "
              f"working set {ws_mb} MB vs 126 MB of L2): no flush")
    else:
        l2 = (f"working set {ws_mb} MB is L2-resident by design (SURVEY 8(d): the latency-bound parity config; "
              "every step of the iteration re-reads A and the bases, so no flush between steps; "
              "its HBM fraction is not meaningful)")
    return {"workload": name, "m": int(m), "n": int(n), "nnz": int(nnz), "k": int(k), "t": int(t),
            "tol": tol, "maxit": int(maxit), "l2": l2,
            "parallelism": f"rows{world}" if world > 1 else "single",
            "reorth": ("full CGS2 every half-step (PAPER.md:121)" if reorth == 2 else
                       "partial (omega recurrence, DESIGN.md Q20; not the paper's method; "
                       "step_bytes_model still counts every half-step's CGS2)")}


def run_loopback(args):
    """--comm loopback: N ranks as threads of this process (svdsc_group_*), each
    with its own handle, stream, rank-local rows and device (rank % visible).
    Same workload recipe, partition and max-over-ranks timing as the NCCL path;
    the collectives synchronize on the host, so the number is not a scaling
    measurement (the line says so)."""
    import numpy as np
    import torch

    import workloads as W
    from paper_2405_18966_b200 import build as B
    from paper_2405_18966_b200 import svdsc as S
    B.build()
    P, cid = args.gpus, args.workload
    ndev = max(1, torch.cuda.device_count())
    deg = W.degrees(cid)
    if deg is not None:
        rp = np.zeros(deg.size + 1, dtype=np.int64)
        rp[1:] = np.cumsum(deg)
        kt = {3: (100, 300), 4: (100, 300), 5: (200, 600)}[cid]
        bounds = S.partition_rows(rp, (kt[0] + kt[1]) // 2, P)
        m_global, nnz_global, full = int(deg.size), int(rp[-1]), None
    else:
        full = W.config(cid)
        m_global, nnz_global = full.A.m, full.A.nnz
        bounds = (S.partition_rows(full.A.row_ptr, (full.k + full.t) // 2, P) if full.A.kind == "csr"
                  else np.linspace(0, full.A.m, P + 1).astype(np.int64))
    g = S.Group(P)
    res = [None] * P
    barrier = threading.Barrier(P)

    def rank_main(r):
        try:
            dev = r % ndev
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream(device=dev)
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            if full is None:
                wl = W.config(cid, r0=r0, r1=r1)
                Al = wl.A
            else:
                wl = full
                A = full.A
                if A.kind == "csr":
                    Al = W.Matrix("csr", r1 - r0, A.n, row_ptr=A.row_ptr[r0:r1 + 1] - A.row_ptr[r0],
                                  col_idx=A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]],
                                  values=A.values[A.row_ptr[r0]:A.row_ptr[r1]])
                else:
                    Al = W.dense_matrix(np.ascontiguousarray(A.dense[r0:r1]))
            with torch.cuda.stream(st):
                h = S.Handle(st)
                h.comm_init_group(g, r)
                M = S.Matrix.from_host(h, Al, row_offset=r0, m_global=m_global)
                v0 = torch.from_numpy(wl.v0).cuda()
                ws = torch.empty(S.workspace_size(M, wl.k, t=wl.t), dtype=torch.uint8, device="cuda")

                def solve():
                    return S.svds_c(M, wl.k, tol=wl.tol, maxit=wl.maxit, t=wl.t, v0=v0, workspace=ws)

                for _ in range(args.warmup):
                    solve()
                st.synchronize()
                barrier.wait()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                steps, passes = 0, []
                for _ in range(args.steps):
                    out = solve()
                    steps += out.info["steps"]
                    passes.append(out.info["passes"])
                e1.record(st)
                st.synchronize()
                res[r] = (e0.elapsed_time(e1), steps, passes, out.S.cpu().numpy(), wl.name, wl.k, wl.t, Al.n)
        except Exception as e:  # noqa: BLE001
            res[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t_ in th:
        t_.start()
    for t_ in th:
        t_.join()
    g.close()
    for x in res:
        if isinstance(x, Exception):
            raise x
    ms = max(x[0] for x in res)
    _, steps, passes, s0, name, k, t, n = res[0]
    same = all(np.array_equal(x[3], s0) for x in res)
    print(json.dumps({
        "metric": METRIC, "value": steps / (ms / 1e3), "unit": "steps/s", "n_gpus": P, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "comm": f"loopback: {P} ranks as threads on {min(P, ndev)} GPU(s), host-synchronized collectives "
                "(a test of the multi-rank path, not a scaling measurement)",
        "config": {"workload": name, "m": m_global, "n": n, "nnz": nnz_global, "k": k, "t": t,
                   "passes_per_solve": passes, "parallelism": f"rows{P}",
                   "rows_per_rank": [int(bounds[r + 1] - bounds[r]) for r in range(P)]},
        "sigma_identical_on_all_ranks": same, "sigma_1": float(s0[0]),
        "e2e": None,  # (a host-logic harness: no end-to-end measurement)
    }), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", type=int, default=4, help="BASELINE.json config id (1-based)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true", help="skip the live SpMV gather-ceiling measurement")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-rows", action="store_true",
                    help="measure e2e the multi-GPU way (each rank copies its rows in and U/S/V out around "
                         "svdsc_matrix_csr + svdsc_solve) even on one GPU (the default for --gpus > 1)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "loopback"],
                    help="nccl: one process per GPU (the product path); loopback: --gpus N ranks as threads "
                         "of this process on the visible GPUs (round robin), host-synchronized collectives "
                         "-- exercises the multi-rank path on one GPU, not a scaling measurement")
    ap.add_argument("--reorth", type=int, default=2, choices=[1, 2],
                    help="2: full CGS2 every half-step (the paper's method, the headline); "
                         "1: partial re-orthogonalization (DESIGN.md Q20, SURVEY 8(f4)), an extra line")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and args.comm == "loopback":
        return run_loopback(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(sys.argv[1:], args.gpus)

    import numpy as np
    import workloads as W

    if args.impl == "reference":
        if rank != 0:
            return 0
        wl = W.config(args.workload)
        # reference arm = the CPU oracle as it stands, 1 thread on one pinned core.
        # One timed "step" = one Lanczos step of this workload at the restart
        # passes' average basis size i_r = (k + 1 + t) / 2: the
        # oracle's A v and A^T u (or_spmv / or_spmv_t, or the dense GEMVs) and its
        # CGS2 of an m- and an n-vector against i_r-column basis blocks
        # (synthetic Gaussian blocks: the cost does not depend on their values)
        import oracle as O
        O.lib()
        A = wl.A
        i_r = (wl.k + 1 + wl.t) // 2
        rng = np.random.default_rng(7)
        QU = np.asfortranarray(rng.standard_normal((A.m, i_r)))
        QV = np.asfortranarray(rng.standard_normal((A.n, i_r)))
        x = np.ascontiguousarray(wl.v0)
        u = rng.standard_normal(A.m)
        times = []
        with PinnedCore() as pc:
            for it in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                z = O.spmv(A, x)
                w = O.spmv_t(A, u)
                O.cgs2(QU, z)
                O.cgs2(QV, w)
                dt = time.perf_counter() - t0
                if it >= args.warmup:
                    times.append(dt)
        val = len(times) / sum(times)
        line = {
            "impl": "reference", "metric": METRIC, "value": val, "unit": "steps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(wl.name, A.m, A.n, A.nnz, wl.k, wl.t, wl.tol, wl.maxit,
                                      A.kind == "dense", args.gpus, args.reorth),
            "cpu_baseline": {"value": val, "unit": "steps/s", "cores": 1, "kind": "oracle",
                             "sample": f"each step = one Lanczos step of {wl.name} at basis size i_r = {i_r} "
                                       f"(the restart passes' average): the oracle's A v, A^T u and CGS2 of "
                                       f"an m- and an n-vector against {i_r}-column blocks; plain C -O2, "
                                       f"1 thread pinned to core {pc.core}", **host_info()},
            "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    from paper_2405_18966_b200 import build as B
    from paper_2405_18966_b200 import svdsc as S

    B.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- workload: rank-local rows of A (row partition) ----
    cid = args.workload
    deg = W.degrees(cid) if world > 1 else None
    if world > 1 and deg is not None:
        # every rank generates only its rows (counter-based per-row streams)
        rp = np.zeros(deg.size + 1, dtype=np.int64)
        rp[1:] = np.cumsum(deg)
        kt = {3: (100, 300), 4: (100, 300), 5: (200, 600)}[cid]  # (k, t) of configs 3-5
        bounds = S.partition_rows(rp, (kt[0] + kt[1]) // 2, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        wl_full = W.config(cid, r0=r0, r1=r1)
        Al = wl_full.A
        m_global = int(deg.size)
        nnz_global = int(rp[-1])
    else:
        wl_full = W.config(cid)
        A = wl_full.A
        m_global, nnz_global = A.m, A.nnz
        if world > 1:
            bounds = np.linspace(0, A.m, world + 1).astype(np.int64)
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            if A.kind == "csr":
                rpl = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
                Al = W.Matrix("csr", r1 - r0, A.n, row_ptr=rpl, col_idx=A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]],
                              values=A.values[A.row_ptr[r0]:A.row_ptr[r1]])
            else:
                Al = W.dense_matrix(A.dense[r0:r1])
        else:
            r0, r1, Al = 0, A.m, A
    n_cols = Al.n

    stream = torch.cuda.current_stream()
    H = S.Handle(stream)
    if world > 1:
        uid = [S.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        H.comm_init(world, rank, uid[0])
        H.comm_check()  # fail fast on a broken NCCL / NVLink setup (one small collective of each kind)
    M = S.Matrix.from_host(H, Al, device=dev, row_offset=r0, m_global=m_global)
    v0 = torch.from_numpy(wl_full.v0).to(dev)
    k, t = wl_full.k, wl_full.t
    ws = torch.empty(S.workspace_size(M, k, t=t), dtype=torch.uint8, device=dev)

    def solve():
        return S.svds_c(M, k, tol=wl_full.tol, maxit=wl_full.maxit, t=t, v0=v0, workspace=ws, reorth=args.reorth)

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    # per-family breakdown from one untimed, fully profiled solve; it also picks
    # the dominant kernel family whose CUDA events are kept in the timed region
    # (one family only: every event record between kernels costs a few us)
    H.profile(True)
    solve()
    torch.cuda.synchronize()
    prof_all = H.profile_read()
    H.profile(False)
    # (reorth = 1: the CGS2 byte model assumes every half-step re-orthogonalizes,
    # so the roofline line is taken on the products)
    fam = max(("Av", "ATu", "cgs2_fused") if args.reorth == 2 else ("Av", "ATu"), key=lambda f: prof_all[f][0])

    # ---- timed region (no event records between kernels: the library replays
    # each restart pass as one CUDA graph) ----
    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    steps_total, launches, passes, res, bytes_model, bytes_reorth = 0, 0, [], None, 0, 0
    for _ in range(args.steps):
        res = solve()
        steps_total += res.info["steps"]
        launches += res.info["launches"]
        passes.append(res.info["passes"])
        bytes_model += res.info["bytes_model"]
        bytes_reorth += res.info["bytes_reorth"]
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = steps_total / (ms / 1e3)

    # ---- roofline region: the same solves again, with CUDA events (library
    # stream) around the dominant kernel family only; launches are eager here
    # (event records inside a graph capture are not supported by this build) ----
    H.profile(True, families=(fam,))
    torch.cuda.synchronize()
    e0r, e1r = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0r.record(stream)
    rf_bytes_reorth = 0
    for _ in range(args.steps):
        rf_bytes_reorth += solve().info["bytes_reorth"]
    e1r.record(stream)
    torch.cuda.synchronize()
    ms_roof = e0r.elapsed_time(e1r)
    prof = H.profile_read()
    H.profile(False)

    # ---- roofline of the dominant kernel family (by device time in the timed region) ----
    peak, peak_src = load_peaks()
    f_ms, f_calls = prof[fam]
    bA = Al.bytes_one_pass() if Al.kind == "dense" else 12 * Al.nnz + 4 * (Al.m + 1)
    bAt = Al.bytes_one_pass() if Al.kind == "dense" else 12 * Al.nnz + 4 * (Al.n + 1)
    if fam == "cgs2_fused":
        # algorithmic CGS2 bytes, 8 N (3 i + 5) per re-orthogonalization (SURVEY.md
        # 8(d)), counted by the library per call (svdsc_info.bytes_reorth)
        bytes_per_launch = rf_bytes_reorth / max(f_calls, 1)
    else:
        bytes_per_launch = bA if fam == "Av" else bAt
    traffic, traffic_src = None, None
    try:  # DRAM bytes per launch of this kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        ent = tj.get(wl_full.name.split("_div")[0], {}).get(fam)
        if ent and world == 1:
            # the capture's DRAM/algorithmic ratio applied to this launch size
            traffic = ent["dram_bytes"] / ent["algorithmic_bytes"] * bytes_per_launch
            traffic_src = ent
    except Exception:
        traffic = None
    achieved = bytes_per_launch / (f_ms / f_calls / 1e3) / 1e9 if f_calls else None
    step_bytes = res.info["bytes_model"] / max(res.info["steps"], 1)
    total_prof = sum(v[0] for v in prof_all.values())

    # ---- sparse products against their own ceiling: random 8-byte gathers are
    # bound by L1 wavefronts / L2 sectors, not HBM, so each SpMV
    # family is also reported against the live gather ceiling of its shape ----
    spmv_ceiling = None
    if Al.kind == "csr" and world == 1 and not args.no_ceiling:
        # both sides measured the same way, back to back: 10 products through
        # svdsc_op_matvec (the solver's kernel for this operand) between CUDA
        # events on the library stream, then the ceiling kernels (10 launches each)
        spmv_ceiling = {}
        for f, trans, ncol_x in (("Av", False, Al.n), ("ATu", True, Al.m)):
            xin = torch.randn(ncol_x, dtype=torch.float64, device=dev)
            S.matvec(M, xin, trans=trans)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(10):
                S.matvec(M, xin, trans=trans)
            a1.record(stream)
            torch.cuda.synchronize()
            us = 1e3 * a0.elapsed_time(a1) / 10
            ceil = gather_ceiling(Al.nnz, ncol_x)
            f_ms_all, calls = prof_all[f]
            ent = {"isolated_us": us, "gnnz_per_s": Al.nnz / (us * 1e3),
                   "alg_GBps": (bA if f == "Av" else bAt) / (us * 1e3), "ceiling": ceil,
                   "in_solve_us": 1e3 * f_ms_all / calls if calls else None}
            if ceil:
                ent["frac_of_ceiling"] = ceil["us"] / us
            spmv_ceiling[f] = ent
            del xin

    # ---- end to end, multi-GPU: every rank copies its rows of A (pinned host)
    # in, analyses and solves through the device-buffer C ABI (svdsc_matrix_*
    # + svdsc_solve, the calls a multi-GPU user makes) and copies S, its rows of
    # U and V out; timed per rank on its stream between barriers, max over ranks
    e2e = None
    if not args.no_e2e and (world > 1 or args.e2e_rows):
        if Al.kind == "dense":
            hA = torch.from_numpy(np.asfortranarray(Al.dense).T.copy()).pin_memory()  # (n, m): column-major A
            h2d_r = 8 * Al.m * Al.n
        else:
            hrp = torch.from_numpy(np.ascontiguousarray(Al.row_ptr, np.int64)).pin_memory()
            hci = torch.from_numpy(np.ascontiguousarray(Al.col_idx, np.int32)).pin_memory()
            hva = torch.from_numpy(np.ascontiguousarray(Al.values, np.float64)).pin_memory()
            h2d_r = 8 * (Al.m + 1) + 12 * Al.nnz
        hv0 = torch.from_numpy(wl_full.v0).pin_memory()
        h2d_r += 8 * wl_full.v0.size
        hS = torch.empty(k, dtype=torch.float64).pin_memory()
        hU = torch.empty((k, Al.m), dtype=torch.float64).pin_memory()
        hV = torch.empty((k, n_cols), dtype=torch.float64).pin_memory()
        d2h_r = 8 * (k + Al.m * k + n_cols * k)

        def e2e_solve():
            if Al.kind == "dense":
                Md = S.Matrix.dense(H, hA.to(dev, non_blocking=True).t(), row_offset=r0, m_global=m_global)
            else:
                Md = S.Matrix.csr(H, hrp.to(dev, non_blocking=True), hci.to(dev, non_blocking=True),
                                  hva.to(dev, non_blocking=True), n_cols, row_offset=r0, m_global=m_global)
            r = S.svds_c(Md, k, tol=wl_full.tol, maxit=wl_full.maxit, t=t, v0=hv0.to(dev, non_blocking=True),
                         reorth=args.reorth)
            hS.copy_(r.S, non_blocking=True)
            hU.copy_(r.U.t(), non_blocking=True)
            hV.copy_(r.V.t(), non_blocking=True)
            torch.cuda.current_stream().synchronize()  # the host buffers are the result
            Md.close()
            return r.info["steps"]

        e2e_solve()  # warm
        e2e_steps, e2e_ms = 0, 0.0
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_steps += e2e_solve()
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms += e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([e2e_ms, float(h2d_r), float(d2h_r)], device=dev, dtype=torch.float64)
            mx = tt[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            e2e_ms, h2d, d2h = float(mx.item()), int(tt[1].item()), int(tt[2].item())
        else:
            h2d, d2h = h2d_r, d2h_r
        e2e = {"value": e2e_steps / (e2e_ms / 1e3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.e2e_steps,
               "note": "every rank: pinned host rows of A and v0 in, S and its rows of U / V out, matrix analysis "
                       "and solve through svdsc_matrix_* + svdsc_solve; bytes summed over the ranks, time = max "
                       "over the ranks"}
    # ---- end to end through the host-buffer C-ABI entry point ----
    if not args.no_e2e and world == 1 and not args.e2e_rows:
        e2e_steps, e2e_ms, h2d, d2h = 0, 0.0, 0, 0
        if Al.kind == "dense":
            hostA = torch.empty((Al.n, Al.m), dtype=torch.float64).pin_memory()
            hostA.copy_(torch.from_numpy(np.asfortranarray(Al.dense).T))
            Ahost = W.Matrix("dense", Al.m, Al.n, dense=hostA.numpy().T)
            h2d = 8 * Al.m * Al.n + 8 * Al.n
        else:
            Ahost = W.Matrix("csr", Al.m, Al.n,
                             row_ptr=torch.from_numpy(Al.row_ptr).pin_memory().numpy(),
                             col_idx=torch.from_numpy(Al.col_idx).pin_memory().numpy(),
                             values=torch.from_numpy(Al.values).pin_memory().numpy())
            h2d = 8 * (Al.m + 1) + 12 * Al.nnz + 8 * Al.n
        d2h = 8 * (k + Al.m * k + Al.n * k + k)
        v0h = torch.from_numpy(wl_full.v0).pin_memory().numpy()
        # pinned host outputs, as a user who cares about transfer speed passes them
        outh = tuple(torch.empty(sh, dtype=torch.float64).pin_memory().numpy()
                     for sh in ((k,), (k, Al.m), (k, Al.n), (k,)))
        S.svds_c_host(H, Ahost, k, tol=wl_full.tol, maxit=wl_full.maxit, t=t, v0=v0h, reorth=args.reorth,
                      out=outh)  # warm
        an = 0.0
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = S.svds_c_host(H, Ahost, k, tol=wl_full.tol, maxit=wl_full.maxit, t=t, v0=v0h, reorth=args.reorth,
                                out=outh)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms += e0.elapsed_time(e1)
            e2e_steps += out[5]["steps"]
            an += out[5]["seconds_analysis"]
        e2e = {"value": e2e_steps / (e2e_ms / 1e3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.e2e_steps,
               "analysis_ms_per_step": 1e3 * an / args.e2e_steps,
               "note": "pinned host buffers in and out; includes per-solve matrix analysis (validation" +
                       (", row bins, CSC build" if Al.kind == "csr" else "") + ")"}

    # ---- CPU oracle baseline (rank 0, N = 1 only) ----
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        fit = cpu_fit(wl_full, seconds_target=15.0)
        sched = step_schedule(k, t, passes[-1])
        t_solve = sum(fit["a"] + fit["b"] * i for i in sched)
        cpu = {"value": len(sched) / t_solve, "unit": "steps/s", "cores": 1, "kind": "oracle",
               "time_to_k_s": t_solve,
               "sample": (f"extrapolated: per-step cost t(i) = a + b i of the oracle on {wl_full.name}, "
                          f"b from its CGS2 of one U- and one V-side vector against a {fit['c']}-column basis "
                          f"block, a from its first {fit['s']} Lanczos steps (Alg. 1 + CGS2) minus their CGS2 "
                          f"share ({fit['sample_seconds']:.1f} s of plain C -O2, 1 thread pinned to core "
                          f"{fit['core']}): a = {fit['a']:.4g} s, b = {fit['b']:.4g} s per basis column, "
                          f"summed over the GPU solve's {len(sched)} steps ({passes[-1]} passes)"),
               **host_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(wl_full.name, m_global, n_cols, nnz_global, k, t, wl_full.tol, wl_full.maxit,
                                      Al.kind == "dense", world, args.reorth),
            "run": {"passes_per_solve": passes, "lanczos_steps_per_solve": steps_total // args.steps,
                    "time_to_k_ms": ms / args.steps, "rank0_rows": [r0, r1],
                    "step_hbm_gb_per_s": step_bytes * (steps_total / (ms / 1e3)) / 1e9,
                    "step_bytes_model": step_bytes},
            "roofline": {"bound": "hbm",
                         "kernel": ("fused CGS2 re-orthogonalization (the streaming kernel: 2 sweeps of U_i / V_i "
                                    "per half-step with the deferred second update, DESIGN.md G5)" if fam == "cgs2_fused"
                                    else f"{fam} product ({'gemv' if Al.kind == 'dense' else 'spmv'})"),
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "bytes_per_launch": bytes_per_launch, "avg_launch_us": 1e3 * f_ms / max(f_calls, 1),
                         "bytes_note": ("bytes the executed CGS2 moves, 8N(2i+5) (+8N forming the pending column) "
                                        "per deferred half-step; the paper's three-sweep CGS2 moves 8N(3i+5), ~1.5x "
                                        "these bytes for the same result" if fam == "cgs2_fused" else None),
                         "share_of_step": f_ms / ms_roof if ms_roof else None, "peak_source": peak_src,
                         "timing": "CUDA events around every launch of the family in a second timed region "
                                   "of the same solves (eager launches), right after the headline one"},
            "spmv_vs_gather_ceiling": spmv_ceiling,
            "breakdown_ms_one_solve": {f: round(v[0], 3) for f, v in prof_all.items() if v[1]},
            "breakdown_share": {f: round(v[0] / total_prof, 4) for f, v in prof_all.items() if v[1] and total_prof},
            "clocks": clk, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
