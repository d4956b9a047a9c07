"""Thin Python binding of libsvdsc.so (C ABI in include/svdsc.h).

Argument marshalling only: torch CUDA tensors are passed as raw device
pointers with the current CUDA stream; every step of the method runs in the
library's sm_100a kernels.  There is no CPU fallback: if the shared library is
missing this module raises at import of the first call.

Layouts: dense matrices and bases are column-major, i.e. a torch tensor of
shape (m, n) with stride (1, ld) (``colmajor(...)`` makes one).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsvdsc.so")
_lib = None

OK, NOT_CONVERGED = 0, 1
STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL",
          -5: "ESVD_NOCONV", -6: "ERANKDEF"}


class SvdscError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"svdsc {STATUS.get(status, status)}: {msg}")
        self.status = status


class Opts(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("tol", ctypes.c_double), ("t", ctypes.c_int32),
                ("maxit", ctypes.c_int32), ("seed", ctypes.c_uint64), ("v0", ctypes.c_void_p),
                ("fixed_passes", ctypes.c_int32), ("reorth", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int32), ("restarts", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("t_used", ctypes.c_int32),
                ("steps", ctypes.c_int64), ("matvecs", ctypes.c_int64),
                ("breakdowns", ctypes.c_int64), ("max_resid", ctypes.c_double),
                ("seconds_total", ctypes.c_double), ("launches", ctypes.c_int64),
                ("bytes_model", ctypes.c_int64), ("reorths", ctypes.c_int64),
                ("bytes_reorth", ctypes.c_int64), ("seconds_analysis", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PaperCsr(ctypes.Structure):
    """mat_csr of PAPER.md:293-299: 1-based cols, pointerB / pointerE (MKL LP64)."""
    _fields_ = [("nnz", ctypes.c_int64), ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64),
                ("values", ctypes.POINTER(ctypes.c_double)), ("cols", ctypes.POINTER(ctypes.c_int)),
                ("pointerB", ctypes.POINTER(ctypes.c_int)), ("pointerE", ctypes.POINTER(ctypes.c_int))]


class PaperMat(ctypes.Structure):
    """mat of PAPER.md:301-304: column-major nrows x ncols."""
    _fields_ = [("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64), ("d", ctypes.POINTER(ctypes.c_double))]


EXPORTS = ["svdsc_create", "svdsc_set_stream", "svdsc_destroy", "svdsc_last_error", "svdsc_version",
           "svdsc_matrix_csr", "svdsc_matrix_dense", "svdsc_matrix_destroy", "svdsc_workspace_size",
           "svdsc_solve", "svdsc_solve_host_csr", "svdsc_solve_host_dense", "svdsc_op_matvec",
           "svdsc_op_cgs2", "svdsc_op_cgs2_peer_emulate", "svdsc_op_small_svd", "svdsc_op_recombine", "svdsc_op_lbp",
           "svdsc_comm_unique_id", "svdsc_comm_init", "svdsc_partition_rows",
           "svdsc_profile_enable", "svdsc_profile_read", "svdsc_set_policy",
           "svdsc_group_create", "svdsc_group_destroy", "svdsc_comm_init_group", "svdsc_comm_check"]
# svdsc_set_policy keys / values (include/svdsc.h)
POLICY_SPMV, POLICY_CGS2, POLICY_SMALL_SVD, POLICY_DEFER = 0, 1, 2, 3
SPMV = {"auto": 0, "bins": 1, "seg": 2}
CGS2 = {"auto": 0, "split": 1, "qs": 2, "stream": 3, "tma": 4, "cluster": 5, "peer": 6, "phased": 7}
SMALL_SVD = {"auto": 0, "one_cta": 1, "register": 2, "block": 3}
DEFER = {"auto": 0, "off": 1}
PROF_FAMILIES = ["Av", "ATu", "cgs_p1", "cgs_p2", "cgs_p3", "normalize", "small_svd", "residuals",
                 "recombine", "restart_misc", "collectives", "cgs2_fused", "pro_decide"]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is missing: build it with `python -m paper_2405_18966_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(_SO)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.svdsc_create.argtypes = [ctypes.POINTER(P), P]
        L.svdsc_set_stream.argtypes = [P, P]
        L.svdsc_destroy.argtypes = [P]
        L.svdsc_destroy.restype = None
        L.svdsc_last_error.argtypes = [P]
        L.svdsc_last_error.restype = ctypes.c_char_p
        L.svdsc_version.restype = ctypes.c_char_p
        L.svdsc_matrix_csr.argtypes = [P, I64, I64, I64, P, P, P, I64, I64, ctypes.POINTER(P)]
        L.svdsc_matrix_dense.argtypes = [P, I64, I64, I64, P, I64, I64, ctypes.POINTER(P)]
        L.svdsc_matrix_destroy.argtypes = [P]
        L.svdsc_matrix_destroy.restype = None
        L.svdsc_workspace_size.argtypes = [P, ctypes.POINTER(Opts), ctypes.POINTER(ctypes.c_size_t)]
        L.svdsc_solve.argtypes = [P, ctypes.POINTER(Opts), P, ctypes.c_size_t, P, P, I64, P, I64, P,
                                  ctypes.POINTER(Info)]
        L.svdsc_solve_host_csr.argtypes = [P, I64, I64, I64, P, P, P, ctypes.POINTER(Opts), P, P, P, P,
                                           ctypes.POINTER(Info)]
        L.svdsc_solve_host_dense.argtypes = [P, I64, I64, P, ctypes.POINTER(Opts), P, P, P, P,
                                             ctypes.POINTER(Info)]
        L.svdsc_op_matvec.argtypes = [P, ctypes.c_int, P, P, P, P]
        L.svdsc_op_cgs2.argtypes = [P, I64, I64, P, I64, P, P]
        L.svdsc_op_cgs2_peer_emulate.argtypes = [P, I32, P, I64, P, I64, P, P]
        L.svdsc_op_small_svd.argtypes = [P, I32, P, P, P, P, ctypes.POINTER(I32)]
        L.svdsc_op_recombine.argtypes = [P, I64, I32, I32, P, I64, P, I32, P, I64]
        L.svdsc_op_lbp.argtypes = [P, ctypes.POINTER(Opts), I32, P, P, I64, P, I64, P,
                                   ctypes.POINTER(Info)]
        L.svdsc_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.svdsc_comm_init.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        L.svdsc_partition_rows.argtypes = [I64, P, I64, ctypes.c_int, P]
        L.svdsc_profile_enable.argtypes = [P, ctypes.c_int]
        L.svdsc_profile_read.argtypes = [P, P, P]
        L.svdsc_set_policy.argtypes = [P, I32, I32]
        L.svdsc_group_create.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        L.svdsc_group_destroy.argtypes = [P]
        L.svdsc_group_destroy.restype = None
        L.svdsc_comm_init_group.argtypes = [P, P, ctypes.c_int]
        L.svdsc_comm_check.argtypes = [P]
        # the paper's interface (include/svdsc_paper.h)
        PM, PC = ctypes.POINTER(PaperMat), ctypes.POINTER(PaperCsr)
        for f in ("svds_C", "svds_C_opt"):
            getattr(L, f).argtypes = [PC, PM, PM, PM, ctypes.c_int] + (
                [ctypes.c_double, ctypes.c_int, ctypes.c_int] if f.endswith("opt") else [])
        for f in ("svds_C_dense", "svds_C_dense_opt"):
            getattr(L, f).argtypes = [PM, PM, PM, PM, ctypes.c_int] + (
                [ctypes.c_double, ctypes.c_int, ctypes.c_int] if f.endswith("opt") else [])
        L.svdsc_mat_free.argtypes = [PM]
        L.svdsc_mat_free.restype = None
        L.svdsc_mat_csr_free.argtypes = [PC]
        L.svdsc_mat_csr_free.restype = None
        L.svdsc_paper_csr_to_csr.argtypes = [PC, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                             ctypes.POINTER(I64)]
        L.svdsc_read_mm.argtypes = [ctypes.c_char_p, PC, PM, ctypes.POINTER(ctypes.c_int)]
        L.svdsc_write_mm.argtypes = [ctypes.c_char_p, PC, PM]
        L.svdsc_paper_last_error.restype = ctypes.c_char_p
        for name in EXPORTS:
            f = getattr(L, name)
            if f.restype is ctypes.c_int:  # default
                f.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def colmajor(rows, cols, device="cuda", dtype=torch.float64):
    """Empty (rows, cols) tensor with column-major strides (1, rows)."""
    return torch.empty((cols, rows), device=device, dtype=dtype).t()


def _ld(t):
    assert t.dim() == 2 and t.stride(0) == 1, "expected a column-major 2-D tensor (stride(0) == 1)"
    return max(t.stride(1), t.shape[0])


class Handle:
    """svdsc_create on the current device and CUDA stream."""

    def __init__(self, stream=None):
        self.ptr = ctypes.c_void_p()
        s = (stream or torch.cuda.current_stream()).cuda_stream
        self._check(lib().svdsc_create(ctypes.byref(self.ptr), ctypes.c_void_p(s)))
        self.nranks, self.rank = 1, 0

    def _check(self, st):
        if st < 0:
            msg = lib().svdsc_last_error(self.ptr).decode() if self.ptr else ""
            raise SvdscError(st, msg)
        return st

    def set_stream(self, stream):
        self._check(lib().svdsc_set_stream(self.ptr, ctypes.c_void_p(stream.cuda_stream)))

    def comm_init(self, nranks, rank, uid: bytes):
        self._check(lib().svdsc_comm_init(self.ptr, nranks, rank, uid))
        self.nranks, self.rank = nranks, rank

    def comm_check(self):
        """Collective self-check of the communicator (svdsc_comm_check; every rank)."""
        self._check(lib().svdsc_comm_check(self.ptr))

    def comm_init_group(self, group: "Group", rank):
        """Join an in-process loopback group (svdsc_comm_init_group)."""
        self._check(lib().svdsc_comm_init_group(self.ptr, group.ptr, rank))
        self.nranks, self.rank = group.nranks, rank

    def set_policy(self, spmv=None, cgs2=None, small_svd=None, defer=None):
        """Force a kernel schedule (svdsc_set_policy); names from SPMV / CGS2 / SMALL_SVD / DEFER."""
        for key, table, v in ((POLICY_SPMV, SPMV, spmv), (POLICY_CGS2, CGS2, cgs2),
                              (POLICY_SMALL_SVD, SMALL_SVD, small_svd), (POLICY_DEFER, DEFER, defer)):
            if v is not None:
                self._check(lib().svdsc_set_policy(self.ptr, key, table[v] if isinstance(v, str) else int(v)))

    def profile(self, enable=True, families=None):
        """CUDA-event timing per operation family; `families`: names to record
        (None: all) -- fewer events inside a timed region."""
        v = int(bool(enable))
        if enable and families is not None:
            v = -sum(1 << PROF_FAMILIES.index(f) for f in families)
        self._check(lib().svdsc_profile_enable(self.ptr, v))

    def profile_read(self):
        ms = np.zeros(16)
        calls = np.zeros(16, dtype=np.int64)
        self._check(lib().svdsc_profile_read(self.ptr, ms.ctypes.data, calls.ctypes.data))
        return {name: (float(ms[i]), int(calls[i])) for i, name in enumerate(PROF_FAMILIES)}

    def close(self):
        if self.ptr:
            lib().svdsc_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """In-process loopback group of nranks ranks (svdsc_group_create)."""

    def __init__(self, nranks):
        self.ptr = ctypes.c_void_p()
        self.nranks = nranks
        st = lib().svdsc_group_create(nranks, ctypes.byref(self.ptr))
        if st < 0:
            raise SvdscError(st, "svdsc_group_create")

    def close(self):
        if self.ptr:
            lib().svdsc_group_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().svdsc_comm_unique_id(buf)
    if st < 0:
        raise SvdscError(st, "ncclGetUniqueId")
    return buf.raw


def partition_rows(row_ptr: np.ndarray, basis_cols: int, nparts: int) -> np.ndarray:
    """Host partitioner (svdsc_partition_rows): contiguous balanced row blocks."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    b = np.zeros(nparts + 1, dtype=np.int64)
    st = lib().svdsc_partition_rows(rp.size - 1, rp.ctypes.data, basis_cols, nparts, b.ctypes.data)
    if st < 0:
        raise SvdscError(st, "partition_rows")
    return b


class Matrix:
    """svdsc_matrix over caller-owned device arrays (kept alive here)."""

    def __init__(self, h: Handle, kind, m, n, keep, ptr, row_offset=0, m_global=None):
        self.h, self.kind, self.m, self.n, self._keep, self.ptr = h, kind, m, n, keep, ptr
        self.row_offset = row_offset
        self.m_global = m if m_global is None else m_global

    @classmethod
    def csr(cls, h: Handle, row_ptr, col_idx, values, ncols, row_offset=0, m_global=None):
        assert row_ptr.dtype == torch.int64 and col_idx.dtype == torch.int32 and values.dtype == torch.float64
        assert row_ptr.is_cuda and col_idx.is_cuda and values.is_cuda
        row_ptr, col_idx, values = row_ptr.contiguous(), col_idx.contiguous(), values.contiguous()
        m = row_ptr.numel() - 1
        mg = m if m_global is None else m_global
        p = ctypes.c_void_p()
        h._check(lib().svdsc_matrix_csr(h.ptr, m, ncols, values.numel(), _ptr(row_ptr), _ptr(col_idx),
                                        _ptr(values), row_offset, mg, ctypes.byref(p)))
        return cls(h, "csr", m, ncols, (row_ptr, col_idx, values), p, row_offset, mg)

    @classmethod
    def dense(cls, h: Handle, A, row_offset=0, m_global=None):
        assert A.dtype == torch.float64 and A.is_cuda
        m, n = A.shape
        mg = m if m_global is None else m_global
        p = ctypes.c_void_p()
        h._check(lib().svdsc_matrix_dense(h.ptr, m, n, _ld(A), _ptr(A), row_offset, mg, ctypes.byref(p)))
        return cls(h, "dense", m, n, (A,), p, row_offset, mg)

    @classmethod
    def from_host(cls, h: Handle, A, device="cuda", row_offset=0, m_global=None):
        """From a workloads.Matrix (host numpy) -> device copy + analysis."""
        if A.kind == "csr":
            rp = torch.from_numpy(np.ascontiguousarray(A.row_ptr, np.int64)).to(device)
            ci = torch.from_numpy(np.ascontiguousarray(A.col_idx, np.int32)).to(device)
            va = torch.from_numpy(np.ascontiguousarray(A.values, np.float64)).to(device)
            return cls.csr(h, rp, ci, va, A.n, row_offset, m_global)
        D = torch.from_numpy(np.asfortranarray(A.dense, np.float64).T.copy()).to(device).t()
        return cls.dense(h, D, row_offset, m_global)

    def close(self):
        if self.ptr:
            lib().svdsc_matrix_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _opts(k, tol, t, maxit, seed, v0, fixed_passes, reorth):
    return Opts(k=k, tol=tol, t=t or 0, maxit=maxit, seed=seed,
                v0=None if v0 is None else v0.data_ptr(), fixed_passes=fixed_passes, reorth=reorth)


@dataclass
class Result:
    S: torch.Tensor
    U: torch.Tensor
    V: torch.Tensor
    resid: torch.Tensor
    status: int
    info: dict


def svds_c(M: Matrix, k, tol=1e-10, maxit=100, t=None, seed=0, v0=None, fixed_passes=0, reorth=2,
           workspace=None) -> Result:
    """Alg. 2 of the paper: k largest singular triplets of M (svdsc_solve)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    if v0 is not None:
        v0 = v0.to(device=dev, dtype=torch.float64).contiguous()
    o = _opts(k, tol, t, maxit, seed, v0, fixed_passes, reorth)
    S = torch.empty(k, device=dev, dtype=torch.float64)
    U = colmajor(M.m, k, dev)
    V = colmajor(M.n, k, dev)
    R = torch.empty(k, device=dev, dtype=torch.float64)
    info = Info()
    ws, wsb = (None, 0) if workspace is None else (workspace, workspace.numel() * workspace.element_size())
    st = M.h._check(lib().svdsc_solve(M.ptr, ctypes.byref(o), _ptr(ws), wsb, _ptr(S), _ptr(U), max(M.m, 1),
                                      _ptr(V), M.n, _ptr(R), ctypes.byref(info)))
    return Result(S, U, V, R, st, info.as_dict())


def workspace_size(M: Matrix, k, t=None, tol=1e-10, maxit=100) -> int:
    o = _opts(k, tol, t, maxit, 0, None, 0, 2)
    n = ctypes.c_size_t()
    M.h._check(lib().svdsc_workspace_size(M.ptr, ctypes.byref(o), ctypes.byref(n)))
    return n.value


def svds_c_host(h: Handle, A, k, tol=1e-10, maxit=100, t=None, seed=0, v0=None, fixed_passes=0,
                reorth=2, out=None):
    """End-to-end with HOST buffers (svdsc_solve_host_*): numpy in, numpy out.
    out: optional (S[k], U[k, m], V[k, n], R[k]) host arrays to fill (e.g. views
    of pinned memory: device-to-host copies into pageable memory are several
    times slower); U / V are returned transposed views (column-major m x k)."""
    m, n = A.m, A.n
    if out is None:
        S, U, V, R = (np.zeros(k), np.zeros((k, m)), np.zeros((k, n)), np.zeros(k))
    else:
        S, U, V, R = out
        assert S.shape == (k,) and U.shape == (k, m) and V.shape == (k, n) and R.shape == (k,)
        assert all(x.dtype == np.float64 and x.flags.c_contiguous for x in (S, U, V, R))
    v0h = None if v0 is None else np.ascontiguousarray(v0, np.float64)
    o = Opts(k=k, tol=tol, t=t or 0, maxit=maxit, seed=seed,
             v0=None if v0h is None else v0h.ctypes.data, fixed_passes=fixed_passes, reorth=reorth)
    info = Info()
    if A.kind == "csr":
        rp = np.ascontiguousarray(A.row_ptr, np.int64)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        va = np.ascontiguousarray(A.values, np.float64)
        st = lib().svdsc_solve_host_csr(h.ptr, m, n, va.size, rp.ctypes.data, ci.ctypes.data,
                                        va.ctypes.data, ctypes.byref(o), S.ctypes.data, U.ctypes.data,
                                        V.ctypes.data, R.ctypes.data, ctypes.byref(info))
    else:
        D = np.asfortranarray(A.dense, np.float64)
        st = lib().svdsc_solve_host_dense(h.ptr, m, n, D.ctypes.data, ctypes.byref(o), S.ctypes.data,
                                          U.ctypes.data, V.ctypes.data, R.ctypes.data, ctypes.byref(info))
    h._check(st)
    return S, U.T, V.T, R, st, info.as_dict()


# ---- step-level ops ----------------------------------------
def matvec(M: Matrix, x, trans=False, c=None, yprev=None):
    """a1/a5: y = op(A) x - c * yprev (c: 1-element device tensor)."""
    dev = x.device
    y = torch.empty(M.n if trans else M.m, device=dev, dtype=torch.float64)
    M.h._check(lib().svdsc_op_matvec(M.ptr, int(trans), _ptr(x), _ptr(y), _ptr(c), _ptr(yprev)))
    return y


def cgs2(h: Handle, Q, w):
    """a2-a4/a6: w <- (I - QQ^T)^2 w in place on a copy; returns (w, ||w||)."""
    N = w.numel()
    wp = torch.zeros(-(-N // 32) * 32, device=w.device, dtype=torch.float64)  # padded like a basis column
    wp[:N] = w
    w = wp[:N]
    ncols = 0 if Q is None else Q.shape[1]
    nrm = torch.empty(1, device=w.device, dtype=torch.float64)
    ldq = _ld(Q) if ncols else N
    h._check(lib().svdsc_op_cgs2(h.ptr, N, ncols, _ptr(Q) if ncols else None, ldq, _ptr(w), _ptr(nrm)))
    return w, nrm


def cgs2_peer_emulate(h: Handle, Q, w, row0):
    """f2: the multi-GPU CGS2 (in-kernel peer all-reduces) with len(row0)-1 ranks
    emulated on one GPU; rank q owns rows row0[q]:row0[q+1].  Returns (w, betas)
    with w re-orthogonalized and normalized in place on a padded copy."""
    N = w.numel()
    wp = torch.zeros(-(-N // 32) * 32, device=w.device, dtype=torch.float64)
    wp[:N] = w
    w = wp[:N]
    ncols = 0 if Q is None else Q.shape[1]
    r0 = np.ascontiguousarray(row0, dtype=np.int64)
    betas = np.zeros(len(r0) - 1)
    ldq = _ld(Q) if ncols else N
    h._check(lib().svdsc_op_cgs2_peer_emulate(h.ptr, len(r0) - 1, r0.ctypes.data, ncols,
                                              _ptr(Q) if ncols else None, ldq, _ptr(w), betas.ctypes.data))
    return w, betas


def small_svd(h: Handle, T):
    """a7: device one-sided Jacobi SVD of a p x p column-major matrix."""
    p = T.shape[0]
    U, V = colmajor(p, p, T.device), colmajor(p, p, T.device)
    S = torch.empty(p, device=T.device, dtype=torch.float64)
    sw = ctypes.c_int32()
    h._check(lib().svdsc_op_small_svd(h.ptr, p, _ptr(T), _ptr(U), _ptr(S), _ptr(V), ctypes.byref(sw)))
    return U, S, V, sw.value


def recombine(h: Handle, Q, W, k, out=None):
    """a8/a9: out(:, :k) = Q(:, :t) W(:, :k); out may be Q (in place)."""
    N, t = Q.shape[0], W.shape[0]
    if out is None:
        out = colmajor(N, k, Q.device)
    h._check(lib().svdsc_op_recombine(h.ptr, N, t, k, _ptr(Q), _ld(Q), _ptr(W), _ld(W), _ptr(out),
                                      _ld(out)))
    return out


def lbp(M: Matrix, t, v0, seed=0, reorth=2):
    """One first pass LBP(A, t+1): U (m x t+1), V (n x t+1), T (t+1 x t+1), info."""
    dev = v0.device
    U, V, T = colmajor(M.m, t + 1, dev), colmajor(M.n, t + 1, dev), colmajor(t + 1, t + 1, dev)
    o = _opts(1, 1e-10, 0, 1, seed, None, 0, reorth)
    info = Info()
    M.h._check(lib().svdsc_op_lbp(M.ptr, ctypes.byref(o), t, _ptr(v0.contiguous()), _ptr(U), _ld(U),
                                  _ptr(V), _ld(V), _ptr(T), ctypes.byref(info)))
    return U, V, T, info.as_dict()


# ---- the paper's interface and Matrix Market I/O ----------------
class PaperError(RuntimeError):
    pass


def _paper_check(st):
    if st < 0:
        raise PaperError(f"status {st}: {lib().svdsc_paper_last_error().decode()}")
    return st


def paper_csr(nrows, ncols, values, cols1, pointerB, pointerE):
    """Build a PaperCsr over numpy arrays (kept alive on the returned object)."""
    values = np.ascontiguousarray(values, np.float64)
    cols1 = np.ascontiguousarray(cols1, np.int32)
    pointerB = np.ascontiguousarray(pointerB, np.int32)
    pointerE = np.ascontiguousarray(pointerE, np.int32)
    A = PaperCsr(values.size, nrows, ncols, values.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                 cols1.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                 pointerB.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                 pointerE.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    A._keep = (values, cols1, pointerB, pointerE)
    return A


def paper_csr_to_csr(A: PaperCsr):
    """svdsc_paper_csr_to_csr: the paper layout -> (row_ptr, col_idx, values), 0-based."""
    rp, ci, va, nk = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    _paper_check(lib().svdsc_paper_csr_to_csr(ctypes.byref(A), ctypes.byref(rp), ctypes.byref(ci),
                                              ctypes.byref(va), ctypes.byref(nk)))
    libc = ctypes.CDLL(None)
    libc.free.argtypes = [ctypes.c_void_p]
    out = (np.ctypeslib.as_array(ctypes.cast(rp, ctypes.POINTER(ctypes.c_int64)), (A.nrows + 1,)).copy(),
           np.ctypeslib.as_array(ctypes.cast(ci, ctypes.POINTER(ctypes.c_int32)), (max(nk.value, 1),))[:nk.value].copy(),
           np.ctypeslib.as_array(ctypes.cast(va, ctypes.POINTER(ctypes.c_double)), (max(nk.value, 1),))[:nk.value].copy())
    for p in (rp, ci, va):
        libc.free(p)
    return out


def _mat_to_numpy(M: PaperMat):
    a = np.ctypeslib.as_array(M.d, (M.ncols * M.nrows,)).reshape(M.ncols, M.nrows).T.copy()
    lib().svdsc_mat_free(ctypes.byref(M))
    return a


def read_mm(path):
    """svdsc_read_mm -> ("csr", PaperCsr-as-numpy dict) or ("dense", ndarray)."""
    A, D, dense = PaperCsr(), PaperMat(), ctypes.c_int()
    _paper_check(lib().svdsc_read_mm(str(path).encode(), ctypes.byref(A), ctypes.byref(D), ctypes.byref(dense)))
    if dense.value:
        return "dense", _mat_to_numpy(D)
    K = A.nnz
    d = {"nrows": A.nrows, "ncols": A.ncols,
         "values": np.ctypeslib.as_array(A.values, (max(K, 1),))[:K].copy(),
         "cols": np.ctypeslib.as_array(A.cols, (max(K, 1),))[:K].copy(),
         "pointerB": np.ctypeslib.as_array(A.pointerB, (max(A.nrows, 1),))[:A.nrows].copy(),
         "pointerE": np.ctypeslib.as_array(A.pointerE, (max(A.nrows, 1),))[:A.nrows].copy()}
    lib().svdsc_mat_csr_free(ctypes.byref(A))
    return "csr", d


def write_mm(path, csr=None, dense=None):
    if csr is not None:
        A = paper_csr(csr["nrows"], csr["ncols"], csr["values"], csr["cols"], csr["pointerB"], csr["pointerE"])
        _paper_check(lib().svdsc_write_mm(str(path).encode(), ctypes.byref(A), None))
    else:
        D = np.asfortranarray(dense, np.float64)
        M = PaperMat(D.shape[0], D.shape[1], D.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        _paper_check(lib().svdsc_write_mm(str(path).encode(), None, ctypes.byref(M)))


def svds_C(A, k, tol=None, t=None, r=None):
    """The paper's svds_C / svds_C_opt (sparse PaperCsr) or svds_C_dense(_opt)
    (numpy 2-D array): host in, host out; returns (U, S, V, status)."""
    U, Sm, V = PaperMat(), PaperMat(), PaperMat()
    opt = tol is not None or t is not None or r is not None
    extra = (1e-10 if tol is None else tol, 0 if t is None else t, 10 if r is None else r)
    if isinstance(A, PaperCsr):
        f = lib().svds_C_opt if opt else lib().svds_C
        args = [ctypes.byref(A), ctypes.byref(U), ctypes.byref(Sm), ctypes.byref(V), k]
    else:
        D = np.asfortranarray(A, np.float64)
        M = PaperMat(D.shape[0], D.shape[1], D.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        f = lib().svds_C_dense_opt if opt else lib().svds_C_dense
        args = [ctypes.byref(M), ctypes.byref(U), ctypes.byref(Sm), ctypes.byref(V), k]
    st = _paper_check(f(*args, *extra) if opt else f(*args))
    return _mat_to_numpy(U), _mat_to_numpy(Sm)[:, 0], _mat_to_numpy(V), st
