"""ctypes wrapper of the plain C fp64 oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: importable by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2405_18966_b200) never imports this module.

Each function cites the paper passage its C counterpart follows; see the
header of oracle.c.  "parity unpinned" items: none (every function is pinned
by tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

OR_OK, OR_NOT_CONVERGED = 0, 1


def build() -> str:
    src = os.path.join(_HERE, "oracle.c")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", "-o", _SO, src, "-lm"])
    return _SO


class _Matrix(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("dense", ctypes.c_void_p), ("ld", ctypes.c_int64)]


class _Opts(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("tol", ctypes.c_double), ("t", ctypes.c_int32),
                ("maxit", ctypes.c_int32), ("fixed_passes", ctypes.c_int32),
                ("reorth", ctypes.c_int32), ("seed", ctypes.c_uint64), ("pro_delta", ctypes.c_double)]


class _Info(ctypes.Structure):
    _fields_ = [("passes", ctypes.c_int32), ("restarts", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("t_used", ctypes.c_int32),
                ("steps", ctypes.c_int64), ("matvecs", ctypes.c_int64),
                ("breakdowns", ctypes.c_int64), ("max_resid", ctypes.c_double),
                ("reorths", ctypes.c_int64)]


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "oracle.c")
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_SO)
        P, I64 = ctypes.c_void_p, ctypes.c_int64
        L.or_spmv.argtypes = [I64, P, P, P, P, P]
        L.or_spmv_t.argtypes = [I64, I64, P, P, P, P, P]
        L.or_gemv_n.argtypes = [I64, I64, P, I64, P, P]
        L.or_gemv_t.argtypes = [I64, I64, P, I64, P, P]
        L.or_norm2.argtypes = [I64, P]
        L.or_norm2.restype = ctypes.c_double
        L.or_cgs2.argtypes = [I64, I64, P, I64, P, P]
        L.or_jacobi_svd.argtypes = [I64, I64, P, P, P, P, ctypes.c_int]
        L.or_jacobi_svd.restype = ctypes.c_int
        L.or_breakdown_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.or_breakdown_uniform.restype = ctypes.c_double
        L.or_svds.argtypes = [ctypes.POINTER(_Matrix), ctypes.POINTER(_Opts), P, P, P, P, P,
                              ctypes.POINTER(_Info)]
        L.or_svds.restype = ctypes.c_int
        L.or_lbp.argtypes = [ctypes.POINTER(_Matrix), ctypes.POINTER(_Opts), I64, P, P, P, P,
                             ctypes.POINTER(_Info)]
        L.or_lbp.restype = ctypes.c_int
        D = ctypes.c_double
        L.or_pro_anorm.argtypes = [P, I64, I64]
        L.or_pro_anorm.restype = D
        L.or_pro_nu_update.argtypes = [P, I64, I64, P, P, D, D]
        L.or_pro_mu_update.argtypes = [P, I64, I64, P, P, D, D]
        L.or_pro_restart.argtypes = [I64, I64, P, P, P, P]
        L.or_pro_restart.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _matrix(A):
    """A: workloads.Matrix.  Returns (ctypes struct, keepalive list)."""
    keep = []
    M = _Matrix()
    M.m, M.n = A.m, A.n
    if A.kind == "csr":
        rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
        va = _f64(A.values)
        keep += [rp, ci, va]
        M.kind, M.row_ptr, M.col_idx, M.val = 0, _p(rp), _p(ci), _p(va)
    else:
        D = np.asfortranarray(A.dense, dtype=np.float64)
        keep.append(D)
        M.kind, M.dense, M.ld = 1, D.ctypes.data, A.m
    return M, keep


# --- primitives ------------------------------------------------------------
def spmv(A, x):
    """y = A x (Alg. 1 line 7)."""
    x = _f64(x)
    y = np.empty(A.m)
    if A.kind == "csr":
        rp = np.ascontiguousarray(A.row_ptr, np.int64)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        va = _f64(A.values)
        lib().or_spmv(A.m, _p(rp), _p(ci), _p(va), _p(x), _p(y))
    else:
        D = np.asfortranarray(A.dense, np.float64)
        lib().or_gemv_n(A.m, A.n, D.ctypes.data, A.m, _p(x), _p(y))
    return y


def spmv_t(A, x):
    """y = A^T x (Alg. 1 line 5)."""
    x = _f64(x)
    y = np.empty(A.n)
    if A.kind == "csr":
        rp = np.ascontiguousarray(A.row_ptr, np.int64)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        va = _f64(A.values)
        lib().or_spmv_t(A.m, A.n, _p(rp), _p(ci), _p(va), _p(x), _p(y))
    else:
        D = np.asfortranarray(A.dense, np.float64)
        lib().or_gemv_t(A.m, A.n, D.ctypes.data, A.m, _p(x), _p(y))
    return y


def norm2(x):
    x = _f64(x)
    return lib().or_norm2(x.size, _p(x))


def cgs2(Q, w):
    """w <- (I - Q Q^T) w, two classical Gram-Schmidt passes."""
    Q = np.asfortranarray(Q, dtype=np.float64)
    w = _f64(w).copy()
    h = np.zeros(max(Q.shape[1], 1))
    lib().or_cgs2(Q.shape[0], Q.shape[1], Q.ctypes.data, Q.shape[0], _p(w), _p(h))
    return w


def jacobi_svd(M, max_sweeps=50):
    """One-sided Jacobi SVD (Alg. 2 step 4 small SVD).  Returns U, S, V, sweeps."""
    M = np.asfortranarray(M, dtype=np.float64)
    p, q = M.shape
    assert q <= p
    U = np.zeros((p, q), order="F")
    S = np.zeros(q)
    V = np.zeros((q, q), order="F")
    sw = lib().or_jacobi_svd(p, q, M.ctypes.data, U.ctypes.data, _p(S), V.ctypes.data, max_sweeps)
    if sw < 0:
        raise RuntimeError(f"jacobi_svd failed: {sw}")
    return U, S, V, sw


def breakdown_uniform(seed, stream, n):
    return np.array([lib().or_breakdown_uniform(seed, stream, r) for r in range(n)])


@dataclass
class Result:
    S: np.ndarray
    U: np.ndarray
    V: np.ndarray
    resid: np.ndarray
    status: int
    passes: int
    restarts: int
    converged: bool
    t: int
    steps: int
    matvecs: int
    breakdowns: int
    max_resid: float
    reorths: int = 0


def svds(A, k, v0, tol=1e-10, t=0, maxit=100, fixed_passes=0, reorth=2, seed=0, pro_delta=0.0) -> Result:
    """Alg. 2: the restarted truncated SVD.  reorth: 2 full
    CGS2, 1 partial (omega recurrence, reading Q20), 0 off."""
    M, keep = _matrix(A)
    o = _Opts(k=k, tol=tol, t=t, maxit=maxit, fixed_passes=fixed_passes, reorth=reorth, seed=seed,
              pro_delta=pro_delta)
    v0 = _f64(v0)
    S = np.zeros(k)
    U = np.zeros((A.m, k), order="F")
    V = np.zeros((A.n, k), order="F")
    res = np.zeros(k)
    info = _Info()
    st = lib().or_svds(ctypes.byref(M), ctypes.byref(o), _p(v0), _p(S), U.ctypes.data,
                       V.ctypes.data, _p(res), ctypes.byref(info))
    if st < 0:
        raise RuntimeError(f"or_svds failed with status {st}")
    return Result(S, U, V, res, st, info.passes, info.restarts, bool(info.converged),
                  info.t_used, info.steps, info.matvecs, info.breakdowns, info.max_resid, info.reorths)


def lbp(A, t, v0, reorth=2, seed=0, pro_delta=0.0):
    """Alg. 1 first pass LBP(A, t+1): returns U (m x t+1), V (n x t+1), T, info."""
    M, keep = _matrix(A)
    o = _Opts(k=1, tol=1e-10, t=t, maxit=1, fixed_passes=1, reorth=reorth, seed=seed, pro_delta=pro_delta)
    U = np.zeros((A.m, t + 1), order="F")
    V = np.zeros((A.n, t + 1), order="F")
    T = np.zeros((t + 1, t + 1), order="F")
    info = _Info()
    v0 = _f64(v0)
    st = lib().or_lbp(ctypes.byref(M), ctypes.byref(o), t, _p(v0), U.ctypes.data, V.ctypes.data,
                      T.ctypes.data, ctypes.byref(info))
    if st < 0:
        raise RuntimeError(f"or_lbp failed with status {st}")
    return U, V, T, info


# ---- partial re-orthogonalization (reading Q20): one omega update each ----
def pro_anorm(T, ncols):
    T = np.asfortranarray(T, dtype=np.float64)
    return lib().or_pro_anorm(T.ctypes.data, T.shape[0], ncols)


def pro_nu_update(T, i, mu, nu, beta, eps1):
    """row of v_{i-1} (nu) -> row of v_i, given the row mu of u_{i-1}"""
    T = np.asfortranarray(T, dtype=np.float64)
    mu = _f64(mu)
    out = np.zeros(max(len(nu), i + 1))
    out[:len(nu)] = nu
    lib().or_pro_nu_update(T.ctypes.data, T.shape[0], i, _p(mu), _p(out), beta, eps1)
    return out[:i + 1]


def pro_restart(t, k, Vh, nu, mu):
    """or_pro_restart: the omega rows after an augmented restart (reading Q20)"""
    Vh = np.asfortranarray(Vh, dtype=np.float64)
    nu_o = np.zeros(t + 1)
    nu_o[:len(nu)] = nu
    mu_o = np.zeros(t + 1)
    mu_o[:len(mu)] = mu
    tmp = np.zeros(max(k, 1))
    lib().or_pro_restart(t, k, Vh.ctypes.data, _p(nu_o), _p(mu_o), _p(tmp))
    return nu_o[:k + 1], mu_o[:k + 1]


def pro_mu_update(T, i, nu, mu, alpha, eps1):
    """row of u_{i-1} (mu) -> row of u_i, given the row nu of v_i"""
    T = np.asfortranarray(T, dtype=np.float64)
    nu = _f64(nu)
    out = np.zeros(max(len(mu), i + 1))
    out[:len(mu)] = mu
    lib().or_pro_mu_update(T.ctypes.data, T.shape[0], i, _p(nu), _p(out), alpha, eps1)
    return out[:i + 1]
