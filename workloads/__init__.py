"""Seeded synthetic inputs for the svds-C hot path (oracle and CUDA path alike).

This module is the only code the oracle side and the CUDA side share, and it
holds none of the method's arithmetic: it only draws matrices and start
vectors.  The paper's datasets are not available; the
BASELINE.json configs stand in for their shapes.

Sparse rows come from ``gen.c`` (counter-based per-row streams, multithreaded,
thread-count independent); dense matrices with a prescribed spectrum use
numpy's LAPACK Householder QR (BASELINE.json config 2).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STREAM_V0 = 3
STREAM_DENSE_U = 7
STREAM_DENSE_V = 8
STREAM_CELLS = 11


def _lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(_HERE, "libworkloads.so")
        src = os.path.join(_HERE, "gen.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            build()
        lib = ctypes.CDLL(so)
        lib.wl_zipf2.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        lib.wl_fill_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.wl_fill_rows.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def build():
    so = os.path.join(_HERE, "libworkloads.so")
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", so,
                           os.path.join(_HERE, "gen.c"), "-lm"])


# ---------------------------------------------------------------------------
@dataclass
class Matrix:
    """A host matrix: CSR (0-based int64 row_ptr, int32 col_idx, f64 values,
    distinct sorted columns per row) or dense column-major f64."""
    kind: str                      # "csr" | "dense"
    m: int
    n: int
    row_ptr: np.ndarray | None = None
    col_idx: np.ndarray | None = None
    values: np.ndarray | None = None
    dense: np.ndarray | None = None   # Fortran-ordered (m, n)
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if self.kind == "csr" else self.m * self.n

    def to_dense(self) -> np.ndarray:
        if self.kind == "dense":
            return np.asarray(self.dense)
        A = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.m), np.diff(self.row_ptr))
        np.add.at(A, (rows, self.col_idx.astype(np.int64)), self.values)
        return A

    def bytes_one_pass(self) -> int:
        """Bytes one A x (or A^T x) pass must stream: 12 B/nnz + row pointers
        (int32 col + f64 value), or 8 m n dense."""
        if self.kind == "dense":
            return 8 * self.m * self.n
        return 12 * self.nnz + 4 * (self.m + 1)


@dataclass
class Workload:
    name: str
    A: Matrix
    v0: np.ndarray
    k: int
    t: int
    tol: float
    maxit: int
    meta: dict = field(default_factory=dict)


def csr_from_dense(D: np.ndarray) -> Matrix:
    D = np.asarray(D, dtype=np.float64)
    m, n = D.shape
    rows, cols = np.nonzero(D)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int64)
    return Matrix("csr", m, n, row_ptr=row_ptr, col_idx=cols.astype(np.int32),
                  values=D[rows, cols].astype(np.float64))


def dense_matrix(D: np.ndarray) -> Matrix:
    D = np.asfortranarray(np.asarray(D, dtype=np.float64))
    return Matrix("dense", D.shape[0], D.shape[1], dense=D)


def start_vector(n: int, seed: int = 0) -> np.ndarray:
    """v0 ~ N(0,1)^n from its own stream (Alg. 1 line 1 "randn(n,1)", reading Q8)."""
    return np.random.default_rng([seed, STREAM_V0]).standard_normal(n)


# ---------------------------------------------------------------------------
# Spectra of PAPER.md Eq. (16) (lines 334-345) and BASELINE config 2.
def spectrum(kind: str, length: int) -> np.ndarray:
    i = np.arange(1, length + 1, dtype=np.float64)
    if kind == "decay1":
        return np.where(i <= 20, 10.0 ** (-(4.0 / 19.0) * (i - 1)),
                        1e-4 / np.maximum(i - 20, 1.0) ** 0.1)
    if kind == "decay2":
        return i ** -2.0
    if kind == "decay3":
        return i ** -3.0
    if kind == "exp40":
        return np.exp(-i / 40.0)
    raise ValueError(kind)


def random_orthonormal(rows: int, cols: int, rng: np.random.Generator) -> np.ndarray:
    """Thin Q of the Householder QR (LAPACK geqrf/orgqr) of a Gaussian matrix."""
    G = rng.standard_normal((rows, cols))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))  # unique Haar-distributed Q


def dense_with_spectrum(m: int, n: int, sigma: np.ndarray, seed: int = 0,
                        keep_factors: bool = False) -> Matrix:
    """A = Q_U diag(sigma) Q_V^T, column-major (SPEC.md:349-357 construction)."""
    p = min(m, n)
    assert sigma.shape == (p,)
    QU = random_orthonormal(m, p, np.random.default_rng([seed, STREAM_DENSE_U]))
    QV = random_orthonormal(n, p, np.random.default_rng([seed, STREAM_DENSE_V]))
    A = np.asfortranarray((QU * sigma) @ QV.T)
    M = Matrix("dense", m, n, dense=A, meta={"sigma": sigma})
    if keep_factors:
        M.meta["QU"] = QU
        M.meta["QV"] = QV
    return M


def sparse_uniform_cells(m: int, n: int, nnz: int, seed: int = 0) -> Matrix:
    """Exactly nnz distinct positions uniform over the m*n cells, N(0,1) values
    (BASELINE config 1)."""
    rng = np.random.default_rng([seed, STREAM_CELLS])
    cells = np.sort(rng.choice(m * n, size=nnz, replace=False))
    rows = cells // n
    cols = (cells % n).astype(np.int32)
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.int64)
    vals = rng.standard_normal(nnz)
    return Matrix("csr", m, n, row_ptr=row_ptr, col_idx=cols, values=vals)


def _fill(kind: int, val_kind: int, m: int, n: int, deg: np.ndarray, seed: int,
          band: int = 0, r0: int = 0, r1: int | None = None) -> Matrix:
    r1 = m if r1 is None else r1
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(deg.astype(np.int64))
    lo, hi = int(row_ptr[r0]), int(row_ptr[r1])
    col = np.empty(hi - lo, dtype=np.int32)
    val = np.empty(hi - lo, dtype=np.float64)
    nth = os.cpu_count() or 1
    _lib().wl_fill_rows(kind, val_kind, m, n, band, seed, r0, r1,
                        row_ptr.ctypes.data, col.ctypes.data, val.ctypes.data, nth)
    local_ptr = row_ptr[r0:r1 + 1] - lo
    return Matrix("csr", r1 - r0, n, row_ptr=local_ptr, col_idx=col, values=val,
                  meta={"row_offset": r0, "m_global": m})


def sparse_fixed_rows(m: int, n: int, d: int, values: str = "u01", seed: int = 0,
                      r0: int = 0, r1: int | None = None) -> Matrix:
    """Exactly d distinct uniform columns per row (BASELINE config 3)."""
    vk = {"normal": 0, "u01": 1, "upm1": 2}[values]
    return _fill(0, vk, m, n, np.full(m, d, dtype=np.int64), seed, 0, r0, r1)


def zipf_degrees(m: int, n: int, target_nnz: int, cap: int, seed: int = 0):
    """d_r = min(cap, max(1, round(s X_r))), X_r ~ Zipf(2), s bisected so that
    sum d_r is closest to target_nnz (BASELINE config 4, reading Q19)."""
    X = np.empty(m, dtype=np.int64)
    _lib().wl_zipf2(seed, 0, m, X.ctypes.data)
    cap = min(cap, n)
    Xf = X.astype(np.float64)

    def total(s):
        return int(np.minimum(cap, np.maximum(1, np.rint(s * Xf))).sum())

    lo, hi = 1e-3, 1e3
    for _ in range(100):
        mid = np.sqrt(lo * hi)
        if total(mid) < target_nnz:
            lo = mid
        else:
            hi = mid
    s = lo if abs(total(lo) - target_nnz) <= abs(total(hi) - target_nnz) else hi
    deg = np.minimum(cap, np.maximum(1, np.rint(s * Xf))).astype(np.int64)
    return deg, s


def sparse_powerlaw(m: int, n: int, target_nnz: int, cap: int = 100_000, seed: int = 0,
                    r0: int = 0, r1: int | None = None) -> Matrix:
    deg, s = zipf_degrees(m, n, target_nnz, cap, seed)
    M = _fill(0, 0, m, n, deg, seed, 0, r0, r1)
    M.meta["zipf_scale"] = s
    return M


def sparse_banded(m: int, n: int, d: int = 20, band: int = 1000, seed: int = 0,
                  r0: int = 0, r1: int | None = None) -> Matrix:
    """d distinct columns per row: d/2 within +-band of the scaled diagonal
    floor(r n / m), d/2 uniform elsewhere; U(-1,1) values (BASELINE config 5)."""
    return _fill(1, 2, m, n, np.full(m, d, dtype=np.int64), seed, band, r0, r1)


# ---------------------------------------------------------------------------
# BASELINE.json configs (1-based ids as in SURVEY.md).  `scale` divides m and
# n (scaled replicas for oracle parity at configs 3-5).
CONFIG_NAMES = {
    1: "sparse5000x3000_k10",
    2: "dense20000x5000_exp40_k50",
    3: "sparse200000x100000_r50_k100",
    4: "powerlaw4Mx2M_k100",
    5: "banded30Mx5M_k200",
    # the paper's own dense workload Dense1-3,
    # 10,000 x 10,000 with the Decay1/2/3 spectra of Eq. (16)
    6: "dense1_10000_decay1_k100",
    7: "dense2_10000_decay2_k100",
    8: "dense3_10000_decay3_k100",
}


def degrees(cid: int, seed: int = 0, scale: int = 1) -> np.ndarray | None:
    """Row lengths of a sparse config's generator, without generating the rows
    (for the row partition of a multi-GPU run: every rank then
    generates only its own rows with config(cid, r0=..., r1=...)).  None for
    configs generated as a whole (1: uniform cells; dense)."""
    f = scale
    if cid == 3:
        return np.full(200_000 // f, 50, dtype=np.int64)
    if cid == 4:
        return zipf_degrees(4_000_000 // f, 2_000_000 // f, 150_000_000 // f, 100_000, seed)[0]
    if cid == 5:
        return np.full(30_000_000 // f, 20, dtype=np.int64)
    return None


def config(cid: int, seed: int = 0, scale: int = 1, r0: int = 0, r1: int | None = None,
           keep_factors: bool = False) -> Workload:
    f = scale
    if cid == 1:
        m, n = 5000 // f, 3000 // f
        A = sparse_uniform_cells(m, n, 150_000 // (f * f), seed)
        k, t = 10, 30
    elif cid == 2:
        m, n = 20000 // f, 5000 // f
        A = dense_with_spectrum(m, n, spectrum("exp40", min(m, n)), seed, keep_factors)
        k, t = 50, 150
    elif cid == 3:
        m, n = 200_000 // f, 100_000 // f
        A = sparse_fixed_rows(m, n, 50, "u01", seed, r0, r1)
        k, t = 100, 300
    elif cid == 4:
        m, n = 4_000_000 // f, 2_000_000 // f
        A = sparse_powerlaw(m, n, 150_000_000 // f, 100_000, seed, r0, r1)
        k, t = 100, 300
    elif cid == 5:
        m, n = 30_000_000 // f, 5_000_000 // f
        A = sparse_banded(m, n, 20, max(1000 // f, 10), seed, r0, r1)
        k, t = 200, 600
    elif cid in (6, 7, 8):
        m = n = 10_000 // f
        A = dense_with_spectrum(m, n, spectrum(f"decay{cid - 5}", m), seed, keep_factors)
        k, t = 100, 300
    else:
        raise ValueError(cid)
    name = CONFIG_NAMES[cid] + (f"_div{f}" if f != 1 else "")
    v0 = start_vector(A.n, seed)
    return Workload(name, A, v0, k, t, 1e-10, 100, meta={"config": cid, "scale": f})
