"""Test-side helpers (not product code): principal angles from sines,
certificates of Proposition 1, reduction-order error budgets."""
import numpy as np

U_RND = 2.0 ** -53


def gamma(n):
    """gamma_n = n u / (1 - n u), the standard dot-product error constant."""
    return n * U_RND / (1 - n * U_RND)


def orth(X):
    Q, _ = np.linalg.qr(X)
    return Q


def sin_max_angle(A, B):
    """sin of the largest principal angle between span(A) and span(B),
    computed as ||Qb - Qa (Qa^T Qb)||_2 (never arccos of cosines)."""
    Qa, Qb = orth(np.asarray(A)), orth(np.asarray(B))
    R = Qb - Qa @ (Qa.T @ Qb)
    return np.linalg.norm(R, 2)


def orth_error(Q):
    Q = np.asarray(Q)
    return np.abs(Q.T @ Q - np.eye(Q.shape[1])).max()


def matvec(A, x):
    if A.kind == "dense":
        return A.dense @ x
    out = np.zeros(A.m)
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    np.add.at(out, rows, A.values * x[A.col_idx])
    return out


def matvec_t(A, x):
    if A.kind == "dense":
        return A.dense.T @ x
    out = np.zeros(A.n)
    rows = np.repeat(np.arange(A.m), np.diff(A.row_ptr))
    np.add.at(out, A.col_idx.astype(np.int64), A.values * x[rows])
    return out


def certificates(A, S, U, V):
    """Proposition 1: ||A v_j - s_j u_j|| and
    ||A^T u_j - s_j v_j|| / s_j for every returned triplet."""
    k = len(S)
    r1 = np.array([np.linalg.norm(matvec(A, V[:, j]) - S[j] * U[:, j]) for j in range(k)])
    r2 = np.array([np.linalg.norm(matvec_t(A, U[:, j]) - S[j] * V[:, j]) / S[j] for j in range(k)])
    return r1, r2
