"""Pins of the oracle's partial re-orthogonalization (reorth = 1, SURVEY.md
8(f4), reading Q20).  The paper names the method class only
(PROPACK lansvd), so the pins are what the mathematics fixes:

- limits: delta -> 0 re-orthogonalizes every half-step and must reproduce
  full CGS2 bit for bit; delta -> inf never does and must
  reproduce plain Alg. 1 (reorth = 0) bit for bit;
- the omega recurrence against brute-force inner products of real Lanczos
  vectors that have lost orthogonality (first pass: bidiagonal T; after an
  augmented restart: the arrow T of Alg. 2 step 9), with the rounding term
  switched off, so a dropped term, a wrong index or sign shows up at the size
  of the inner products themselves;
- semi-orthogonality (|U^T U - I| stays near sqrt(eps)) where plain Alg. 1
  loses all orthogonality, and the closed-form Decay2 spectrum to tolerance.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

EPS = 2.0 ** -52


def decay2(m=400, n=300, seed=4):
    return W.dense_with_spectrum(m, n, W.spectrum("decay2", n), seed=seed)


@pytest.mark.parametrize("which", ["dense", "sparse"])
def test_pro_delta_limits_reduce_to_full_and_none(which):
    A = decay2() if which == "dense" else W.config(1, scale=2).A
    t = 60
    v0 = np.random.default_rng(3).standard_normal(A.n)
    U2, V2, T2, i2 = O.lbp(A, t, v0, reorth=2)
    U1, V1, T1, i1 = O.lbp(A, t, v0, reorth=1, pro_delta=1e-300)
    assert np.array_equal(U1, U2) and np.array_equal(V1, V2) and np.array_equal(T1, T2)
    assert i1.reorths == i2.reorths == 2 * t
    U0, V0, T0, _ = O.lbp(A, t, v0, reorth=0)
    Ui, Vi, Ti, ii = O.lbp(A, t, v0, reorth=1, pro_delta=1e300)
    assert np.array_equal(Ui, U0) and np.array_equal(Vi, V0) and np.array_equal(Ti, T0)
    assert ii.reorths == 0


def _check_row(pred, true, scale, what):
    # exact algebra up to rounding of the products and of the vectors themselves
    err = np.abs(pred - true)
    assert err.max() <= 1e-9 * scale + 1e-12, f"{what}: max err {err.max():.3e}"


def test_pro_recurrence_first_pass_against_inner_products():
    # plain Alg. 1 (no re-orthogonalization) on Decay2 loses orthogonality
    # completely within 120 steps: the inner products span 1e-16 .. 1
    A = decay2()
    t = 120
    U, V, T, _ = O.lbp(A, t, np.random.default_rng(1).standard_normal(A.n), reorth=0)
    assert np.abs(V.T @ V - np.eye(t + 1)).max() > 0.5
    big = 0
    for i in range(1, t):
        mu = U[:, :i].T @ U[:, i - 1]              # row of u_{i-1}
        nu_prev = V[:, :i].T @ V[:, i - 1]         # row of v_{i-1}
        beta, alpha = T[i - 1, i], T[i, i]          # reorth = 0: the unnormalized norms
        nu = O.pro_nu_update(T, i, mu, nu_prev, beta, 0.0)
        true_nu = V[:, :i].T @ V[:, i]
        _check_row(nu[:i], true_nu, np.abs(true_nu).max() + 1.0 / beta * EPS * 1e4, f"nu step {i}")
        assert nu[i] == 1.0
        true_nu_full = V[:, :i + 1].T @ V[:, i]
        mu_new = O.pro_mu_update(T, i, true_nu_full, mu, alpha, 0.0)
        true_mu = U[:, :i].T @ U[:, i]
        _check_row(mu_new[:i], true_mu, np.abs(true_mu).max() + 1.0 / alpha * EPS * 1e4, f"mu step {i}")
        big += int(np.abs(true_mu).max() > 1e-3)
    assert big > 20  # the check was made where the inner products are large


def test_pro_recurrence_after_restart_arrow():
    # augmented restart state (Alg. 2 steps 8-11) built in numpy from a full-CGS2
    # first pass, then continued WITHOUT re-orthogonalization so that the new
    # vectors lose orthogonality against the Ritz vectors: the arrow column
    # T(0:k, k) = rho and rows T(j, j), T(j, k) enter the recurrence
    A = decay2(300, 200, seed=9)
    D = A.dense
    k, t = 5, 8  # short first pass: rho = beta_t Uh(t, 1:k) is far from zero
    U, V, T, _ = O.lbp(A, t, np.random.default_rng(2).standard_normal(A.n), reorth=2)
    Uh, s, Vht = np.linalg.svd(T[:t, :t])
    Vh = Vht.T
    beta_t = T[t - 1, t]
    K = k + 1 + 90
    Tn = np.zeros((K + 1, K + 1), order="F")
    Un = np.zeros((A.m, K + 1))
    Vn = np.zeros((A.n, K + 1))
    Un[:, :k] = U[:, :t] @ Uh[:, :k]
    Vn[:, :k] = V[:, :t] @ Vh[:, :k]
    rho = beta_t * Uh[t - 1, :k]
    Tn[np.arange(k), np.arange(k)] = s[:k]
    Tn[:k, k] = rho
    assert np.abs(rho).max() > 1e-3 * s[0]
    Vn[:, k] = V[:, t]
    z = D @ Vn[:, k] - Un[:, :k] @ rho
    for _ in range(2):  # full CGS2 of u_k against the Ritz vectors
        z -= Un[:, :k] @ (Un[:, :k].T @ z)
    Tn[k, k] = np.linalg.norm(z)
    Un[:, k] = z / Tn[k, k]
    for i in range(k + 1, K):
        w = D.T @ Un[:, i - 1] - Tn[i - 1, i - 1] * Vn[:, i - 1]
        Tn[i - 1, i] = np.linalg.norm(w)
        Vn[:, i] = w / Tn[i - 1, i]
        z = D @ Vn[:, i] - Tn[i - 1, i] * Un[:, i - 1]
        Tn[i, i] = np.linalg.norm(z)
        Un[:, i] = z / Tn[i, i]
    assert np.abs(Vn[:, :K].T @ Vn[:, :K] - np.eye(K)).max() > 1e-3
    big = 0
    for i in range(k + 1, K):
        mu = Un[:, :i].T @ Un[:, i - 1]
        nu_prev = Vn[:, :i].T @ Vn[:, i - 1]
        nu = O.pro_nu_update(Tn, i, mu, nu_prev, Tn[i - 1, i], 0.0)
        true_nu = Vn[:, :i].T @ Vn[:, i]
        _check_row(nu[:i], true_nu, np.abs(true_nu).max() + EPS * 1e4 / Tn[i - 1, i], f"arrow nu step {i}")
        mu_new = O.pro_mu_update(Tn, i, Vn[:, :i + 1].T @ Vn[:, i], mu, Tn[i, i], 0.0)
        true_mu = Un[:, :i].T @ Un[:, i]
        _check_row(mu_new[:i], true_mu, np.abs(true_mu).max() + EPS * 1e4 / Tn[i, i], f"arrow mu step {i}")
        big += int(np.abs(true_mu[:k]).max() > 1e-4)
    assert big > 10  # large inner products against the Ritz vectors were checked


def test_pro_anorm_is_max_column_one_norm():
    T = np.zeros((5, 5), order="F")
    T[0, 0], T[0, 1], T[1, 1], T[1, 2], T[2, 2] = 3.0, -1.0, 0.5, 4.0, -0.25
    assert O.pro_anorm(T, 1) == 3.0
    assert O.pro_anorm(T, 2) == 3.0          # |-1| + |0.5|
    assert O.pro_anorm(T, 3) == 4.25         # |4| + |-0.25|


def test_pro_keeps_semi_orthogonality_with_fewer_reorths():
    A = decay2()
    t = 120
    v0 = np.random.default_rng(1).standard_normal(A.n)
    U, V, T, info = O.lbp(A, t, v0, reorth=1)
    n = t + 1
    assert np.abs(U.T @ U - np.eye(n)).max() < 10 * np.sqrt(EPS)
    assert np.abs(V.T @ V - np.eye(n)).max() < 10 * np.sqrt(EPS)
    assert 0 < info.reorths < 2 * t * 0.75
    U0, V0, _, _ = O.lbp(A, t, v0, reorth=0)
    assert np.abs(U0.T @ U0 - np.eye(n)).max() > 0.1


def test_pro_svds_closed_form_decay2_and_config1():
    A = decay2()
    k = 8
    v0 = np.random.default_rng(5).standard_normal(A.n)
    r1 = O.svds(A, k, v0, tol=1e-10, t=30, maxit=50, reorth=1)
    r2 = O.svds(A, k, v0, tol=1e-10, t=30, maxit=50, reorth=2)
    assert r1.status == 0 and r1.converged
    assert np.abs(r1.S - W.spectrum("decay2", k)).max() <= 1e-10
    assert r1.reorths < r2.reorths
    # residual certificate of Eq. (4) on the returned triplets
    R = A.dense @ r1.V - r1.U * r1.S
    assert np.linalg.norm(R, axis=0).max() <= 1e-9 * r1.S[0]
    wl = W.config(1)
    v0 = np.random.default_rng(0).standard_normal(wl.A.n)
    a = O.svds(wl.A, wl.k, v0, tol=1e-10, maxit=30, reorth=1)
    b = O.svds(wl.A, wl.k, v0, tol=1e-10, maxit=30, reorth=2)
    assert a.converged and b.converged
    assert np.abs(a.S - b.S).max() <= 1e-12 * b.S[0]
    assert a.reorths < 0.2 * b.reorths


@pytest.mark.parametrize("t,k", [(60, 20), (31, 10), (12, 1)])
def test_pro_restart_against_inner_products(t, k):
    """or_pro_restart (the omega rows after an augmented restart, reading Q20):
    with V holding real Lanczos vectors that lost orthogonality and Vh a
    non-symmetric orthogonal t x t matrix, the new row of v_{k+1} = old v_{t+1}
    must equal the brute-force inner products v_{t+1}^T (V(:, 1:t) Vh(:, j))
    with the Ritz vectors Ṽ_k (Alg. 2 step 8); the row of u_{k+1}, which is
    re-orthogonalized in full, is eps, both diagonals are 1.
    A transposed Vh, a wrong column range or a dropped term fails."""
    A = decay2()
    U, V, T, _ = O.lbp(A, t, np.random.default_rng(t).standard_normal(A.n), reorth=0)
    nu = V[:, :t].T @ V[:, t]                       # row of the newest vector, brute force
    assert np.abs(nu).max() > 1e-6                 # orthogonality really lost (not all ~eps)
    Vh = np.linalg.qr(np.random.default_rng(k).standard_normal((t, t)))[0]
    assert np.abs(Vh - Vh.T).max() > 0.1
    nu_new, mu_new = O.pro_restart(t, k, Vh, nu, np.full(t, 0.5))
    ritz = V[:, :t] @ Vh[:, :k]                    # Ṽ_k
    true = ritz.T @ V[:, t]
    assert np.abs(nu_new[:k] - true).max() <= 1e-12 * max(1.0, np.abs(true).max())
    assert nu_new[k] == 1.0 and mu_new[k] == 1.0
    assert np.all(mu_new[:k] == EPS)
