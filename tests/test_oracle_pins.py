"""Pins of the CPU oracle (oracle/oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.  CPU only (-m "not gpu").

Each test names the oracle part it pins and the passage it follows.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from helpers import certificates, gamma, orth_error, sin_max_angle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# kernels: spmv / spmv_t / gemv / norm2 / project_out
def test_spec_hand_examples():
    g = gold("spec_examples.json")
    for e in g["spmv"]:
        A = W.csr_from_dense(np.array(e["A"], float))
        assert np.array_equal(O.spmv(A, e["x"]), np.array(e["y"], float)), e["cite"]
    for e in g["spmv_t"]:
        A = W.csr_from_dense(np.array(e["A"], float))
        assert np.array_equal(O.spmv_t(A, e["x"]), np.array(e["y"], float)), e["cite"]
    for e in g["gemv"]:
        A = W.dense_matrix(np.array(e["A"], float))
        assert np.array_equal(O.spmv(A, e["x"]), np.array(e["y"], float)), e["cite"]
    for e in g["project_out"]:
        out = O.cgs2(np.array(e["Q"], float), np.array(e["w"], float))
        assert np.array_equal(out, np.array(e["out"], float)), e["cite"]
    for e in g["norm2"]:
        assert O.norm2(e["x"]) == e["out"], e["cite"]
    for e in g["svd"]:
        _, S, _, _ = O.jacobi_svd(np.array(e["M"], float))
        assert np.allclose(S, e["S"], rtol=0, atol=1e-15), e["cite"]


@pytest.mark.parametrize("seed", range(5))
def test_spmv_matches_dense_expansion(seed):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((20, 15)) * (rng.random((20, 15)) < 0.3)
    D[3, :] = 0.0  # an empty row
    A = W.csr_from_dense(D)
    x, u = rng.standard_normal(15), rng.standard_normal(20)
    # reduction-order budget per element: gamma_{len+2} * sum |a x|
    y, yt = O.spmv(A, x), O.spmv_t(A, u)
    assert np.all(np.abs(y - D @ x) <= gamma(17) * (np.abs(D) @ np.abs(x)) + 1e-300)
    assert np.all(np.abs(yt - D.T @ u) <= gamma(22) * (np.abs(D.T) @ np.abs(u)) + 1e-300)
    Dd = W.dense_matrix(D)
    assert np.allclose(O.spmv(Dd, x), D @ x, rtol=1e-14, atol=1e-14)
    assert np.allclose(O.spmv_t(Dd, u), D.T @ u, rtol=1e-14, atol=1e-14)


def test_cgs2_orthogonality_and_idempotence():
    rng = np.random.default_rng(3)
    for N, c in [(10, 4), (200, 30), (1000, 150)]:
        Q = np.linalg.qr(rng.standard_normal((N, c)))[0]
        w = rng.standard_normal(N)
        w1 = O.cgs2(Q, w)
        assert np.abs(Q.T @ w1).max() <= 1e-13 * np.linalg.norm(w)
        w2 = O.cgs2(Q, w1)
        assert np.linalg.norm(w2 - w1) <= 1e-14 * np.linalg.norm(w)
        # the projection removes exactly the span: (I - QQ^T) w
        assert np.allclose(w1, w - Q @ (Q.T @ w), atol=1e-13 * np.linalg.norm(w))


# --------------------------------------------------------------------------
# small SVD: one-sided Jacobi (Alg. 2 step 4)
def test_jacobi_vs_numpy_svd_many():
    rng = np.random.default_rng(11)
    for it in range(1000):
        p = int(rng.integers(1, 65))
        q = int(rng.integers(1, p + 1))
        M = rng.uniform(-1, 1, (p, q))
        if it % 7 == 0:
            M[:, rng.integers(0, q)] = 0.0  # rank deficiency
        U, S, V, _ = O.jacobi_svd(M)
        ref = np.linalg.svd(M, compute_uv=False)
        nrm = max(1.0, np.linalg.norm(M))
        assert np.abs(S - ref).max() <= 1e-12 * nrm
        assert np.all(np.diff(S) <= 0)
        assert orth_error(U) <= 1e-12 and orth_error(V) <= 1e-12
        assert np.linalg.norm(M - (U * S) @ V.T) <= 1e-12 * nrm


def test_jacobi_sign_rule_scale_transpose():
    rng = np.random.default_rng(5)
    M = rng.uniform(-1, 1, (9, 9))
    U, S, V, _ = O.jacobi_svd(M)
    for j in range(9):
        i = np.argmax(np.abs(U[:, j]))
        assert U[i, j] >= 0
    _, S3, _, _ = O.jacobi_svd(3.0 * M)
    assert np.allclose(S3, 3.0 * S, rtol=1e-12, atol=0)
    _, St, _, _ = O.jacobi_svd(M.T.copy())
    assert np.allclose(St, S, rtol=1e-12, atol=0)
    # diag(3,1,2): permuted identity up to sign
    U, S, V, _ = O.jacobi_svd(np.diag([3.0, 1.0, 2.0]))
    assert np.array_equal(S, [3.0, 2.0, 1.0])
    assert np.array_equal(np.abs(U), np.abs(V))


# --------------------------------------------------------------------------
# LBP = Alg. 1 + full re-orthogonalization
def test_lbp_exact_on_diagonal():
    e = gold("spec_examples.json")["lbp_diag"][0]
    A = W.dense_matrix(np.array(e["A"], float))
    U, V, T, info = O.lbp(A, e["t"], np.array([1.0, 1.0, 1.0]))
    S = np.linalg.svd(T, compute_uv=False)
    assert np.allclose(S, e["S"], atol=1e-12), e["cite"]


@pytest.mark.parametrize("sparse", [False, True])
def test_lbp_recurrence_orthogonality_matvecs(sparse):
    rng = np.random.default_rng(8)
    D = rng.standard_normal((40, 30)) * (rng.random((40, 30)) < (0.4 if sparse else 1.0))
    A = W.csr_from_dense(D) if sparse else W.dense_matrix(D)
    t = 9
    U, V, T, info = O.lbp(A, t, rng.standard_normal(30))
    smax = np.linalg.svd(T[:t, :t], compute_uv=False)[0]
    for i in range(t):  # 0-based column i = paper's i+1
        a, b = T[i, i], T[i, i + 1]
        r1 = D.T @ U[:, i] - a * V[:, i] - b * V[:, i + 1]       # Alg. 1 line 5
        r2 = D @ V[:, i + 1] - b * U[:, i] - T[i + 1, i + 1] * U[:, i + 1]  # line 7
        assert np.linalg.norm(r1) <= 1e-10 * smax
        assert np.linalg.norm(r2) <= 1e-10 * smax
    assert orth_error(U) <= 1e-10 and orth_error(V) <= 1e-10
    assert info.matvecs == 2 * t + 1  # Eq. (8) (2t+1) nnz term
    # T is upper bidiagonal with nonnegative entries
    assert np.allclose(np.triu(np.tril(T, 1)), T) and np.all(T >= 0)


def test_reorth_is_load_bearing():
    """PAPER.md:121 'suffer from losing orthogonality': without re-orth the
    basis loses orthogonality on a Decay1 matrix (acceptance 6)."""
    A = W.dense_with_spectrum(300, 200, W.spectrum("decay1", 200), seed=1)
    v0 = W.start_vector(200, 1)
    _, V0, _, _ = O.lbp(A, 60, v0, reorth=0)
    _, V2, _, _ = O.lbp(A, 60, v0, reorth=2)
    assert orth_error(V0) > 1e-6
    assert orth_error(V2) <= 1e-10


def test_breakdown_scaled_identity():
    """A = c I: alpha_1 = c, beta_1 collapses -> breakdown path."""
    A = W.dense_matrix(2.5 * np.eye(5))
    U, V, T, info = O.lbp(A, 3, np.arange(1.0, 6.0))
    assert info.breakdowns >= 1
    assert abs(T[0, 0] - 2.5) < 1e-14 and T[0, 1] == 0.0
    assert orth_error(U) <= 1e-12 and orth_error(V) <= 1e-12


def test_breakdown_generator_definition():
    """Counter-based replacement vectors (Q7): SplitMix64 of
    (seed, stream, r), 53 bits -> [-1, 1).  Checked against an independent
    Python transcription of the documented definition."""
    M64 = (1 << 64) - 1

    def sm(z):
        z = (z + 0x9E3779B97F4A7C15) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def ref(seed, stream, r):
        key = sm(seed ^ sm((stream * 0xD1B54A32D192ED03 + 1) & M64))
        z = sm((key + r * 0x9E3779B97F4A7C15) & M64)
        return (z >> 11) * 2.0 ** -53 * 2.0 - 1.0

    got = O.breakdown_uniform(7, 3, 16)
    assert np.array_equal(got, [ref(7, 3, r) for r in range(16)])
    assert np.all(got >= -1) and np.all(got < 1)


# --------------------------------------------------------------------------
# svds = Alg. 2
def test_svds_diagonal_trivial():
    e = gold("spec_examples.json")["svds_diag"][0]
    D = np.diag(np.array(e["A_diag"], float))
    # t is clamped to min(m,n)-1 = 1 < k+2 -> contract violation
    with pytest.raises(RuntimeError):
        O.svds(W.dense_matrix(D), e["k"], np.ones(2))
    # the same spectrum embedded in a 6x6 diagonal solves exactly
    D6 = np.diag([2.0, 1.0, 0.5, 0.25, 0.125, 0.0625])
    r = O.svds(W.dense_matrix(D6), 1, np.ones(6), t=4)
    assert abs(r.S[0] - 2.0) < 1e-14 and r.converged
    assert abs(abs(r.U[0, 0]) - 1) < 1e-12 and abs(abs(r.V[0, 0]) - 1) < 1e-12


def test_svds_random_small_vs_numpy():
    """>= 200 random matrices m, n <= 64, dense and sparse."""
    rng = np.random.default_rng(2024)
    count = 0
    while count < 200:
        m, n = int(rng.integers(12, 65)), int(rng.integers(12, 65))
        k = int(rng.integers(1, 9))
        if min(m, n) - 1 < k + 2:
            continue
        D = rng.standard_normal((m, n))
        if count % 2:
            D *= rng.random((m, n)) < 0.5
            A = W.csr_from_dense(D)
        else:
            A = W.dense_matrix(D)
        r = O.svds(A, k, rng.standard_normal(n), maxit=100)
        ref = np.linalg.svd(D, compute_uv=False)
        if r.converged:
            keep = ref[:k] > 1e-12 * ref[0]
            assert np.all(np.abs(r.S - ref[:k])[keep] <= 1e-8 * ref[:k][keep])
            count += 1


@pytest.mark.parametrize("kind", ["decay1", "decay2", "decay3"])
def test_svds_decay_certificates(kind):
    """Acceptance 2/3/6: Eq. (4) residual equals ||A^T u - s v|| / s (Prop. 1,
    PAPER.md:130-143); Decay2 recovers i^-2."""
    A = W.dense_with_spectrum(500, 400, W.spectrum(kind, 400), seed=2)
    r = O.svds(A, 10, W.start_vector(400, 2))
    assert r.converged and np.all(r.resid < 1e-10)
    r1, r2 = certificates(A, r.S, r.U, r.V)
    assert np.all(r1 <= 1e-10 * r.S[0])
    assert np.all(np.abs(r2 - r.resid) <= 1e-8)
    assert orth_error(r.U) <= 1e-10 and orth_error(r.V) <= 1e-10
    sig = W.spectrum(kind, 10)
    assert np.all(np.abs(r.S - sig) <= 1e-8 * sig)


def test_svds_repeated_singular_values():
    """Acceptance 4 (LargeRegFile analog)."""
    s = np.concatenate([np.ones(10), 0.5 * np.ones(10), 1e-3 * 0.9 ** np.arange(280)])
    A = W.dense_with_spectrum(300, 300, s, seed=4)
    r = O.svds(A, 15, W.start_vector(300, 4))
    assert r.converged
    assert np.all(np.abs(r.S[:10] - 1.0) <= 1e-8)
    assert np.all(np.abs(r.S[10:15] - 0.5) <= 1e-8)


def test_svds_forced_restart_and_matvec_count():
    """Acceptance 5 + 7: t = k + 3 forces restarts (Eqs. 5-7); matvecs =
    (2t+1) + R (2(t-k)+1)  (Eq. (8), reading Q2)."""
    A = W.dense_with_spectrum(500, 400, W.spectrum("decay1", 400), seed=5)
    k, t = 10, 13
    r = O.svds(A, k, W.start_vector(400, 5), t=t, maxit=500)
    assert r.restarts >= 1 and r.converged
    R = r.restarts
    assert r.matvecs == (2 * t + 1) + R * (2 * (t - k) + 1)
    assert r.steps == t + R * (t - k)
    r1, r2 = certificates(A, r.S, r.U, r.V)
    assert np.all(r1 <= 1e-10 * r.S[0]) and np.all(np.abs(r2 - r.resid) <= 1e-8)
    sig = W.spectrum("decay1", 10)
    assert np.all(np.abs(r.S - sig) <= 1e-8 * sig)


def test_restart_identities_unconverged():
    """After each restart Prop. 1 still holds: A v_j = s_j u_j and the Eq. (4)
    residual equals ||A^T u_j - s_j v_j|| / s_j.  A wrong
    Eq. (6)/(7) coefficient breaks the first identity."""
    wl = W.config(1, seed=3)
    for passes in (1, 2, 3):
        r = O.svds(wl.A, wl.k, wl.v0, t=wl.t, fixed_passes=passes)
        assert r.passes == passes
        r1, r2 = certificates(wl.A, r.S, r.U, r.V)
        assert np.all(r1 <= 1e-10 * r.S[0])
        assert np.all(np.abs(r2 - r.resid) <= 1e-8 * max(1.0, r.resid.max()))
        assert orth_error(r.U) <= 1e-10 and orth_error(r.V) <= 1e-10


def test_svds_deterministic():
    wl = W.config(1, seed=1, scale=2)
    a = O.svds(wl.A, wl.k, wl.v0, t=wl.t)
    b = O.svds(wl.A, wl.k, wl.v0, t=wl.t)
    assert a.S.tobytes() == b.S.tobytes() and a.U.tobytes() == b.U.tobytes()
    assert a.V.tobytes() == b.V.tobytes() and a.resid.tobytes() == b.resid.tobytes()


def test_config1_vs_library_svd():
    """BASELINE config 1: sigma within 1e-10 sigma_1 of numpy.linalg.svd of the
    dense expansion; subspaces within the Wedin bound tol s sqrt(k) / gap."""
    wl = W.config(1)
    r = O.svds(wl.A, wl.k, wl.v0, t=wl.t, maxit=wl.maxit)
    assert r.converged
    D = wl.A.to_dense()
    Uf, s, Vt = np.linalg.svd(D, full_matrices=False)
    k = wl.k
    assert np.abs(r.S - s[:k]).max() <= 1e-10 * s[0]
    gap = s[k - 1] - s[k]
    bound = 10 * wl.tol * s[0] * np.sqrt(k) / gap
    assert sin_max_angle(Uf[:, :k], r.U) <= bound
    assert sin_max_angle(Vt[:k].T, r.V) <= bound


def test_config2_closed_form_scaled():
    """BASELINE config 2 recipe at 1/4 size: sigma_i = exp(-i/40) closed form and
    the generator's known singular subspaces."""
    wl = W.config(2, scale=4, keep_factors=True)
    r = O.svds(wl.A, wl.k, wl.v0, t=wl.t, maxit=wl.maxit)
    assert r.converged
    sig = W.spectrum("exp40", wl.k)
    assert np.abs(r.S - sig).max() <= 1e-10 * sig[0]
    gap = np.exp(-wl.k / 40) - np.exp(-(wl.k + 1) / 40)
    bound = 10 * 1e-10 * np.sqrt(wl.k) / gap
    assert sin_max_angle(wl.A.meta["QU"][:, :wl.k], r.U) <= bound
    assert sin_max_angle(wl.A.meta["QV"][:, :wl.k], r.V) <= bound


def test_decay_spectra_golden():
    g = gold("decay_spectra.json")
    for kind in ("decay1", "decay2", "decay3", "exp40"):
        e = g[kind]
        s = W.spectrum(kind, max(e["i"]))
        got = s[np.array(e["i"]) - 1]
        assert np.allclose(got, e["sigma"], rtol=1e-15, atol=0), e["cite"]


@pytest.mark.parametrize("cid", [6, 7, 8])
def test_dense1_3_closed_form(cid):
    """Dense1-3 at 1/20 scale: the oracle's
    k = 100 Ritz values equal the Decay1/2/3 spectra of Eq. (16),
    which the generator imposes exactly (closed form), and its residual
    certificates hold."""
    wl = W.config(cid, scale=20)
    r = O.svds(wl.A, wl.k, wl.v0, tol=wl.tol, t=wl.t, maxit=wl.maxit)
    sig = W.spectrum(f"decay{cid - 5}", wl.A.m)[: wl.k]
    assert r.converged
    assert np.abs(r.S - sig).max() <= 1e-10 * sig[0]
    D = wl.A.dense
    assert np.linalg.norm(D @ r.V - r.U * r.S, axis=0).max() <= 1e-10 * sig[0]
