"""Pins for the oracle's interior-point method (§IV-B).

Pins: the 3x3-block Newton system eq.`matrix equation` solved densely and directly
(textbook reduction) agrees with the normal-equation recovery eq.`Delta y/x/z`;
hand-worked 2x2 normal system; step-length arithmetic; Cholesky step vs LAPACK
solve; final IPM point vs an independent solver (scipy HiGHS) on random pool LPs.
"""
import numpy as np
import pytest
from scipy.optimize import linprog

from oracle.lp import (newton_direction, step_lengths, ipm_solve, cholesky_solve, step_solve_exact,
                       normal_matrix, augmented_lp, DEFAULT_PARAMS, find_violated_cut)
from synth.codes import regular_code


def test_newton_block_system_matches_dense_direct():
    rng = np.random.default_rng(1)
    for _ in range(20):
        p, n = 4, 7
        q = n + p
        A = np.zeros((p, q))
        A[:, :n] = rng.choice([-1.0, 0.0, 1.0], size=(p, n), p=[0.3, 0.4, 0.3])
        A[:, n:] = np.eye(p)
        x = rng.uniform(0.1, 2, q)
        z = rng.uniform(0.1, 2, q)
        rb = rng.normal(size=p)
        rc = rng.normal(size=q)
        mu = 0.3
        dx, dy, dz = newton_direction(A, x, z, rb, rc, mu)
        # eq.`matrix equation`: [A 0 0; 0 A^T I; Z 0 X] [dx dy dz] = [rb rc re]
        K = np.zeros((p + 2 * q, 2 * q + p))
        K[:p, :q] = A
        K[p:p + q, q:q + p] = A.T
        K[p:p + q, q + p:] = np.eye(q)
        K[p + q:, :q] = np.diag(z)
        K[p + q:, q + p:] = np.diag(x)
        rhs = np.concatenate([rb, rc, mu - x * z])
        sol = np.linalg.solve(K, rhs)
        np.testing.assert_allclose(dx, sol[:q], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(dy, sol[q:q + p], rtol=1e-9, atol=1e-10)
        np.testing.assert_allclose(dz, sol[q + p:], rtol=1e-9, atol=1e-10)


def test_normal_system_hand_example():
    # A = [[1,1,0],[0,1,1]], D = I: Q = [[2,1],[1,2]]; Q dy = (1,1) -> dy = (1/3, 1/3)
    A = np.array([[1.0, 1, 0], [0, 1, 1]])
    Q = normal_matrix(A, np.ones(3))
    np.testing.assert_array_equal(Q, [[2, 1], [1, 2]])
    np.testing.assert_allclose(cholesky_solve(Q, np.array([1.0, 1.0])), [1 / 3, 1 / 3], rtol=1e-15)


def test_step_lengths_examples():
    assert step_lengths(np.array([1.0, 1]), np.ones(2), np.array([-2.0, 1]), np.zeros(2), 0.99)[0] == pytest.approx(0.495)
    assert step_lengths(np.array([1.0, 1]), np.ones(2), np.array([2.0, 1]), np.zeros(2), 0.99)[0] == 1.0
    assert step_lengths(np.array([1.0, 0.1]), np.ones(2), np.array([-1.0, -1]), np.zeros(2), 0.99)[0] == pytest.approx(0.099)


def test_cholesky_vs_lapack_and_safeguard():
    rng = np.random.default_rng(3)
    B = rng.normal(size=(30, 30))
    Q = B @ B.T + 30 * np.eye(30)
    w = rng.normal(size=30)
    np.testing.assert_allclose(cholesky_solve(Q, w), np.linalg.solve(Q, w), rtol=1e-12)
    # singular Q: the safeguard (C-29) keeps the solve finite and zeroes the null direction
    Qs = np.array([[1.0, 1.0], [1.0, 1.0]])
    info = {}
    dy = cholesky_solve(Qs, np.array([2.0, 2.0]), info)
    assert info["chol_fixes"] == 1 and np.all(np.isfinite(dy))
    np.testing.assert_allclose(Qs @ dy, [2.0, 2.0], rtol=1e-12)


def _random_pool_lp(seed, n=24, dv=3, dc=6):
    rng = np.random.default_rng(seed)
    code = regular_code(n, dv, dc, seed=seed)
    gamma = rng.normal(1.0, 1.5, n)
    u = rng.uniform(size=n)
    pool = {}
    for j in range(code.m):
        V, lhs, _ = find_violated_cut(u[code.N(j)])
        if rng.uniform() < 0.7:
            pool[j] = V
    return code, gamma, pool


@pytest.mark.parametrize("seed", range(12))
def test_ipm_matches_highs(seed):
    code, gamma, pool = _random_pool_lp(seed)
    lp = augmented_lp(code, pool, gamma)
    res = ipm_solve(lp["A"], lp["b"], lp["c"])
    assert res["status"] == 0
    ref = linprog(lp["c"], A_eq=lp["A"], b_eq=lp["b"], bounds=[(0, None)] * lp["q"], method="highs")
    assert ref.status == 0
    obj = float(lp["c"] @ res["x"])
    assert obj == pytest.approx(ref.fun, rel=1e-7, abs=1e-7)
    # primal feasibility at the C-8 tolerance and positivity
    assert np.max(np.abs(lp["A"] @ res["x"] - lp["b"])) <= 1e-8 * (1 + np.max(np.abs(lp["b"])))
    assert np.all(res["x"] > 0) and np.all(res["z"] > 0)


def test_augmented_form_hand_examples():
    from synth.codes import code_from_rows
    code = code_from_rows([[0, 1, 2]], 3)
    # V = N(j), no flips: u1+u2+u3 <= 2 -> x1+x2+x3+s = 2
    lp = augmented_lp(code, {0: np.array([True, True, True])}, np.array([1.0, 1.0, 1.0]))
    np.testing.assert_array_equal(lp["A"], [[1, 1, 1, 1]])
    assert lp["b"][0] == 2
    # gamma_2 < 0 flips x2 = 1 - u2: x1 - x2 + x3 + s = 1
    lp = augmented_lp(code, {0: np.array([True, True, True])}, np.array([1.0, -1.0, 1.0]))
    np.testing.assert_array_equal(lp["A"], [[1, -1, 1, 1]])
    assert lp["b"][0] == 1
    np.testing.assert_array_equal(lp["c"], [1, 1, 1, 0])


def test_empty_pool_lp_optimum_is_zero():
    A = np.zeros((0, 3))
    res = ipm_solve(A, np.zeros(0), np.array([1.0, 2.0, 3.0]))
    assert res["status"] == 0
    assert np.max(res["x"]) < 1e-8


def _exact_rational_solve(A, d2, w):
    """Gauss-Jordan over the rationals (fractions.Fraction): the exact solution."""
    from fractions import Fraction as Fr
    p, q = A.shape
    d2f = [Fr(float(v)) for v in d2]
    Q = [[sum(Fr(int(A[a, i])) * d2f[i] * Fr(int(A[b, i])) for i in range(q) if A[a, i] and A[b, i])
          for b in range(p)] for a in range(p)]
    M = [Q[a] + [Fr(float(w[a]))] for a in range(p)]
    for k in range(p):
        piv = next(r for r in range(k, p) if M[r][k] != 0)
        M[k], M[piv] = M[piv], M[k]
        for r in range(p):
            if r != k and M[r][k] != 0:
                f = M[r][k] / M[k][k]
                M[r] = [a - f * b for a, b in zip(M[r], M[k])]
    return np.array([float(M[k][p] / M[k][k]) for k in range(p)])


@pytest.mark.parametrize("seed,span", [(0, 2), (1, 8), (2, 14), (3, 20), (4, 24)])
def test_step_solve_exact_matches_rational_solution(seed, span):
    """Pin: on small config-5-like systems (one random odd cut per check, slack columns, d^2
    log-uniform over span decades, kappa up to ~1e20+) the refined solve equals the exact
    rational solution (Gaussian elimination in fractions) to 1e-14 relative; fp64 Cholesky is
    off by ~4e-9 already at kappa 1e10, long-double refinement alone by up to ~1e-7."""
    from synth import c5_systems
    from tests.helpers import dense_step_matrix, step_weights
    code = regular_code(24, 3, 6, seed=10 + seed)
    sy = c5_systems([seed], code, lo=-span / 2, hi=span / 2)
    A, rows = dense_step_matrix(code, sy.masks[0])
    d2 = step_weights(code, sy.d[0], rows)
    w = sy.r[0][rows]
    exact = _exact_rational_solve(A, d2, w)
    got = step_solve_exact(A, d2, w)
    assert np.linalg.norm(got - exact) <= 1e-14 * np.linalg.norm(exact)


def test_step_solve_exact_agrees_with_lapack_when_well_conditioned():
    rng = np.random.default_rng(5)
    code = regular_code(60, 3, 6, seed=3)
    from synth import c5_systems
    from tests.helpers import dense_step_matrix, step_weights
    sy = c5_systems([7], code, lo=-0.5, hi=0.5)
    A, rows = dense_step_matrix(code, sy.masks[0])
    d2 = step_weights(code, sy.d[0], rows)
    w = rng.normal(size=len(rows))
    np.testing.assert_allclose(step_solve_exact(A, d2, w), np.linalg.solve(normal_matrix(A, d2), w),
                               rtol=1e-12)
