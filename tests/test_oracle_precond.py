"""Pins for the oracle's triangular preconditioner (§V) and PCG (Alg. 4).

Pins: hand traces of Alg. 6/7/8 (golden); direct verification of triangularity and
of M z = r by dense multiplication; Alg. 5 <=> no stopping set (independent peeling
loop); PCG special cases M = I (converges to the direct solve), M = Q (one
iteration), CG on a diagonal Q within the sqrt(kappa) bound of P:534.
"""
import json
import os

import numpy as np
import pytest

from oracle.precond import (mts_columnwise, mts_incremental, mts_rowwise, triangulation_step,
                            precond_apply, is_triangular_set, pcg)
from oracle.peeling import contains_stopping_set, rows_of_matrix
from oracle.lp import normal_matrix, cholesky_solve

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold():
    return json.load(open(os.path.join(GOLD, "precond_examples.json")))


def test_hand_traces():
    g = _gold()
    A = np.array(g["A"])
    w = np.array(g["w"], dtype=float)
    col, row = mts_columnwise(A, w)
    assert col == g["columnwise"]["col"] and row == g["columnwise"]["row"]
    col, row = mts_incremental(A, w)
    assert sorted(col) == g["incremental_set"]
    col, row = mts_rowwise(A, w)
    assert sorted(col) == g["rowwise_set"]


def test_step_system_example():
    s = _gold()["step_system"]
    A = np.array(s["A"], dtype=float)
    Q = normal_matrix(A, np.ones(5))
    np.testing.assert_array_equal(Q, s["Q"])
    np.testing.assert_allclose(cholesky_solve(Q, np.array(s["r"], float)), s["dy"], rtol=1e-14)
    col, row = mts_columnwise(A, np.ones(5))
    assert col == s["pivots_col"] and row == s["pivots_row"]
    AM = A[:, col]
    np.testing.assert_array_equal(AM @ AM.T, s["M"])


def _random_lp_matrix(rng, p=12, n=24, dv=3):
    A = np.zeros((p, n + p))
    for i in range(n):
        rows = rng.choice(p, size=dv, replace=False)
        A[rows, i] = rng.choice([-1.0, 1.0], size=dv)
    A[:, n:] = np.eye(p)
    return A


@pytest.mark.parametrize("seed", range(10))
def test_greedy_sets_are_triangular_and_apply_inverts_M(seed):
    rng = np.random.default_rng(seed)
    A = _random_lp_matrix(rng)
    p, q = A.shape
    d2 = 10.0 ** rng.uniform(-6, 6, q)
    for algo in (mts_columnwise, mts_incremental, mts_rowwise):
        col, row = algo(A, d2)
        assert len(col) == p and len(set(col)) == p and sorted(row) == list(range(p))
        assert is_triangular_set(A, col, row)
        r = rng.normal(size=p)
        z = precond_apply(A, d2, col, r)
        AM = A[:, col]
        M = AM @ np.diag(d2[col]) @ AM.T
        # backward error of the 3-stage solve (multiply back)
        scale = np.linalg.norm(np.abs(M) @ np.abs(z)) + np.linalg.norm(r)
        assert np.linalg.norm(M @ z - r) <= 1e-12 * scale
    # column-wise: upper triangular in pick order
    col, row = mts_columnwise(A, d2)
    T = A[np.ix_(row, col)] != 0
    assert np.all(np.tril(T, -1) == 0)


def test_columnwise_picks_max_weight_degree1_each_step():
    rng = np.random.default_rng(42)
    A = _random_lp_matrix(rng, p=15, n=30)
    w = rng.uniform(size=A.shape[1])
    col, row = mts_columnwise(A, w)
    live = np.ones(A.shape[0], dtype=bool)
    for c, r in zip(col, row):
        deg = ((A[live] != 0).sum(axis=0))
        cand = [i for i in range(A.shape[1]) if deg[i] == 1]
        best = max(cand, key=lambda i: (w[i], -i))
        assert c == best
        live[r] = False


def test_triangulation_step_iff_no_stopping_set():
    rng = np.random.default_rng(5)
    for _ in range(200):
        A = _random_lp_matrix(rng, p=8, n=14)
        q = A.shape[1]
        S = list(rng.choice(q, size=rng.integers(1, 9), replace=False))
        ok = triangulation_step(A, S) is not None
        # extended Tanner graph: variable nodes = columns; checks = rows
        rows = rows_of_matrix(A)
        assert ok == (not contains_stopping_set(rows, S))


def test_pcg_special_cases():
    rng = np.random.default_rng(9)
    B = rng.normal(size=(20, 20))
    Q = B @ B.T + np.eye(20)
    w = rng.normal(size=20)
    x, it, rel, st = pcg(lambda v: Q @ v, w, None, tol=1e-12, maxit=200)
    assert st == 0
    np.testing.assert_allclose(x, np.linalg.solve(Q, w), rtol=1e-8)
    # M = Q: one iteration
    x, it, rel, st = pcg(lambda v: Q @ v, w, lambda r: np.linalg.solve(Q, r), tol=1e-10)
    assert it == 1 and st == 0
    # diagonal Q, kappa = 1e4: iterations within the sqrt(kappa) bound of P:534
    D = np.diag(np.linspace(1.0, 1e4, 200))
    w = rng.normal(size=200)
    x, it, rel, st = pcg(lambda v: D @ v, w, None, tol=1e-8, maxit=5000)
    bound = np.ceil(0.5 * np.sqrt(1e4) * np.log(2 / 1e-8 * np.sqrt(1e4)))
    assert st == 0 and it <= bound


def test_precond_pcg_on_decoding_like_system():
    """With the column-wise preconditioner PCG reaches 1e-8 far sooner than plain CG
    on a log-uniform (late-IPM-like) weighting (qualitative P:820-822)."""
    rng = np.random.default_rng(11)
    A = _random_lp_matrix(rng, p=60, n=120)
    d2 = 10.0 ** rng.uniform(-6, 6, A.shape[1])
    Q = normal_matrix(A, d2)
    w = rng.normal(size=60)
    col, _ = mts_columnwise(A, d2)
    xp, itp, relp, stp = pcg(lambda v: Q @ v, w, lambda r: precond_apply(A, d2, col, r), tol=1e-8, maxit=2000)
    xc, itc, relc, stc = pcg(lambda v: Q @ v, w, None, tol=1e-8, maxit=2000)
    assert stp == 0 and itp < itc
