"""ORACLE (test infrastructure only — see oracle/__init__.py).

The plain definitions ALP converges to (Thm 2c), for tiny codes:

  feldman_rows    every parity inequality of every check (eq.`constraints`),
                  2^{d_j - 1} per check, plus the boxes u_i <= 1 (u_i >= 0 implicit)
  simplex_min     dense tableau simplex with Bland's rule (P:388-397 background; a
                  from-scratch textbook method, independent of the IPM)
  lp_decode_full  u* = argmin gamma^T u over the fundamental polytope (eq.`LP decoding`)
  codewords       all codewords by brute force over {0,1}^n (n <= 22)
  ml_decode       argmin_{u in C} gamma^T u (eq.`ML decoding`)
"""
from __future__ import annotations

from itertools import combinations
import numpy as np


def feldman_rows(code):
    """Rows G, rhs h of G u <= h: all odd-V parity inequalities, then u_i <= 1."""
    n = code.n
    G, h = [], []
    for j in range(code.m):
        Nj = [int(i) for i in code.N(j)]
        d = len(Nj)
        for k in range(1, d + 1, 2):
            for V in combinations(Nj, k):
                row = np.zeros(n)
                row[list(Nj)] = -1.0
                row[list(V)] = 1.0
                G.append(row)
                h.append(len(V) - 1.0)
    for i in range(n):
        row = np.zeros(n)
        row[i] = 1.0
        G.append(row)
        h.append(1.0)
    return np.array(G), np.array(h)


def simplex_min(c, G, h, max_pivots=200000):
    """min c^T u s.t. G u <= h, u >= 0, with h >= 0 (so u = 0 is a feasible basis).

    Dense tableau over [G | I]; Bland's rule: entering = lowest-index column with a
    negative reduced cost, leaving = minimum ratio with ties to the lowest basic index.
    Returns (u, objective).
    """
    G = np.asarray(G, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    if np.any(h < 0):
        raise ValueError("simplex_min needs h >= 0")
    mrow, n = G.shape
    T = np.zeros((mrow + 1, n + mrow + 1))
    T[:mrow, :n] = G
    T[:mrow, n:n + mrow] = np.eye(mrow)
    T[:mrow, -1] = h
    T[-1, :n] = c                       # reduced costs (basis = slacks, cost 0)
    basis = list(range(n, n + mrow))
    eps = 1e-11
    for _ in range(max_pivots):
        rc = T[-1, :-1]
        enter = next((k for k in range(n + mrow) if rc[k] < -eps), None)
        if enter is None:
            break
        col = T[:mrow, enter]
        ratios = np.full(mrow, np.inf)
        pos = col > eps
        ratios[pos] = T[:mrow, -1][pos] / col[pos]
        best = np.min(ratios)
        if not np.isfinite(best):
            raise RuntimeError("unbounded")
        cand = [r for r in range(mrow) if ratios[r] <= best + 1e-12 * max(1.0, abs(best))]
        leave = min(cand, key=lambda r: basis[r])
        T[leave] /= T[leave, enter]
        for r in range(mrow + 1):
            if r != leave and T[r, enter] != 0.0:
                T[r] -= T[r, enter] * T[leave]
        basis[leave] = enter
    else:
        raise RuntimeError("simplex pivot cap")
    u = np.zeros(n + mrow)
    for r, bidx in enumerate(basis):
        u[bidx] = T[r, -1]
    u = u[:n]
    return u, float(c @ u)


def lp_decode_full(code, gamma):
    """The LP decoding optimum over the full fundamental polytope (eq.`LP decoding`)."""
    G, h = feldman_rows(code)
    return simplex_min(np.asarray(gamma, dtype=np.float64), G, h)


def codewords(code) -> np.ndarray:
    """All u in {0,1}^n with H u = 0 mod 2 (brute force, n <= 22)."""
    n = code.n
    if n > 22:
        raise ValueError("brute force limited to n <= 22")
    words = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1).astype(np.uint8)
    H = code.dense().astype(np.int64)
    ok = np.all((words.astype(np.int64) @ H.T) % 2 == 0, axis=1)
    return words[ok]


def ml_decode(code, gamma):
    """argmin over codewords of gamma^T u (eq.`ML decoding`).  Returns (u, cost, n_ties)."""
    C = codewords(code)
    costs = C.astype(np.float64) @ np.asarray(gamma, dtype=np.float64)
    k = int(np.argmin(costs))
    ties = int(np.sum(np.abs(costs - costs[k]) <= 1e-12 * max(1.0, abs(costs[k]))))
    return C[k], float(costs[k]), ties
