"""ORACLE (test infrastructure only — see oracle/__init__.py).

Triangular ("encoding-like") preconditioner of PAPER.md §V and PCG (Alg. 4).

A is given by its sparsity pattern and signs as a dense p x q array (rows = LP
constraints, columns = standard variables then slack variables).  Weights w are
the column weights the greedy searches rank by (d_i or d_i^2 = x_i / z_i: same
order, reading C-10); ties go to the lower column index (C-10).

  triangulation_step   Alg. 5 (G10: zero rows ignored, "any degree-1
                       row" = lowest row index)
  mts_incremental      Alg. 6 (G9: S <- M u {pi_i}, keep if triangulable)
  mts_columnwise       Alg. 7 with a binary heap
  mts_rowwise          Alg. 8 with diagonal expansion (line 14, G11)
  precond_apply        M^-1 r with M = A_M D_M^2 A_M^T by A_M f1 = r, D_M^2 f2 = f1,
                       A_M^T z = f2
  pcg                  Alg. 4, x0 = 0, stop on ||r|| <= tol ||w|| (C-9)
"""
from __future__ import annotations

import heapq
import numpy as np


def _pattern(A):
    A = np.asarray(A)
    rows = [list(np.nonzero(A[j])[0]) for j in range(A.shape[0])]
    cols = [list(np.nonzero(A[:, i])[0]) for i in range(A.shape[1])]
    return rows, cols


def mts_columnwise(A, w):
    """Alg. 7, column-wise greedy search for the MTS.

    DEG1 (line 4) = columns of the residual matrix with exactly one nonzero; each of the
    p steps (lines 5-9) takes the max-weight column i in DEG1 (ties -> lower index) and
    its unique live row j, records (i, j), zeroes row j, and updates DEG1.  A binary heap
    with lazy deletion holds DEG1.  Returns (col, row): the pivot sequence.
    Column i picked at step k has live rows only among earlier-killed rows, so A_M with
    rows in `row` order and columns in `col` order is upper triangular.
    """
    A = np.asarray(A)
    p, q = A.shape
    rows, cols = _pattern(A)
    live_row = np.ones(p, dtype=bool)
    deg = np.array([len(c) for c in cols])
    heap = [(-float(w[i]), i) for i in range(q) if deg[i] == 1]
    heapq.heapify(heap)
    picked = np.zeros(q, dtype=bool)
    col_seq, row_seq = [], []
    for _ in range(p):
        while True:
            negw, i = heapq.heappop(heap)
            if deg[i] == 1 and not picked[i]:
                break
        j = next(r for r in cols[i] if live_row[r])
        picked[i] = True
        col_seq.append(i)
        row_seq.append(j)
        live_row[j] = False
        for i2 in rows[j]:
            deg[i2] -= 1
            if deg[i2] == 1 and not picked[i2]:
                heapq.heappush(heap, (-float(w[i2]), i2))
    return col_seq, row_seq


def triangulation_step(A, S):
    """Alg. 5: peel the columns S of A (erasure decoding on the extended Tanner graph).

    Repeatedly take a row of A~ = A_S with exactly one nonzero (lowest row index), record
    (column, row), and zero that column and row.  Fails (returns None) when no row has
    degree exactly 1 before s picks (G10).  On success returns (col, row) such that A_S
    with rows `row` and columns `col` is lower triangular.
    """
    A = np.asarray(A)
    S = list(S)
    sub = (A[:, S] != 0).astype(np.int64)
    alive_c = np.ones(len(S), dtype=bool)
    col_seq, row_seq = [], []
    for _ in range(len(S)):
        rdeg = sub[:, alive_c].sum(axis=1)
        cand = np.nonzero(rdeg == 1)[0]
        if cand.size == 0:
            return None
        j = int(cand[0])
        loc = [t for t in np.nonzero(sub[j])[0] if alive_c[t]]
        t = loc[0]
        col_seq.append(S[t])
        row_seq.append(j)
        alive_c[t] = False
        sub[j, :] = 0
    return col_seq, row_seq


def mts_incremental(A, w):
    """Alg. 6: sort columns by weight (descending, ties -> lower index), add each column
    whose inclusion keeps the set triangulable (G9), until |M| = p.  O(q^2)."""
    A = np.asarray(A)
    p, q = A.shape
    order = sorted(range(q), key=lambda i: (-float(w[i]), i))
    M: list = []
    res = None
    for i in order:
        if len(M) >= p:
            break
        S = M + [i]
        r = triangulation_step(A, S)
        if r is not None:
            M, res = S, r
    return res  # (col, row) lower-triangular ordering of M


def mts_rowwise(A, w):
    """Alg. 8, row-wise greedy search with diagonal expansion.

    While A~ is not all zero: if a degree-1 row exists take the lowest-index one, record
    its unique column, zero that column; else zero the nonzero column of minimum weight
    (ties -> lower index).  Diagonal expansion (line 14): every row not represented gets
    its own slack column.  The slack column of row j is the unique column whose only
    nonzero is in row j among the last p columns (n + j).
    """
    A = np.asarray(A)
    p, q = A.shape
    n = q - p
    At = (A != 0).astype(np.int64)
    col_seq, row_seq = [], []
    used_rows = set()
    while At.any():
        rdeg = At.sum(axis=1)
        cand = [j for j in np.nonzero(rdeg == 1)[0]]
        if cand:
            j = int(cand[0])
            i = int(np.nonzero(At[j])[0][0])
            col_seq.append(i)
            row_seq.append(j)
            used_rows.add(j)
            At[:, i] = 0
        else:
            nzc = [i for i in range(q) if At[:, i].any()]
            i = min(nzc, key=lambda i: (float(w[i]), i))
            At[:, i] = 0
    for j in range(p):
        if j not in used_rows:
            col_seq.append(n + j)
            row_seq.append(j)
    return col_seq, row_seq


def precond_apply(A, w2, col_seq, z_rhs):
    """z = M^-1 r with M = A_M D_M^2 A_M^T: solve A_M f1 = r, f2 = f1 / d_M^2,
    A_M^T z = f2.  w2 are the squared weights d^2 (the diagonal of D^2)."""
    A = np.asarray(A, dtype=np.float64)
    AM = A[:, list(col_seq)]
    f1 = np.linalg.solve(AM, z_rhs)
    f2 = f1 / np.asarray(w2, dtype=np.float64)[list(col_seq)]
    return np.linalg.solve(AM.T, f2)


def is_triangular_set(A, col_seq, row_seq) -> bool:
    """A with rows `row_seq` and columns `col_seq` is triangular (upper or lower) with a
    nonzero diagonal."""
    A = np.asarray(A)
    T = A[np.ix_(list(row_seq), list(col_seq))] != 0
    if not np.all(np.diag(T)):
        return False
    return bool(np.all(np.triu(T, 1) == 0) or np.all(np.tril(T, -1) == 0))


def pcg(Qmul, w, Minv=None, tol=1e-8, maxit=1000, record=False):
    """Alg. 4 with x0 = 0 (C-9).  Stops after line 9 once
    ||r^{i+1}||_2 <= tol ||w||_2 (un-squared, G15).  Breakdown if h^T l <= 0.
    Returns (x, iters, relres, status) with status 0 ok, 4 maxiter, 8 breakdown."""
    w = np.asarray(w, dtype=np.float64)
    Minv = Minv or (lambda r: r.copy())
    x = np.zeros_like(w)
    r = w.copy()                      # line 2: r0 = w - Q x0
    z = Minv(r)                       # line 3
    h = z.copy()                      # line 4
    wn = float(np.linalg.norm(w))
    rz = float(z @ r)
    hist = [1.0]
    if wn == 0.0:
        return (x, 0, 0.0, 0, hist) if record else (x, 0, 0.0, 0)
    it = 0
    status = 4
    relres = 1.0
    while it < maxit:
        l = Qmul(h)                   # line 6
        hl = float(h @ l)
        if not hl > 0.0:
            status = 8
            break
        alpha = rz / hl               # line 7
        x = x + alpha * h             # line 8
        r = r - alpha * l             # line 9
        it += 1
        relres = float(np.linalg.norm(r)) / wn
        hist.append(relres)
        if relres <= tol:
            status = 0
            break
        z = Minv(r)                   # line 10
        rz_new = float(z @ r)
        nu = rz_new / rz              # line 11
        h = z + nu * h                # line 12
        rz = rz_new
    return (x, it, relres, status, hist) if record else (x, it, relres, status)
