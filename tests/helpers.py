"""Shared test helpers: dense LP matrices from mask words (test-side construction)."""
from __future__ import annotations

import numpy as np


def dense_step_matrix(code, mask_row, flip_row=None):
    """Dense A (p x (n+p)) of an ipm_step_pcg system, rows = present checks ascending, slack of
    compact row r at column n + r.  Returns (A, rows)."""
    n = code.n
    rows = [j for j in range(code.m) if (int(mask_row[j]) >> 15) & 1]
    p = len(rows)
    A = np.zeros((p, n + p))
    for r, j in enumerate(rows):
        Nj = code.N(j)
        w = int(mask_row[j])
        for t, i in enumerate(Nj):
            a = 1.0 if (w >> t) & 1 else -1.0
            s = -1.0 if (flip_row is not None and flip_row[i]) else 1.0
            A[r, i] = a * s
        A[r, n + r] = 1.0
    return A, rows


def step_weights(code, d_row, rows):
    """d^2 restricted to the LP columns (standard, then slacks of present rows)."""
    n = code.n
    d2 = np.asarray(d_row, dtype=np.float64) ** 2
    return np.concatenate([d2[:n], d2[[n + j for j in rows]]])


def oracle_col_to_gpu(code, rows, c):
    return c if c < code.n else code.n + rows[c - code.n]
