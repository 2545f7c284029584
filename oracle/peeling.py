"""ORACLE (test infrastructure only — see oracle/__init__.py).

Erasure peeling on a Tanner graph and stopping sets (§II-A; used by
Thm 4 P:320-358 and Lemma 2).  A set S of variable nodes is a stopping set
if no check has exactly one neighbour in S; peeling of the erased set S succeeds iff S
contains no non-empty stopping set.
"""
from __future__ import annotations

import numpy as np


def peel(check_rows, erased) -> set:
    """Peel the erased variable set; returns the residual set (empty = success)."""
    E = set(int(i) for i in erased)
    changed = True
    while changed and E:
        changed = False
        for row in check_rows:
            inter = [int(i) for i in row if int(i) in E]
            if len(inter) == 1:
                E.discard(inter[0])
                changed = True
    return E


def is_stopping_set(check_rows, S) -> bool:
    S = set(int(i) for i in S)
    if not S:
        return False
    return all(sum(1 for i in row if int(i) in S) != 1 for row in check_rows)


def contains_stopping_set(check_rows, S) -> bool:
    """S contains a non-empty stopping set iff peeling S leaves a non-empty residual
    (the residual of peeling is the largest stopping set inside S)."""
    return len(peel(check_rows, S)) > 0


def rows_of_matrix(A) -> list:
    A = np.asarray(A)
    return [list(np.nonzero(A[j])[0]) for j in range(A.shape[0])]
