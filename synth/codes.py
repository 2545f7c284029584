"""Parity-check matrices (Tanner graphs) for the benchmark and test workloads.

The paper's codes are random (3,6)-regular codes built by the authors
(§III-D l.363-365, §VI-B l.815-818); they are not available, so a
seeded configuration model stands in for them:
edge e = 0..E-1 joins variable e // d_v to check pi[e] // d_c with
pi = default_rng(code_seed).permutation(E); while a (variable, check) pair
repeats, the duplicate's check socket is swapped with socket
rng.integers(E) drawn from the same stream.  Double edges are resampled;
4-cycles are kept (reading C-21 in DESIGN.md).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np


@dataclass(frozen=True)
class Code:
    """An m x n binary parity-check matrix H stored as check-major CSR.

    row_ptr[j] .. row_ptr[j+1] index col_idx, the sorted neighbourhood N(j)
    of check j (§II-A l.72-74).  All indices are 0-based.
    """
    n: int
    m: int
    row_ptr: np.ndarray   # int32 [m+1]
    col_idx: np.ndarray   # int32 [E], strictly increasing within a row
    name: str = ""

    @property
    def E(self) -> int:
        return int(self.row_ptr[-1])

    def N(self, j: int) -> np.ndarray:
        """Sorted neighbourhood of check j."""
        return self.col_idx[self.row_ptr[j]:self.row_ptr[j + 1]]

    def checks(self) -> list[np.ndarray]:
        return [self.N(j) for j in range(self.m)]

    def var_checks(self) -> list[list[int]]:
        """Neighbourhood of every variable node (ascending check index)."""
        out: list[list[int]] = [[] for _ in range(self.n)]
        for j in range(self.m):
            for i in self.N(j):
                out[int(i)].append(j)
        return out

    def dense(self) -> np.ndarray:
        H = np.zeros((self.m, self.n), dtype=np.uint8)
        for j in range(self.m):
            H[j, self.N(j)] = 1
        return H

    @property
    def max_check_degree(self) -> int:
        return int(np.max(np.diff(self.row_ptr))) if self.m else 0


def code_from_rows(rows, n: int, name: str = "") -> Code:
    """Build a Code from a list of per-check variable lists (any order)."""
    rows = [sorted(int(i) for i in r) for r in rows]
    for r in rows:
        if len(set(r)) != len(r):
            raise ValueError("duplicate variable in a check")
        if r and (r[0] < 0 or r[-1] >= n):
            raise ValueError("variable index out of range")
    row_ptr = np.zeros(len(rows) + 1, dtype=np.int32)
    row_ptr[1:] = np.cumsum([len(r) for r in rows])
    col_idx = np.array([i for r in rows for i in r], dtype=np.int32)
    return Code(n=n, m=len(rows), row_ptr=row_ptr, col_idx=col_idx, name=name)


def code_from_dense(H: np.ndarray, name: str = "") -> Code:
    H = np.asarray(H)
    return code_from_rows([np.nonzero(H[j])[0] for j in range(H.shape[0])],
                          H.shape[1], name)


def regular_code(n: int, dv: int, dc: int, seed: int, name: str = "", girth6: bool = False) -> Code:
    """Seeded (dv, dc)-regular configuration-model code, double edges resampled; girth6 also
    removes every 4-cycle (the paper's codes; reading C-21 keeps them for the configs)."""
    if (n * dv) % dc:
        raise ValueError("n*dv must be divisible by dc")
    E = n * dv
    m = E // dc
    rng = np.random.default_rng(seed)
    pi = rng.permutation(E)
    var_of_edge = np.arange(E) // dv
    while True:
        chk = pi // dc
        key = var_of_edge.astype(np.int64) * m + chk
        # first occurrence of each (var, check) pair keeps its socket; later ones are duplicates
        _, first = np.unique(key, return_index=True)
        dup_mask = np.ones(E, dtype=bool)
        dup_mask[first] = False
        dups = np.nonzero(dup_mask)[0]
        if dups.size == 0:
            break
        e = int(dups[0])
        e2 = int(rng.integers(E))
        pi[e], pi[e2] = pi[e2], pi[e]
    if girth6:
        # optional 4-cycle removal (C-21; the paper's codes): while two variables
        # share two checks, swap the check socket of one edge of that cycle with a random edge
        # (same stream), keeping the graph free of double edges
        for _ in range(200 * E):
            chk = pi // dc
            cyc = _find_4cycle_edge(var_of_edge, chk, n, m, dv)
            if cyc < 0:
                break
            e2 = int(rng.integers(E))
            pi[cyc], pi[e2] = pi[e2], pi[cyc]
            chk = pi // dc
            key = var_of_edge.astype(np.int64) * m + chk
            if np.unique(key).size != E:       # created a double edge: undo
                pi[cyc], pi[e2] = pi[e2], pi[cyc]
        else:
            raise RuntimeError("4-cycle removal did not converge")
    chk = pi // dc
    rows: list[list[int]] = [[] for _ in range(m)]
    for e in range(E):
        rows[int(chk[e])].append(int(var_of_edge[e]))
    return code_from_rows(rows, n, name or f"rnd({dv},{dc}) n={n} seed={seed}" + (" girth6" if girth6 else ""))


def _find_4cycle_edge(var_of_edge, chk, n, m, dv) -> int:
    """An edge on some 4-cycle (two variables sharing two checks), or -1 if the graph has none."""
    vc = chk.reshape(n, dv)
    seen = {}
    for i in range(n):
        cs = sorted(int(c) for c in vc[i])
        for a in range(dv):
            for b in range(a + 1, dv):
                key = (cs[a], cs[b])
                if key in seen and seen[key] != i:
                    # edge (i, cs[a]) lies on the cycle i - cs[a] - seen[key] - cs[b] - i
                    return int(i * dv + list(vc[i]).index(cs[a]))
                seen[key] = i
    return -1


# BASELINE.json configs (SURVEY.md §8(d) d.1 code seeds)
CONFIG_CODES = {
    1: dict(n=120, dv=3, dc=6, seed=1001),
    2: dict(n=1000, dv=3, dc=6, seed=1002),
    3: dict(n=4000, dv=3, dc=12, seed=1003),
    4: dict(n=32000, dv=3, dc=6, seed=1004),
    5: dict(n=2000, dv=3, dc=6, seed=1005),
}


def config_code(cfg: int) -> Code:
    p = CONFIG_CODES[cfg]
    return regular_code(p["n"], p["dv"], p["dc"], p["seed"], name=f"C{cfg}")
