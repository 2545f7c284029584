"""Isolated step-direction systems (BASELINE.json config 5).

65,536 systems A D^2 A^T dy = r over a (3,6)-regular n=2000 code with one cut
row per check:
  rng = default_rng([2005, 0, s]) per system s, draws in this order:
  idx = rng.integers(0, 32, size=m)   -> V_j = idx_j-th odd-popcount 6-bit mask
                                         (increasing numeric order), bit t <-> N(j)[t]
  d   = 10 ** rng.uniform(-6, 6, size=q), q = n + m (standard then slack)
  r   = rng.standard_normal(m)
Mask word layout (shared with include/alp.h): bit t set <=> N(j)[t] in V
(coefficient +1, else -1); bit 15 set <=> row present.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from .codes import Code, config_code

PRESENT = np.uint16(1 << 15)


def odd_masks(d: int) -> np.ndarray:
    """All d-bit masks with odd popcount, in increasing numeric order."""
    return np.array([v for v in range(1 << d) if bin(v).count("1") % 2 == 1], dtype=np.uint16)


@dataclass
class StepSystems:
    code: Code
    sys_ids: np.ndarray
    masks: np.ndarray   # [S, m] uint16
    d: np.ndarray       # [S, n+m] float64, diagonal of D (Q = A diag(d)^2 A^T)
    r: np.ndarray       # [S, m] float64

    @property
    def S(self) -> int:
        return int(self.masks.shape[0])


def c5_systems(systems, code: Code | None = None, seed: int = 2005,
               lo: float = -6.0, hi: float = 6.0, present_frac: float = 1.0) -> StepSystems:
    """Config-5 systems for the given system indices.

    present_frac < 1 drops rows (test-only variant; drawn after r from the same stream).
    """
    code = code or config_code(5)
    systems = np.asarray(list(systems) if not isinstance(systems, np.ndarray) else systems,
                         dtype=np.int64)
    m, n = code.m, code.n
    q = n + m
    deg = np.diff(code.row_ptr)
    tables = {int(dj): odd_masks(int(dj)) for dj in np.unique(deg)}
    S = systems.size
    masks = np.zeros((S, m), dtype=np.uint16)
    d = np.zeros((S, q))
    r = np.zeros((S, m))
    for t, s in enumerate(systems):
        rng = np.random.default_rng([seed, 0, int(s)])
        idx = rng.integers(0, 32, size=m)
        for dj, tab in tables.items():
            sel = deg == dj
            masks[t, sel] = tab[idx[sel] % tab.size] | PRESENT
        d[t] = 10.0 ** rng.uniform(lo, hi, size=q)
        r[t] = rng.standard_normal(m)
        if present_frac < 1.0:
            keep = rng.uniform(size=m) < present_frac
            masks[t, ~keep] = 0
            r[t, ~keep] = 0.0
    return StepSystems(code, systems, masks, d, r)
