"""Pins for the oracle's Alg. 2 cut search and parity inequalities.

Pins: hand-worked examples (golden), brute force over all 2^{d-1} odd subsets
(presence, identity of the minimum-lhs set, Thm 1 uniqueness P:175-178), and the
integral special case (violated <=> parity check fails).
"""
import json
import os
from itertools import combinations

import numpy as np
import pytest

from oracle.lp import find_violated_cut, cut_lhs, hard_decision, mask_word, mask_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_examples():
    g = json.load(open(os.path.join(GOLD, "cut_examples.json")))
    for case in g["cases"]:
        V, lhs, viol = find_violated_cut(np.array(case["u"]))
        assert list(np.nonzero(V)[0]) == case["V"], case
        assert lhs == pytest.approx(case["lhs"], abs=1e-12)
        assert viol == case["violated"]


def _all_odd(d):
    for k in range(1, d + 1, 2):
        for V in combinations(range(d), k):
            m = np.zeros(d, dtype=bool)
            m[list(V)] = True
            yield m


@pytest.mark.parametrize("d", [1, 2, 3, 4, 6, 8, 12])
def test_brute_force_min_and_theorem1(d):
    rng = np.random.default_rng(100 + d)
    for _ in range(300 if d < 10 else 60):
        u = rng.uniform(size=d)
        if rng.uniform() < 0.3:   # push some coordinates to 0/1 and near 1/2
            u[rng.integers(d)] = float(rng.integers(2))
        V, lhs, _ = find_violated_cut(u)
        assert V.sum() % 2 == 1
        lhss = [(cut_lhs(u, m), m) for m in _all_odd(d)]
        best = min(l for l, _ in lhss)
        assert lhs == pytest.approx(best, abs=1e-12)          # Alg. 2 minimises the lhs
        violated = [m for l, m in lhss if l < 1.0]
        assert len(violated) <= 1                             # Thm 1: at most one violated
        if violated:
            assert np.array_equal(violated[0], V)
            others = [l for l, m in lhss if not np.array_equal(m, V)]
            assert all(l > 1.0 for l in others)               # ... and the rest strictly hold


def test_integral_points_equal_parity():
    rng = np.random.default_rng(7)
    for d in range(1, 10):
        for _ in range(50):
            u = rng.integers(0, 2, size=d).astype(float)
            _, lhs, viol = find_violated_cut(u)
            assert viol == (int(u.sum()) % 2 == 1)
            assert lhs == (0.0 if viol else pytest.approx(lhs))


def test_hard_decision_and_tie_convention():
    assert list(hard_decision(np.array([-2.1, 0.7, 0.3, -0.4]))) == [1, 0, 0, 1]
    assert list(hard_decision(np.array([0.0, -1.0]))) == [0, 1]      # gamma = 0 -> 0 (C-16)
    # u_i = 1/2 is not in S (strict, C-2); equal distances -> lowest position
    V, _, _ = find_violated_cut(np.array([0.5, 0.5, 0.2]))
    assert list(np.nonzero(V)[0]) == [0]


def test_mask_word_roundtrip():
    for bits in ([True], [False, True, True], [True] * 12):
        w = mask_word(np.array(bits))
        assert (w >> 15) & 1
        assert list(mask_bits(w, len(bits))) == bits
