"""Pins for the oracle's adaptive LP decoders (Alg. 1, Alg. 3, MALP-B P:242).

Pins: the worked H7 trace and the (7,4,3) pseudocodeword of P:311-313 (golden);
the plain definition — the full Feldman relaxation solved by an independent
hand-written Bland simplex and by scipy HiGHS (Thm 2c); brute-force ML for
integral outputs (ML certificate P:143); invariants Thm 2a/b/c, Thm 3, Cor. 4 (G3),
Cor. 5, Thm 4; the LP-duality certificate on config-1 frames.
"""
import json
import os

import numpy as np
import pytest
from scipy.optimize import linprog

from oracle.lp import malp_decode, hard_decision, find_violated_cut
from oracle.full_lp import lp_decode_full, feldman_rows, ml_decode, codewords
from oracle.certify import dual_certificate
from oracle.peeling import contains_stopping_set
from synth.codes import code_from_dense, code_from_rows, regular_code
from synth import config_code, config_frames

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _h7():
    g = json.load(open(os.path.join(GOLD, "h7_trace.json")))
    H = np.array([[int(c) for c in r] for r in g["H"]])
    return code_from_dense(H, "H7"), g


@pytest.mark.parametrize("variant", ["A", "B"])
def test_h7_golden_trace(variant):
    code, g = _h7()
    gamma = np.array(g["gamma"])
    np.testing.assert_array_equal(hard_decision(gamma), g["lp0_u"])
    assert float(gamma @ hard_decision(gamma)) == pytest.approx(g["lp0_obj"])
    r = malp_decode(code, gamma, variant, record=True)
    assert len(r["trace"]) == len(g["trace"])
    for t, exp in zip(r["trace"], g["trace"]):
        pool = {str(j): [int(code.N(j)[k]) for k in np.nonzero(V)[0]] for j, V in t["pool"].items()}
        assert pool == exp["pool"]
        np.testing.assert_allclose(t["u"], exp["u"], atol=1e-7)
        assert t["obj"] == pytest.approx(exp["obj"], abs=1e-7)
    assert r["cert"] == 0 and g["final_fractional"]
    # [1,1/2,0,1/2,0,0,1/2] has exactly m = 3 fractional entries (Cor. 5 tight)
    frac = np.sum(np.abs(r["u"] - np.round(r["u"])) > 1e-6)
    assert frac == 3 == code.m
    # the same point is the optimum of the full relaxation (independent simplex)
    u_full, obj_full = lp_decode_full(code, gamma)
    np.testing.assert_allclose(u_full, r["u"], atol=1e-7)
    # ML cost and the tie
    cw, cost, ties = ml_decode(code, gamma)
    assert cost == pytest.approx(g["ml_cost"]) and ties == 2


def test_h7_pseudocodeword_is_vertex_of_fundamental_polytope():
    code, _ = _h7()
    G, h = feldman_rows(code)
    u = np.array([1, 0.5, 0, 0.5, 0, 0, 0.5])
    assert np.all(G @ u <= h + 1e-12) and np.all(u >= 0)
    active = np.vstack([G[np.abs(G @ u - h) < 1e-12], np.eye(7)[u == 0]])
    assert np.linalg.matrix_rank(active) == 7


def _tiny_codes():
    codes = [code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1"), _h7()[0]]
    for s in range(3):
        codes.append(regular_code(12, 3, 6, seed=50 + s))
    codes.append(regular_code(16, 3, 12, seed=77))
    return codes


@pytest.mark.parametrize("ci", range(6))
def test_decoders_match_full_relaxation_and_ml(ci):
    code = _tiny_codes()[ci]
    rng = np.random.default_rng(ci)
    G, h = feldman_rows(code)
    for trial in range(8 if code.n <= 12 else 4):
        # continuous LLRs (uniqueness, C-12): all-zero codeword over a noisy channel
        gamma = rng.normal(1.2, 1.6, code.n)
        full = linprog(gamma, A_ub=G, b_ub=h, bounds=[(0, 1)] * code.n, method="highs")
        for variant in ("A", "B", "ALP"):
            r = malp_decode(code, gamma, variant, record=True)
            assert r["status"] == 0
            assert r["obj"] == pytest.approx(full.fun, abs=1e-6)
            np.testing.assert_allclose(r["u"], full.x, atol=2e-5)
            # Thm 2a/b/c
            objs = [float(gamma @ hard_decision(gamma))] + r["objs"]
            assert all(b > a for a, b in zip(objs, objs[1:]))
            assert r["lp_solves"] <= code.n
            for t in r["trace"]:
                assert np.all(t["u"] >= -1e-7) and np.all(t["u"] <= 1 + 1e-7)
            if r["cert"]:
                cw, cost, ties = ml_decode(code, gamma)
                if ties == 1:
                    np.testing.assert_array_equal(r["hard"], cw)
        if trial == 0 and code.n <= 12:
            u_s, obj_s = lp_decode_full(code, gamma)
            assert obj_s == pytest.approx(full.fun, abs=1e-9)


def test_theorem3_and_corollaries_on_config1():
    code = config_code(1)
    fb = config_frames(1, frames=range(12))
    hd_all = []
    for f in range(fb.F):
        gamma = fb.llr[f]
        r = malp_decode(code, gamma, "A", record=True)
        assert r["status"] == 0
        # Thm 3 / Cor. 3: one cut per check, p <= m
        for t in r["trace"]:
            assert len(t["pool"]) <= code.m
        assert r["max_p"] <= code.m
        u = r["u"]
        hd = hard_decision(gamma)
        # Cor. 4 (G3): differs from the hard decision in at most m coordinates
        assert np.sum(np.abs(np.round(u) - hd) > 0.5) <= code.m
        # Cor. 5: at most m fractional entries
        assert np.sum(np.minimum(u, 1 - u) > 1e-5) <= code.m
        # Thm 4: unique integral output -> flip set holds no stopping set
        if r["cert"]:
            E = np.nonzero(np.round(u) != hd)[0]
            assert not contains_stopping_set(code.checks(), E)
        # P6 certificate holds
        c = dual_certificate(code, gamma, u, r["y"], r["masks"])
        assert c["ok"], c["reasons"]
        hd_all.append(r["cert"])
    assert sum(hd_all) >= 6


def test_certificate_rejects_a_wrong_answer():
    code = config_code(1)
    fb = config_frames(1, frames=[0])
    r = malp_decode(code, fb.llr[0], "A")
    bad = r["u"].copy()
    i = int(np.argmax(np.abs(fb.llr[0])))
    bad[i] = 1 - bad[i]
    assert not dual_certificate(code, fb.llr[0], bad, r["y"], r["masks"])["ok"]


def test_hard_decision_codeword_needs_no_lp():
    code = code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1")
    r = malp_decode(code, np.array([1.0, 1.0, 1.0, 1.0]))
    assert r["lp_solves"] == 0 and r["cert"] == 1 and r["obj"] == 4.0 - 4.0 + 0.0 or r["obj"] == 0.0
    r = malp_decode(code, np.array([-3.0, 1.0, 2.0, -1.0]))
    np.testing.assert_allclose(r["u"], [1, 1, 0, 1], atol=1e-7)
    cw, cost, _ = ml_decode(code, np.array([-3.0, 1.0, 2.0, -1.0]))
    assert list(cw) == [1, 1, 0, 1] and cost == -3.0


def test_codeword_enumeration_h1():
    code = code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1")
    words = sorted("".join(map(str, w)) for w in codewords(code))
    assert words == ["0000", "0110", "1011", "1101"]


def test_malp_cycle_detection_stops_at_a_repeated_pool():
    """Reading C-12: MALP-A is a deterministic function of its cut pool, so a pool equal to
    that of an LP already solved cycles forever.  On this C2 frame (3.0 dB) the oracle used
    to run to the 200-LP cap; it must now stop at the first repeat with ALP_MAXITER, and the
    pool it stopped on must equal the pool of one of the LPs it solved."""
    from oracle.lp import mask_word, ST_ALP_MAXITER
    from synth import config_code, config_frames
    code = config_code(2)
    fb = config_frames(2, 2, frames=[1737])
    o = malp_decode(code, fb.llr[0], record=True)
    assert o["status"] & ST_ALP_MAXITER
    assert o["lp_solves"] < 20
    final = {j: mask_word(v) for j, v in o["pool"].items()}
    assert any(final == {j: mask_word(v) for j, v in tr["pool"].items()} for tr in o["trace"])
    # the solved LPs themselves were all distinct
    keys = [frozenset((j, mask_word(v)) for j, v in tr["pool"].items()) for tr in o["trace"]]
    assert len(set(keys)) == len(keys)
