"""Pins for oracle/lp_library.py (MALP with the LP step solved by a library LP solver; the
oracle for config 4, where the dense-IPM oracle runs an hour per frame into its cap).

Pins, none of which re-calls the routine under test:
 * the Bland-rule simplex on the FULL Feldman relaxation (oracle/full_lp.py, hand-written) and
   brute-force ML on tiny codes — the plain definition Alg. 3 must reach (Thm 2c);
 * the oracle's own IPM path (oracle.lp.malp_decode) frame by frame on config 1 and on
   config-2 frames at 2.0 dB (fractional outputs): hard decisions, certificate, objective,
   LP count and the final cut pool;
 * the LP-duality certificate (oracle/certify.py) on its own (u, y, pool): y really is the
   dual of G4 / C-25, and a perturbed answer is rejected;
 * library_lp_solve on a textbook LP with a known optimum and dual.
"""
import numpy as np
import pytest

from oracle.certify import dual_certificate
from oracle.full_lp import lp_decode_full, ml_decode
from oracle.lp import malp_decode
from oracle.lp_library import library_lp_solve, malp_decode_library
from synth import config_code, config_frames
from synth.codes import code_from_rows, regular_code


def test_library_lp_solve_textbook_lp():
    # min -3 x1 - 5 x2  s.t. x1 + s1 = 4, 2 x2 + s2 = 12, 3 x1 + 2 x2 + s3 = 18, x >= 0
    # (the classic 2-variable example): x* = (2, 6), objective -36, duals (0, -3/2, -1)
    A = np.array([[1.0, 0, 1, 0, 0], [0, 2.0, 0, 1, 0], [3.0, 2.0, 0, 0, 1]])
    b = np.array([4.0, 12.0, 18.0])
    c = np.array([-3.0, -5.0, 0, 0, 0])
    r = library_lp_solve(A, b, c)
    assert r["status"] == 0
    np.testing.assert_allclose(r["x"], [2, 6, 2, 0, 0], atol=1e-9)
    np.testing.assert_allclose(r["y"], [0, -1.5, -1.0], atol=1e-9)
    assert float(b @ r["y"]) == pytest.approx(-36.0)          # strong duality (G4: max b^T y)
    assert np.all(r["z"] >= -1e-9) and float(r["x"] @ r["z"]) == pytest.approx(0.0, abs=1e-9)


@pytest.mark.parametrize("seed", [50, 51, 77])
def test_library_malp_reaches_full_relaxation_and_ml(seed):
    code = regular_code(12, 3, 6, seed=seed) if seed != 77 else regular_code(16, 3, 12, seed=77)
    rng = np.random.default_rng(seed)
    for _ in range(6):
        gamma = rng.normal(1.2, 1.6, code.n)
        u_s, obj_s = lp_decode_full(code, gamma)     # independent Bland simplex, all 2^(d-1) rows
        for variant in ("A", "B"):
            r = malp_decode_library(code, gamma, variant)
            assert r["status"] == 0
            assert r["obj"] == pytest.approx(obj_s, abs=1e-8)
            np.testing.assert_allclose(r["u"], u_s, atol=1e-7)
            if r["cert"]:
                cw, cost, ties = ml_decode(code, gamma)
                if ties == 1:
                    np.testing.assert_array_equal(r["hard"], cw)


def test_h1_codeword_needs_no_lp():
    code = code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1")
    r = malp_decode_library(code, np.array([1.0, 2.0, 3.0, 4.0]))
    assert r["lp_solves"] == 0 and r["cert"] == 1 and r["obj"] == 0.0


def _same_as_ipm_path(code, llr, frames):
    n_frac = 0
    for f in frames:
        a = malp_decode(code, llr[f])
        b = malp_decode_library(code, llr[f])
        if a["status"] or b["status"]:
            continue        # the IPM path's own caps (2.0 dB) prove nothing about the library path
        sure = np.abs(a["u"] - 0.5) > 1e-3
        np.testing.assert_array_equal(a["hard"][sure], b["hard"][sure])
        assert a["cert"] == b["cert"]
        scale = max(1.0, abs(a["obj"]), float(np.max(np.abs(llr[f]))))
        assert abs(a["obj"] - b["obj"]) <= 1e-6 * scale
        np.testing.assert_allclose(a["u"], b["u"], atol=1e-5)
        assert a["lp_solves"] == b["lp_solves"]
        np.testing.assert_array_equal(a["masks"], b["masks"])
        n_frac += int(a["cert"] == 0)
        c = dual_certificate(code, llr[f], b["u"], b["y"], b["masks"])
        assert c["ok"], c.get("reasons")
    return n_frac


def test_library_path_equals_ipm_path_config1():
    code = config_code(1)
    fb = config_frames(1, frames=range(30))
    _same_as_ipm_path(code, fb.llr, range(30))


def test_library_path_equals_ipm_path_config2_fractional():
    code = config_code(2)
    fb = config_frames(2, frames=range(6), snr_idx=0, code=code)   # 2.0 dB: fractional outputs occur
    _same_as_ipm_path(code, fb.llr, range(6))


def test_certificate_rejects_perturbed_library_answer():
    code = config_code(1)
    fb = config_frames(1, frames=range(6))
    for f in range(6):
        b = malp_decode_library(code, fb.llr[f])
        if b["lp_solves"] == 0:
            continue
        y = b["y"].copy()
        j = int(np.argmax(np.abs(y)))
        y[j] *= 0.5                                   # no longer the optimal dual: gap opens
        assert not dual_certificate(code, fb.llr[f], b["u"], y, b["masks"])["ok"]
        u = b["u"].copy()
        i = int(np.argmax(fb.llr[f] * (1 - 2 * u)))   # flip a bit the LP did not want flipped
        u[i] = 1.0 - u[i]
        assert not dual_certificate(code, fb.llr[f], u, b["y"], b["masks"])["ok"]
        return
    pytest.skip("no frame needed an LP")


def test_e3_largest_lp_of_malp_smaller_than_alp():
    """The value the paper prints for E3: the largest LP (cut rows) of MALP-A / MALP-B is
    smaller on average than plain ALP's by 17 % (integral outputs) / 30 % (fractional outputs).
    Pins Alg. 1 (no removal) against Alg. 3 (removal) in the oracle on 64 frames of an n = 480
    (3,6) code at 2 dB (the paper's E1 length and SNR); 1000 trials per length are in
    profiles/r2_e3_largest_lp.json (-14 % / -28 % at n = 480, -17 % / -31 % at n = 1920)."""
    from synth import awgn_frames
    code = regular_code(480, 3, 6, seed=3480, girth6=True)
    fb = awgn_frames(code, 2.0, 4480, 0, range(64), random_codeword=False)
    big = {v: {0: [], 1: []} for v in ("ALP", "A", "B")}
    for f in range(fb.F):
        outs = {v: malp_decode(code, fb.llr[f], v, lp_solver=library_lp_solve) for v in ("ALP", "A", "B")}
        assert all(o["status"] == 0 for o in outs.values())
        # Thm 2c: with or without removal the final LP optimum is the same
        assert abs(outs["A"]["obj"] - outs["ALP"]["obj"]) <= 1e-7 and abs(outs["B"]["obj"] - outs["ALP"]["obj"]) <= 1e-7
        assert outs["A"]["max_p"] <= outs["ALP"]["max_p"] and outs["A"]["max_p"] <= code.m   # Cor. 3
        for v, o in outs.items():
            big[v][outs["ALP"]["cert"]].append(o["max_p"])
    for v in ("A", "B"):
        r_int = np.mean(big[v][1]) / np.mean(big["ALP"][1]) - 1.0
        r_frac = np.mean(big[v][0]) / np.mean(big["ALP"][0]) - 1.0
        assert -0.25 <= r_int <= -0.08, (v, r_int)
        assert -0.42 <= r_frac <= -0.18, (v, r_frac)
