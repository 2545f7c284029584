"""SURVEY f-4: BSC frames with LLR jitter — input generation pins (CPU) and the uniqueness
remedy on the oracle (MALP-A on un-jittered BSC LLRs can cycle, C-12; jittered ones decode)."""
import json
import os

import numpy as np

from synth import bsc_llr, bsc_frames, config_code

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bsc_examples.json")


def test_bsc_llr_worked_examples():
    g = json.load(open(GOLD))
    for c in g["cases"]:
        assert bsc_llr(np.array([c["bit"]]), c["p"], c["jitter"])[0] == c["gamma"]
    jb = g["jitter_bound"]
    code = config_code(1)
    fb = bsc_frames(code, jb["p"], jb["jitter"], 3001, range(4), random_codeword=False)
    assert np.all(np.abs(np.abs(fb.llr) - jb["center"]) <= jb["jitter"])
    assert np.unique(np.abs(fb.llr)).size > 100          # jitter makes the magnitudes distinct


def test_bsc_frames_are_codewords_through_the_channel():
    code = config_code(1)
    p = 0.05
    fb = bsc_frames(code, p, 1e-4, 3001, range(64))
    H = np.zeros((code.m, code.n), dtype=np.int64)
    for j in range(code.m):
        H[j, code.N(j)] = 1
    assert np.all((fb.codewords @ H.T) % 2 == 0)
    flips = ((fb.llr < 0).astype(np.uint8) ^ fb.codewords)
    rate = flips.mean()
    assert abs(rate - p) < 0.02                           # crossover probability
    again = bsc_frames(code, p, 1e-4, 3001, [5])
    assert np.array_equal(again.llr[0], fb.llr[5])        # per-frame keyed (any shard regenerates)


def test_jitter_restores_unique_lp_optima_on_the_oracle():
    """Without jitter every |gamma_i| is equal, LP optima are highly non-unique and the MALP
    pool can repeat (C-12 cycle status); with jitter the same frames decode without it."""
    from oracle.lp import malp_decode
    code = config_code(1)
    fb0 = bsc_frames(code, 0.06, 0.0, 3002, range(24), random_codeword=False)
    fbj = bsc_frames(code, 0.06, 1e-3, 3002, range(24), random_codeword=False)
    st0 = [malp_decode(code, fb0.llr[f])["status"] for f in range(24)]
    stj = [malp_decode(code, fbj.llr[f])["status"] for f in range(24)]
    assert sum(s & 1 for s in stj) <= sum(s & 1 for s in st0)
    assert all((s & (1 | 2 | 16)) == 0 for s in stj)


def test_girth6_codes_have_no_4cycles():
    """C-21 option (the paper's codes): 4-cycle removal keeps the (3,6) degrees and
    leaves no two variables sharing two checks."""
    from synth.codes import regular_code
    for n in (120, 480):
        c = regular_code(n, 3, 6, seed=11, girth6=True)
        H = np.zeros((c.m, c.n), dtype=np.int64)
        for j in range(c.m):
            H[j, c.N(j)] = 1
        assert np.all(H.sum(axis=0) == 3) and np.all(H.sum(axis=1) == 6)
        O = H.T @ H
        np.fill_diagonal(O, 0)
        assert O.max() <= 1
