"""GPU parity of ipm_step_pcg (eq.`Delta y` P:479 by Alg. 4 + Alg. 7) against the oracle.

Gates (reading C-27), per system:
  * pivot sequence bit-exact vs the oracle's heap Alg. 7 on identical weights (incl. exact
    float ties and the all-equal weights of the first IPM step);
  * status 0 or the informational PCG_FLOOR; the reported TRUE relative residual <= 1e-8, or,
    flagged PCG_FLOOR, within 1e3x the fp64 evaluation floor 16 eps || |A| D^2 |A|^T |dy| || / ||w||
    (re-checked here from the dense Q; the histogram of residual / floor goes to the report);
  * ||dy - dy*|| / ||dy*|| <= 1e-8 (SURVEY C-27) against the oracle's exact solve dy*
    (long-double Cholesky refined with exact rational residuals; pinned against exact rational
    solutions up to kappa ~1e20+ in tests/test_oracle_ipm.py).
Config 5: the first 1024 systems (c.5), the oracle run in a process pool.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle.lp import step_solve_exact, normal_matrix, find_violated_cut, mask_word
from oracle.precond import mts_columnwise
from synth import config_code, config_frames, c5_systems
from synth.codes import code_from_rows
from tests.helpers import dense_step_matrix, step_weights, oracle_col_to_gpu
from tests.oracle_pool import oracle_step_exact

pytestmark = pytest.mark.gpu
FLOOR = 32                    # ALP_FRAME_PCG_FLOOR (informational)
EPS = np.finfo(np.float64).eps
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _alp():
    import paper_0902_0657_b200 as alp
    return alp


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda")


def _run(code, masks, d, r, flip=None, **pkw):
    alp = _alp()
    c = alp.Code.from_synth(code)
    params = alp.default_params(**pkw)
    res = alp.ipm_step_pcg(c, _t(masks.view(np.int16)), _t(d), _t(r),
                           None if flip is None else _t(flip.astype(np.uint8)), params=params,
                           want_pivots=True)
    torch.cuda.synchronize()
    assert alp.last_launch_count() == 1
    return dict(dy=res.dy.cpu().numpy(), iters=res.iters.cpu().numpy(), relres=res.relres.cpu().numpy(),
                status=res.status.cpu().numpy(), prow=res.pivot_rows.cpu().numpy(),
                pcol=res.pivot_cols.cpu().numpy())


def _check_pivots(code, rows, out, s, col, row):
    exp_rows = [rows[rw] for rw in row]
    exp_cols = [oracle_col_to_gpu(code, rows, c) for c in col]
    p = len(rows)
    assert list(out["prow"][s][:p]) == exp_rows, f"system {s}: pivot rows differ"
    assert list(out["pcol"][s][:p]) == exp_cols, f"system {s}: pivot cols differ"
    assert np.all(out["prow"][s][p:] == -1)


def _check_system(code, mk, dd, rr, fl, out, s, tol_dy=1e-8, check_pivots=True, ref=None, piv=None):
    A, rows = dense_step_matrix(code, mk, fl)
    w2 = step_weights(code, dd, rows)
    if check_pivots:
        col, row = piv if piv is not None else mts_columnwise(A, w2)
        _check_pivots(code, rows, out, s, col, row)
    Q = normal_matrix(A, w2)
    w = rr[rows]
    if ref is None:
        ref = step_solve_exact(A, w2, w)
    got = out["dy"][s][rows]
    st = int(out["status"][s])
    assert (st & ~FLOOR) == 0, f"system {s} status {st}"
    wn = np.linalg.norm(w)
    tres = np.linalg.norm(w - Q @ got) / wn
    floor = 16 * EPS * np.linalg.norm(np.abs(A) @ (w2 * (np.abs(A).T @ np.abs(got)))) / wn
    if not st & FLOOR:
        assert out["relres"][s] <= 1e-8
    else:
        assert out["relres"][s] <= 1e3 * floor
    assert tres <= 1.5 * max(1e-8, 1e3 * floor if st & FLOOR else floor), f"system {s}: true residual {tres:.3e}"
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= tol_dy, f"system {s}: rel err {err:.3e}"
    absent = [j for j in range(code.m) if j not in set(rows)]
    assert np.all(out["dy"][s][absent] == 0.0)
    return err, (out["relres"][s] / floor if floor > 0 else 0.0)


def test_golden_step_system():
    g = json.load(open(os.path.join(GOLD, "precond_examples.json")))["step_system"]
    code = code_from_rows([[0, 1], [1, 2]], 3)
    masks = np.array([[0x8003, 0x8003]], dtype=np.uint16)       # all coefficients +1
    d = np.ones((1, 5))
    r = np.array([g["r"]], dtype=np.float64)
    out = _run(code, masks, d, r)
    np.testing.assert_allclose(out["dy"][0], g["dy"], rtol=1e-14)
    assert list(out["prow"][0]) == g["pivots_row"]
    assert list(out["pcol"][0]) == g["pivots_col"]


def test_c5_first_1024_systems_vs_oracle():
    """Config 5 (kappa(Q) up to ~1e18), the c.5 sample: 1024 systems, each against the exact
    solve and the heap Alg. 7."""
    code = config_code(5)
    S = 1024
    sy = c5_systems(range(S), code)
    out = _run(code, sy.masks, sy.d, sy.r)
    orc = oracle_step_exact(range(S))
    errs, ratios = [], []
    for s in range(S):
        e, q = _check_system(code, sy.masks[s], sy.d[s], sy.r[s], None, out, s, tol_dy=1e-8,
                             ref=orc[s][0], piv=(orc[s][1], orc[s][2]))
        errs.append(e)
        ratios.append(q)
    st = out["status"]
    rep = dict(systems=S, status_counts={int(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))},
               max_rel_err=float(max(errs)), median_rel_err=float(np.median(errs)),
               relres_over_floor_hist=np.histogram(np.log10(np.maximum(ratios, 1e-3)), bins=[-3, -2, -1, 0, 1, 2, 3])[0].tolist(),
               iters_mean=float(out["iters"].mean()), iters_max=int(out["iters"].max()))
    os.makedirs(os.path.join(ROOT, "gpurun_out", "parity"), exist_ok=True)
    json.dump(rep, open(os.path.join(ROOT, "gpurun_out", "parity", "C5_1024.json"), "w"), indent=1)
    print("C5", rep)


@pytest.mark.parametrize("S", [1, 33, 130])
def test_partial_rows_flips_and_ragged_batches(S):
    code = config_code(1)
    rng = np.random.default_rng(S)
    sy = c5_systems(range(S), code, lo=-3, hi=3, present_frac=0.6)
    flip = rng.integers(0, 2, size=(S, code.n)).astype(np.uint8)
    out = _run(code, sy.masks, sy.d, sy.r, flip)
    for s in range(S):
        if (sy.masks[s] >> 15).sum() == 0:
            continue
        _check_system(code, sy.masks[s], sy.d[s], sy.r[s], flip[s], out, s, tol_dy=1e-8)


def test_float_ties_use_exact_weights():
    """Alg. 7 ranks by the exact fp64 weight (C-10): weights that are equal in fp32 but differ
    in fp64 must still be ordered by their fp64 values (the sort's tie fix-up path)."""
    code = config_code(1)
    S = 8
    sy = c5_systems(range(S), code, lo=-1, hi=1)
    rng = np.random.default_rng(7)
    q = code.n + code.m
    d = np.empty((S, q))
    for s in range(S):
        base = 10.0 ** rng.integers(-2, 3, size=q).astype(np.float64)   # few distinct fp32 values
        jitter = 1.0 + rng.integers(0, 4, size=q) * 2.0 ** -40           # invisible in fp32
        d[s] = np.sqrt(base * jitter)
    out = _run(code, sy.masks, d, sy.r)
    for s in range(S):
        _check_system(code, sy.masks[s], d[s], sy.r[s], None, out, s, tol_dy=1e-8)


def test_first_ipm_step_all_equal_weights_on_decode_pools():
    """The first Newton step of every LP has x = z = s0, so d^2 = 1 on every column: Alg. 7 is
    decided by ties alone (lower column index).  Pools = the cuts Alg. 2 finds at the hard
    decision of C2 frames (the first MALP-A LP), flips from the LLR signs."""
    code = config_code(2)
    fb = config_frames(2, 0, frames=range(16))
    S = fb.F
    masks = np.zeros((S, code.m), dtype=np.uint16)
    flips = (fb.llr < 0).astype(np.uint8)
    for s in range(S):
        u = flips[s].astype(np.float64)
        for j in range(code.m):
            inV, lhs, viol = find_violated_cut(u[code.N(j)], 1e-6)
            if viol:
                masks[s, j] = mask_word(inV)
    d = np.ones((S, code.n + code.m))
    r = np.random.default_rng(3).standard_normal((S, code.m))
    out = _run(code, masks, d, r, flips)
    for s in range(S):
        _check_system(code, masks[s], d[s], r[s], flips[s], out, s, tol_dy=1e-8)


def test_plain_cg_option():
    code = config_code(1)
    sy = c5_systems(range(8), code, lo=-0.2, hi=0.2)
    out = _run(code, sy.masks, sy.d, sy.r, precond=1)
    assert np.all(out["prow"] == -1)
    for s in range(8):
        # kappa(Q) ~ 5 here: the refined plain-CG solve reaches 1e-8 forward error
        _check_system(code, sy.masks[s], sy.d[s], sy.r[s], None, out, s, tol_dy=1e-8, check_pivots=False)


def test_empty_batch_and_all_absent_rows():
    alp = _alp()
    code = config_code(1)
    c = alp.Code.from_synth(code)
    z = torch.zeros((0, code.m), dtype=torch.int16, device="cuda")
    res = alp.ipm_step_pcg(c, z, torch.zeros((0, code.n + code.m), dtype=torch.float64, device="cuda"),
                           torch.zeros((0, code.m), dtype=torch.float64, device="cuda"))
    assert res.dy.shape == (0, code.m)
    masks = np.zeros((2, code.m), dtype=np.uint16)
    out = _run(code, masks, np.ones((2, code.n + code.m)), np.ones((2, code.m)))
    assert np.all(out["dy"] == 0) and np.all(out["iters"] == 0) and np.all(out["status"] == 0)


@pytest.mark.slow
def test_c5_full_size_properties_and_sampled_parity():
    """All 65,536 config-5 systems in the bench launch configuration: every system ends with
    status 0 / PCG_FLOOR (property at any size); 64 systems spread over the batch match the
    oracle (pivots + exact solve)."""
    code = config_code(5)
    S = 65536
    sy = c5_systems(range(S), code)
    out = _run(code, sy.masks, sy.d, sy.r)
    st = out["status"]
    assert np.all((st & ~FLOOR) == 0), np.unique(st, return_counts=True)
    assert np.all(out["relres"][(st & FLOOR) == 0] <= 1e-8)
    print("C5 full: status counts", dict(zip(*[a.tolist() for a in np.unique(st, return_counts=True)])),
          "iters mean %.1f max %d" % (out["iters"].mean(), out["iters"].max()))
    sample = np.random.default_rng(0).choice(S, 64, replace=False)
    orc = oracle_step_exact(sample)
    for k, s in enumerate(sample):
        _check_system(code, sy.masks[s], sy.d[s], sy.r[s], None, out, int(s), tol_dy=1e-8,
                      ref=orc[k][0], piv=(orc[k][1], orc[k][2]))


def _check_rowwise(code, masks, d, r, flip=None, S=None):
    """Alg. 8 on the GPU (precond = 2): the pivot sequence, read back in pick order, equals the
    oracle's mts_rowwise (lowest-index degree-1 row, min-weight erasure, diagonal expansion)."""
    from oracle.precond import mts_rowwise
    out = _run(code, masks, d, r, flip, precond=2)
    S = masks.shape[0] if S is None else S
    for s in range(S):
        A, rows = dense_step_matrix(code, masks[s], None if flip is None else flip[s])
        if not rows:
            continue
        w2 = step_weights(code, d[s], rows)
        col, row = mts_rowwise(A, w2)
        p = len(rows)
        exp_rows = [rows[rw] for rw in row][::-1]          # stored reversed (upper triangular)
        exp_cols = [oracle_col_to_gpu(code, rows, c) for c in col][::-1]
        assert list(out["prow"][s][:p]) == exp_rows, f"system {s}: row-wise pivot rows differ"
        assert list(out["pcol"][s][:p]) == exp_cols, f"system {s}: row-wise pivot cols differ"
        _check_system(code, masks[s], d[s], r[s], None if flip is None else flip[s], out, s, tol_dy=1e-8,
                      check_pivots=False)
    return out


def test_rowwise_mts_matches_oracle_alg8():
    """SURVEY f-1: Alg. 8 bit-exact vs the oracle on config-1 systems with partial
    rows and flips, on all-equal weights (tie rules), and on config-5 systems."""
    code = config_code(1)
    S = 24
    sy = c5_systems(range(S), code, lo=-3, hi=3, present_frac=0.7)
    flip = np.random.default_rng(11).integers(0, 2, size=(S, code.n)).astype(np.uint8)
    _check_rowwise(code, sy.masks, sy.d, sy.r, flip)
    _check_rowwise(code, sy.masks, np.ones_like(sy.d), sy.r, flip)
    code5 = config_code(5)
    sy5 = c5_systems(range(8), code5, lo=-2, hi=2)
    _check_rowwise(code5, sy5.masks, sy5.d, sy5.r)


def _check_incremental(code, masks, d, r, flip=None):
    """Alg. 6 on the GPU (precond = 3): the pivot sequence, read back in pick order, equals the
    reversed lower-triangular Triangulation Step ordering of the oracle's mts_incremental."""
    from oracle.precond import mts_incremental
    out = _run(code, masks, d, r, flip, precond=3)
    for s in range(masks.shape[0]):
        A, rows = dense_step_matrix(code, masks[s], None if flip is None else flip[s])
        if not rows:
            continue
        w2 = step_weights(code, d[s], rows)
        col, row = mts_incremental(A, w2)
        p = len(rows)
        assert len(col) == p, "Alg. 6 must reach |M| = p (P:656)"
        exp_rows = [rows[rw] for rw in row][::-1]          # stored reversed (upper triangular)
        exp_cols = [oracle_col_to_gpu(code, rows, c) for c in col][::-1]
        assert list(out["prow"][s][:p]) == exp_rows, f"system {s}: incremental pivot rows differ"
        assert list(out["pcol"][s][:p]) == exp_cols, f"system {s}: incremental pivot cols differ"
        _check_system(code, masks[s], d[s], r[s], None if flip is None else flip[s], out, s, tol_dy=1e-8,
                      check_pivots=False)
    return out


def test_incremental_mts_matches_oracle_alg6():
    """SURVEY f-1: Alg. 6 with the Triangulation Step bit-exact vs the oracle on
    config-1 systems with partial rows and flips, and on all-equal weights (tie rules)."""
    code = config_code(1)
    S = 16
    sy = c5_systems(range(S), code, lo=-3, hi=3, present_frac=0.7)
    flip = np.random.default_rng(12).integers(0, 2, size=(S, code.n)).astype(np.uint8)
    _check_incremental(code, sy.masks, sy.d, sy.r, flip)
    _check_incremental(code, sy.masks[:6], np.ones_like(sy.d[:6]), sy.r[:6], flip[:6])


def test_thm5_rowwise_contains_basic_columns_near_integral_optimum():
    """Thm 5: near the optimum of an LP with an integral solution, the row-wise MTS
    contains every basic column.  Late-IPM weights are formed from the oracle's LP optimum x*
    (basic: x* = 1 or slack > 0 -> d^2 = x*/(mu/x*), nonbasic -> d^2 = (mu/z)/z, z = 1), mu =
    1e-8; the GPU's Alg. 8 pivot columns must include all basic columns.  Column-wise (Alg. 7,
    for which the paper claims no such property) is reported for comparison."""
    from oracle.lp import malp_decode, augmented_lp, ipm_solve
    code = config_code(1)
    fb = config_frames(1, frames=range(12))
    cover_col = []
    for f in range(fb.F):
        o = malp_decode(code, fb.llr[f])
        if o["cert"] != 1 or not o["pool"]:
            continue
        lp = augmented_lp(code, o["pool"], fb.llr[f])
        x = ipm_solve(lp["A"], lp["b"], lp["c"])["x"]
        basic = np.nonzero(x > 0.5)[0]                      # integral LP: x* in {0, 1} on std, slack >= 0
        basic = np.array([c for c in range(lp["q"]) if x[c] > 1e-3])
        mu = 1e-8
        d2 = np.where(x > 1e-3, np.maximum(x, 1e-3) ** 2 / mu, mu)
        rows = lp["rows"]
        masks = np.zeros((1, code.m), dtype=np.uint16)
        for rr, j in enumerate(rows):
            masks[0, j] = o["masks"][j]
        d = np.ones((1, code.n + code.m))
        d[0, :code.n] = np.sqrt(d2[:code.n])
        for rr, j in enumerate(rows):
            d[0, code.n + j] = np.sqrt(d2[code.n + rr])
        flip = (fb.llr[f:f + 1] < 0).astype(np.uint8)
        r = np.random.default_rng(f).standard_normal((1, code.m))
        outs = {}
        for pc in (2, 0):
            out = _run(code, masks, d, r, flip, precond=pc)
            cols = set(int(c) for c in out["pcol"][0][:len(rows)])
            gpu_basic = {c if c < code.n else code.n + rows[c - code.n] for c in basic}
            outs[pc] = gpu_basic <= cols
        assert outs[2], f"frame {f}: row-wise MTS misses a basic column (Thm 5)"
        cover_col.append(outs[0])
    assert cover_col, "no certified frame with cuts in the sample"
    print(f"Thm 5: row-wise covers the basic set on {len(cover_col)}/{len(cover_col)} LPs; "
          f"column-wise on {sum(cover_col)}/{len(cover_col)}")
