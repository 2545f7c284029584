"""GPU parity of alp_decode (Alg. 3 + §IV-B IPM + Alg. 4/7) against the oracle.

Gates, on the c.5 samples (C1 all 100 frames for MALP-A and
MALP-B, C2 the first 256 frames per Eb/N0, C3 the first 128), the oracle run over the same
seeded frames in a process pool:
  P1 hard decisions bit-exact where the oracle's |u_i - 1/2| > 1e-3
  P2 certificate bit-exact where |g_max - tau_cert| > 1e-3
  P3 |obj_gpu - obj_oracle| <= 1e-6 max(1, |obj_oracle|, ||gamma||inf)
  P4 every PCG solve's recursive ||r||/||w|| <= 1e-8: REPORTED as a failure count (the
     recovery of reading C-32 keeps the IPM exact on the rows an inexact dy would break)
  P6 the O(E) LP-duality certificate holds on every GPU frame that finished (any size)
  completion: the fraction of frames that finished their decode without a cap / cycle /
     non-finite status (ALP_MAXITER, IPM_MAXITER, NUMERIC) is at least the oracle's - 0.5 %.
P1-P3 compare frames that finished on both sides.  A parity report (counts per gate, LP- and
IPM-count match rates, P4 failures, PCG iterations integral / fractional) is written to
gpurun_out/parity/<name>.json.
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle.certify import dual_certificate, dual_certificate_batch
from synth import config_code, config_frames
from synth.codes import code_from_dense, code_from_rows
from tests.oracle_pool import oracle_decode

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(os.path.dirname(__file__), "golden")
CAP_BITS = 1 | 2 | 16        # ALP_MAXITER (cap or C-12 cycle), IPM_MAXITER, NUMERIC
P4_BITS = 4 | 8              # PCG_MAXITER / PCG_BREAKDOWN: some solve missed 1e-8 (P4 count)


def _alp():
    import paper_0902_0657_b200 as alp
    return alp


def gpu_decode(code, llr, **pkw):
    alp = _alp()
    c = alp.Code.from_synth(code)
    params = alp.default_params(**pkw)
    res = alp.decode(c, torch.from_numpy(np.ascontiguousarray(llr)).cuda(), params, want_u=True,
                     want_y=True, want_masks=True)
    torch.cuda.synchronize()
    assert alp.last_launch_count() == 1
    return dict(hard=res.hard.cpu().numpy(), obj=res.objective.cpu().numpy(),
                cert=res.certificate.cpu().numpy(), status=res.status.cpu().numpy(),
                stats=res.stats_numpy(), u=res.u.cpu().numpy(), y=res.y.cpu().numpy(),
                masks=res.masks.cpu().numpy().view(np.uint16))


def finished(status):
    return (np.asarray(status) & CAP_BITS) == 0


def write_report(name, rep):
    d = os.path.join(ROOT, "gpurun_out", "parity")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, name + ".json"), "w") as fh:
        json.dump(rep, fh, indent=1, default=float)
    print(name, json.dumps(rep, default=float))


def parity(name, code, llr, g, orc, frames=None, completion=True):
    """P1-P3 on the frames both sides finished, completion vs the oracle, the report."""
    frames = list(range(len(orc))) if frames is None else list(frames)
    st_o = np.array([o["status"] for o in orc])
    fin_o = finished(st_o)
    fin_g = finished(g["status"][frames])
    rep = dict(frames=len(frames), gpu_finished=int(fin_g.sum()), oracle_finished=int(fin_o.sum()),
               gpu_status_bits={str(b): int(((g["status"][frames] & b) != 0).sum()) for b in (1, 2, 4, 8, 16)},
               oracle_status_bits={str(b): int(((st_o & b) != 0).sum()) for b in (1, 2, 16)},
               oracle_chol_fix_frames=int(sum(1 for o in orc if o["chol_fixes"])))
    p1 = p2 = p3 = n_cmp = p2n = lp_m = ipm_m = 0
    bad = []
    for k, f in enumerate(frames):
        o = orc[k]
        if not (fin_o[k] and fin_g[k]):
            continue
        n_cmp += 1
        u = o["u"]
        sure = np.abs(u - 0.5) > 1e-3
        ok1 = np.array_equal(g["hard"][f][sure], o["hard"][sure])
        ok2 = True
        if abs(o["g_max"] - 1e-2) > 1e-3:
            p2n += 1
            ok2 = g["cert"][f] == o["cert"]
            p2 += int(ok2)
        scale = max(1.0, abs(o["obj"]), float(np.max(np.abs(llr[f]))))
        ok3 = abs(g["obj"][f] - o["obj"]) <= 1e-6 * scale
        p1 += int(ok1)
        p3 += int(ok3)
        lp_m += int(g["stats"]["lp_solves"][f] == o["lp_solves"])
        ipm_m += int(g["stats"]["ipm_iters"][f] == o["ipm_iters"])
        if not (ok1 and ok2 and ok3):
            bad.append(dict(frame=int(f), p1=bool(ok1), p2=bool(ok2), p3=bool(ok3),
                            obj_gpu=float(g["obj"][f]), obj_oracle=float(o["obj"]),
                            gpu_status=int(g["status"][f]), lps=(int(g["stats"]["lp_solves"][f]), int(o["lp_solves"]))))
    st = g["stats"][frames]
    integral = g["cert"][frames] == 1
    rep.update(compared=n_cmp, P1=p1, P2=p2, P2_applicable=p2n, P3=p3,
               lp_count_match=lp_m / max(1, n_cmp), ipm_count_match=ipm_m / max(1, n_cmp),
               P4_solves=int(st["pcg_solves"].sum()), P4_failed_solves=int(st["pcg_p4_fail"].sum()),
               P4_frames_with_failure=int((st["pcg_p4_fail"] > 0).sum()),
               true_residual_failed_solves=int(st["pcg_true_fail"].sum()),
               max_recursive_relres=float(st["max_rec_relres"].max()) if len(frames) else 0.0,
               pcg_iters_per_frame_integral=float(st["pcg_iters"][integral].mean()) if integral.any() else None,
               pcg_iters_per_frame_fractional=float(st["pcg_iters"][~integral].mean()) if (~integral).any() else None,
               gpu_cert=int(integral.sum()), oracle_cert=int(sum(o["cert"] for o in orc)),
               mismatches=bad[:20])
    write_report(name, rep)
    assert not bad, bad[:5]
    # completion: GPU finished fraction >= oracle's - 0.5 % (against the oracle's own IPM path;
    # the library-LP oracle has no IPM cap to match)
    if completion:
        assert fin_g.mean() >= fin_o.mean() - 0.005, (fin_g.mean(), fin_o.mean())
    return rep


def assert_certified(code, llr, g):
    """P6 (the O(E) duality certificate of oracle/certify.py) on every frame that finished its
    decode, plus Thm 2a / Cor. 4 / Cor. 5 invariants on those frames."""
    sel = np.nonzero(finished(g["status"]))[0]
    u = g["u"][sel]
    assert np.all(u >= -1.001e-6) and np.all(u <= 1 + 1.001e-6)
    hd = (llr[sel] < 0).astype(np.uint8)
    assert np.all((np.abs(u - hd) > 1e-3).sum(axis=1) <= code.m)          # Cor. 4 (G3)
    assert np.all(((u > 1e-3) & (u < 1 - 1e-3)).sum(axis=1) <= code.m)    # Cor. 5
    cert = dual_certificate_batch(code, llr[sel], g["u"][sel], g["y"][sel], g["masks"][sel])
    badm = ~cert["ok"]
    bad = sel[badm]
    if bad.size:
        f = int(bad[0])
        why = dual_certificate(code, llr[f], g["u"][f], g["y"][f], g["masks"][f])
        print("P6 failure detail, frame", f, why.get("reasons"))
    assert bad.size == 0, (f"P6 certificate fails on frames {bad[:10]}: min_lhs "
                           f"{cert['min_lhs'][badm][:5]}, gap {cert['gap'][badm][:5]}, "
                           f"status {g['status'][bad[:5]]}")
    return sel.size


def test_h7_golden_fractional_output():
    g = json.load(open(os.path.join(GOLD, "h7_trace.json")))
    code = code_from_dense(np.array([[int(c) for c in r] for r in g["H"]]))
    llr = np.array([g["gamma"]])
    for variant in (0, 1):
        out = gpu_decode(code, llr, variant=variant)
        np.testing.assert_allclose(out["u"][0], g["trace"][-1]["u"], atol=1e-7)
        assert out["cert"][0] == 0
        assert out["obj"][0] == pytest.approx(g["trace"][-1]["obj"], abs=1e-7)
        assert out["stats"]["lp_solves"][0] == len(g["trace"])
        assert out["stats"]["max_p"][0] == 3


def test_h1_examples_and_zero_lp_frames():
    code = code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1")
    llr = np.array([[-3.0, 1.0, 2.0, -1.0], [1.0, 1.0, 1.0, 1.0], [-1.0, -2.0, 3.0, 4.0]])
    out = gpu_decode(code, llr)
    np.testing.assert_allclose(out["u"][0], [1, 1, 0, 1], atol=1e-7)
    assert list(out["cert"]) == [1, 1, 0]
    assert out["stats"]["lp_solves"][1] == 0 and out["obj"][1] == 0.0     # C-15
    # (1,1,0,0) violates check 1: two LPs end at the fractional (1, 1/2, 1/2, 0), objective -1/2
    np.testing.assert_allclose(out["u"][2], [1, 0.5, 0.5, 0], atol=1e-7)
    assert out["stats"]["lp_solves"][2] == 2 and abs(out["obj"][2] + 0.5) <= 1e-6


@pytest.mark.parametrize("variant", ["A", "B"])
def test_config1_all_frames(variant):
    code = config_code(1)
    fb = config_frames(1)
    g = gpu_decode(code, fb.llr, variant=0 if variant == "A" else 1)
    orc = oracle_decode(1, range(fb.F), variant=variant)
    rep = parity(f"C1_malp{variant}", code, fb.llr, g, orc)
    assert rep["gpu_finished"] == fb.F
    assert assert_certified(code, fb.llr, g) == fb.F


@pytest.mark.parametrize("snr_idx", [0, 1, 2])
def test_config2_sample(snr_idx):
    """C2, first 256 frames at 2.0 / 2.5 / 3.0 dB (c.5)."""
    code = config_code(2)
    fb = config_frames(2, snr_idx, frames=range(256))
    g = gpu_decode(code, fb.llr)
    orc = oracle_decode(2, range(256), snr_idx=snr_idx)
    parity(f"C2_snr{snr_idx}", code, fb.llr, g, orc)
    # the same frames against Alg. 3 with the LP step by HiGHS (oracle/lp_library.py): it has no
    # IPM cap, so every frame the GPU finished is compared, also those the IPM oracle gave up on
    orl = oracle_decode(2, range(256), snr_idx=snr_idx, library=True, chunk=8)
    for o in orl:
        o["ipm_iters"] = -1
    rep = parity(f"C2_snr{snr_idx}_library", code, fb.llr, g, orl, completion=False)
    assert rep["compared"] >= rep["gpu_finished"] - 2, rep     # (the library path may stop on a C-12 cycle)
    assert_certified(code, fb.llr, g)
    # sanity: certified frames decode to a codeword no worse than the transmitted one
    tx_cost = (fb.codewords * fb.llr).sum(axis=1)
    cf = g["cert"] == 1
    assert np.all(g["obj"][cf] <= tx_cost[cf] + 1e-6)
    assert np.all((g["status"][cf] & (2 | 16)) == 0)    # C-31: only converged LPs certify


def test_config3_sample():
    """C3 (3,12) n=4000, first 128 frames (c.5); objectives ~0, so P3 is the absolute 1e-6."""
    code = config_code(3)
    fb = config_frames(3, frames=range(128))
    g = gpu_decode(code, fb.llr)
    orc = oracle_decode(3, range(128))
    parity("C3", code, fb.llr, g, orc)
    assert_certified(code, fb.llr, g)
    # a wider sample (the first 1,024 frames) against the library-LP oracle (oracle/lp_library.py)
    fw = config_frames(3, frames=range(1024), code=code)
    gw = gpu_decode(code, fw.llr)
    orl = oracle_decode(3, range(1024), library=True, chunk=16)
    for o in orl:
        o["ipm_iters"] = -1
    rep = parity("C3_library_1024", code, fw.llr, gw, orl, completion=False)
    assert rep["compared"] >= 0.98 * 1024, rep
    assert_certified(code, fw.llr, gw)


@pytest.mark.parametrize("F", [1, 37])
def test_ragged_batches_and_determinism(F):
    code = config_code(1)
    fb = config_frames(1, frames=range(F))
    a = gpu_decode(code, fb.llr)
    b = gpu_decode(code, fb.llr)
    for k in ("hard", "obj", "cert", "u", "y", "masks"):
        assert np.array_equal(a[k], b[k]), k
    parity(f"C1_ragged{F}", code, fb.llr, a, oracle_decode(1, range(min(F, 5))), range(min(F, 5)))


def test_rank_shards_equal_single_rank_decode():
    """decoding the frame shards f mod N (N = 2, 3) in separate calls gives,
    frame by frame, bit-identical outputs to one call over all frames (frames are independent;
    the multi-GPU path is exactly this split)."""
    from paper_0902_0657_b200.dist import shard_frame_ids
    code = config_code(2)
    F = 96
    fb = config_frames(2, 1, frames=range(F))
    whole = gpu_decode(code, fb.llr)
    for ws in (2, 3):
        for r in range(ws):
            ids = shard_frame_ids(F // ws, r, ws)
            part = gpu_decode(code, fb.llr[ids])
            for k in ("hard", "obj", "cert", "u", "y", "masks", "status"):
                assert np.array_equal(part[k], whole[k][ids]), (ws, r, k)


def test_empty_batch_and_extreme_llrs():
    alp = _alp()
    code = config_code(1)
    c = alp.Code.from_synth(code)
    r = alp.decode(c, torch.zeros((0, code.n), dtype=torch.float64, device="cuda"))
    assert r.hard.shape == (0, code.n)
    fb = config_frames(1, frames=range(8))
    llr = fb.llr * 100.0
    g = gpu_decode(code, llr)
    assert_certified(code, llr, g)
    parity("C1_llr_x100", code, llr, g, oracle_decode(1, range(8), llr_scale=100.0))


def test_certificate_needs_converged_lp():
    """C-31: with a 3-step IPM cap every LP stops unconverged, so no frame may certify."""
    code = config_code(1)
    fb = config_frames(1, frames=range(16))
    g = gpu_decode(code, fb.llr, ipm_max_iter=3)
    lp = g["stats"]["lp_solves"] > 0
    assert lp.any()
    assert np.all(g["cert"][lp] == 0)
    assert np.all((g["status"][lp] & 2) != 0)


@pytest.mark.slow
def test_config2_full_batch_certified():
    """16,384 frames at 3.0 dB (the bench workload, same launch configuration): P6 on every
    frame that finished; completion and P1-P3 on a 64-frame oracle sample spread over the batch,
    P1-P3 on 2,048 frames against the library-LP oracle."""
    code = config_code(2)
    fb = config_frames(2, 2)
    g = gpu_decode(code, fb.llr)
    n = assert_certified(code, fb.llr, g)
    assert n >= 0.99 * fb.F
    sample = np.random.default_rng(1).choice(fb.F, 64, replace=False)
    orc = oracle_decode(2, sample, snr_idx=2)
    parity("C2_full_sample", code, fb.llr, g, orc, sample)
    # every 8th frame of the batch (2,048 frames) against Alg. 3 with the LP step by HiGHS
    # (oracle/lp_library.py; ~0.3 s per frame per core)
    wide = list(range(0, fb.F, 8))
    orl = oracle_decode(2, wide, snr_idx=2, library=True, chunk=16)
    for o in orl:
        o["ipm_iters"] = -1
    rep = parity("C2_full_library_2048", code, fb.llr, g, orl, wide, completion=False)
    assert rep["compared"] >= 0.99 * len(wide), rep


def test_config1_plain_cg_decode():
    """SURVEY f-1 baseline: the same decode with plain CG (precond = 1) instead of the
    column-wise MTS preconditioner reaches the same LP outputs (P1-P3, P6).  Without a
    preconditioner ~10 % of the Newton solves end at the PCG cap (CG stalls on these
    systems), so the IPM needs more steps than with a direct solve; it gets ipm_max_iter = 200
    (the oracle keeps 100), so completion does not hinge on rounding-chaotic cap hits."""
    code = config_code(1)
    fb = config_frames(1, frames=range(32))
    g = gpu_decode(code, fb.llr, precond=1, ipm_max_iter=200)
    parity("C1_plain_cg", code, fb.llr, g, oracle_decode(1, range(32)))
    assert_certified(code, fb.llr, g)


def test_config4_golden_frames():
    """Config 4 (n = 32,000, m = 16,000, 2.2 dB; the large-n layout: phase window in global
    memory): the first 32 frames against the oracle outputs written offline by
    tools/make_c4_golden_library.py (calls only oracle/: Alg. 3 of oracle/lp.py with the LP step
    solved by HiGHS, oracle/lp_library.py, pinned in tests/test_oracle_library_lp.py — the
    oracle's dense IPM needs an hour per frame and ends on its Newton-step cap there).
    P1-P3 and the LP count on every frame both sides finished, completion, P6 on every frame."""
    import glob
    files = sorted(glob.glob(os.path.join(GOLD, "c4_library_f*.npz")),
                   key=lambda f: int(os.path.basename(f)[len("c4_library_f"):-4]))
    assert len(files) >= 2, "tests/golden/c4_library_f*.npz missing (python tools/make_c4_golden_library.py 0 1 ...)"
    gold = [dict(np.load(f)) for f in files]
    frames = [int(g["frame"]) for g in gold]
    code = config_code(4)
    fb = config_frames(4, frames=frames, code=code)
    orc = []
    for k, o in enumerate(gold):
        assert abs(float(o["llr_checksum"]) - float(np.sum(fb.llr[k] ** 2))) <= 1e-9 * float(o["llr_checksum"])
        assert int(o["p6_ok"]) == 1      # the oracle's own (u, y, pool) passed the duality certificate
        u = np.unpackbits(o["hard_u"])[:code.n].astype(np.float64)
        u[o["frac_idx"]] = o["frac_val"]
        orc.append(dict(u=u, hard=(u > 0.5).astype(np.uint8), obj=float(o["obj"]), g_max=float(o["g_max"]),
                        cert=int(o["cert"]), status=int(o["status"]), lp_solves=int(o["lp_solves"]),
                        ipm_iters=-1, chol_fixes=0))
    g = gpu_decode(code, fb.llr)
    # completion is not gated against this oracle (it has no IPM, hence no cap and no C-12 cycle:
    # at n = 32,000 the IPM's u is accurate to ~1e-5 — its gap tolerance is relative to |c^T x| ~ 5e4 —
    # which is above tau_viol = tau_act = 1e-6, so a few GPU frames end on a repeated pool (C-12)
    # with the last solved u; measured 3 of 32).  Those frames are compared too and reported apart.
    rep = parity("C4_library", code, fb.llr, g, orc, completion=False)
    assert rep["compared"] >= 0.85 * len(frames), rep
    cyc = [k for k, f in enumerate(frames) if g["status"][k] == 1]
    cyc_ok = 0
    for k in cyc:
        o = orc[k]
        scale = max(1.0, abs(o["obj"]), float(np.max(np.abs(fb.llr[k]))))
        cyc_ok += int(np.array_equal(g["hard"][k], o["hard"]) and g["cert"][k] == o["cert"]
                      and abs(g["obj"][k] - o["obj"]) <= 1e-6 * scale)
    rep.update(cycle_frames=len(cyc), cycle_frames_equal_to_oracle=cyc_ok)
    write_report("C4_library", rep)
    # (reported, not gated: the last solved u of a C-12 stop need not be the final LP's optimum)
    assert_certified(code, fb.llr, g)


def test_config1_rowwise_mts_decode():
    """SURVEY f-1: the decode with the row-wise MTS preconditioner (precond = 2, Alg. 8) reaches
    the same LP outputs (P1-P3, P6) as the oracle."""
    code = config_code(1)
    fb = config_frames(1, frames=range(48))
    g = gpu_decode(code, fb.llr, precond=2)
    parity("C1_rowwise", code, fb.llr, g, oracle_decode(1, range(48)))
    assert_certified(code, fb.llr, g)


def test_bsc_jittered_frames_vs_oracle():
    """SURVEY f-4: BSC frames with LLR jitter (synth/bsc.py) decode on the GPU to the
    oracle's LP outputs (P1-P3) and certify (P6)."""
    from synth import bsc_frames
    code = config_code(1)
    fb = bsc_frames(code, 0.04, 1e-3, 3003, range(48))
    g = gpu_decode(code, fb.llr)
    from oracle.lp import malp_decode
    orc = [malp_decode(code, fb.llr[f]) for f in range(fb.F)]
    parity("C1_bsc_jitter", code, fb.llr, g, orc)
    assert_certified(code, fb.llr, g)
