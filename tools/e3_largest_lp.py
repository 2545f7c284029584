""""the size of the largest LP that is solved in each MALP-A or MALP-B
decoding problem is smaller on average than that of ALP decoding by 17 % for integral outputs
and 30 % for fractional outputs".  CPU-only, oracle-only: plain ALP (Alg. 1, several cuts
per check — the one outer-loop variant the GPU path does not implement), MALP-A and
MALP-B through oracle/lp_library.py (Alg. 1 / Alg. 3 with the LP step by HiGHS) on the SAME seeded
codes and frames as tools/iteration_stats.py (E1/E2: code seed 3000 + n, frame seed 4000 + n,
all-zero codeword, AWGN 2 dB), so the MALP rows can be checked against the GPU's `max_p`
statistics in profiles/r2_iteration_stats.json.  Size of an LP = its number of cut rows p.
Output: profiles/r2_e3_largest_lp.json.

  python tools/e3_largest_lp.py            (env: LENGTHS=480,960 TRIALS=1000 SNR=2.0)
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

TRIALS = int(os.environ.get("TRIALS", "1000"))
LENGTHS = [int(v) for v in os.environ.get("LENGTHS", "480").split(",")]
SNR = float(os.environ.get("SNR", "2.0"))


def job(a):
    n, lo, hi = a
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle.lp import malp_decode
    from oracle.lp_library import library_lp_solve
    from synth import awgn_frames
    from synth.codes import regular_code
    code = regular_code(n, 3, 6, seed=3000 + n, girth6=True)
    fb = awgn_frames(code, SNR, 4000 + n, 0, range(lo, hi), random_codeword=False)
    out = []
    for f in range(fb.F):
        row = {}
        for v in ("ALP", "A", "B"):
            o = malp_decode(code, fb.llr[f], v, lp_solver=library_lp_solve)
            row[v] = (int(o["max_p"]), int(o["lp_solves"]), int(o["cert"]), int(o["status"]), float(o["obj"]))
        out.append(row)
    return out


if __name__ == "__main__":
    res = dict(snr_db=SNR, trials=TRIALS, source="oracle/lp_library.py (CPU); codes / frames of tools/iteration_stats.py",
               paper="P:385: MALP's largest LP smaller than ALP's by 17 % (integral) / 30 % (fractional)", lengths={})
    for n in LENGTHS:
        t0 = time.time()
        step = max(1, TRIALS // 64)
        jobs = [(n, lo, min(TRIALS, lo + step)) for lo in range(0, TRIALS, step)]
        with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
            rows = [r for part in pool.map(job, jobs) for r in part]
        ok = [r for r in rows if all(r[v][3] == 0 for v in r)]
        # Thm 2c: all three variants end at the same LP optimum
        dobj = max(max(abs(r["A"][4] - r["ALP"][4]), abs(r["B"][4] - r["ALP"][4])) for r in ok)
        row = dict(frames=len(rows), finished_all_variants=len(ok), max_objective_spread=dobj)
        for cls, sel in (("integral", 1), ("fractional", 0)):
            grp = [r for r in ok if r["ALP"][2] == sel]
            if not grp:
                continue
            m = {v: float(np.mean([r[v][0] for r in grp])) for v in ("ALP", "A", "B")}
            lps = {v: float(np.mean([r[v][1] for r in grp])) for v in ("ALP", "A", "B")}
            row[cls] = dict(n=len(grp), mean_largest_lp=m, mean_lp_solves=lps,
                            malp_a_vs_alp=m["A"] / m["ALP"] - 1.0, malp_b_vs_alp=m["B"] / m["ALP"] - 1.0)
        row["malp_a_mean_largest_lp_all"] = float(np.mean([r["A"][0] for r in ok]))
        row["malp_b_mean_largest_lp_all"] = float(np.mean([r["B"][0] for r in ok]))
        row["seconds"] = time.time() - t0
        res["lengths"][n] = row
        print(n, json.dumps(row), flush=True)
    json.dump(res, open(os.path.join(ROOT, "profiles", "r2_e3_largest_lp.json"), "w"), indent=1)
