"""Writes tests/golden/c4_oracle_f<k>.npz: the ORACLE's MALP-A decode of config-4 frames
(n = 32,000, m = 16,000, 2.2 dB; SURVEY §8(c) c.5 "C4 the first 2 (offline)").  Calls only
oracle/ and synth/ (never the CUDA path); each frame costs about an hour of CPU (dense
Cholesky of p ~ 1e4 per Newton step).  Result (round 2): frames 0 and 1 both ended on the
oracle's Newton-step cap (status IPM_MAXITER after 5436 s / 3894 s, > 1e5 C-29 pivot fixes), so
these outputs cannot gate P1-P3 and are no longer committed; the config-4 parity test uses
tools/make_c4_golden_library.py (the same Alg. 3 with the LP step solved by HiGHS) instead.

  python tools/make_c4_golden.py FRAME [FRAME ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle.lp import malp_decode
from synth import config_code, config_frames

if __name__ == "__main__":
    code = config_code(4)
    frames = [int(a) for a in sys.argv[1:]] or [0, 1]
    fb = config_frames(4, frames=frames, code=code)
    for t, f in enumerate(frames):
        t0 = time.time()
        o = malp_decode(code, fb.llr[t])
        out = os.path.join(ROOT, "tests", "golden", f"c4_oracle_f{f}.npz")
        np.savez_compressed(out, frame=f, u=o["u"], y=o["y"], masks=o["masks"], hard=o["hard"],
                            obj=o["obj"], g_max=o["g_max"], cert=o["cert"], status=o["status"],
                            lp_solves=o["lp_solves"], ipm_iters=o["ipm_iters"], max_p=o["max_p"],
                            chol_fixes=o["chol_fixes"], llr_checksum=float(np.sum(fb.llr[t] ** 2)),
                            seconds=time.time() - t0)
        print(f"frame {f}: status {o['status']} lps {o['lp_solves']} ipm {o['ipm_iters']} p {o['max_p']} "
              f"cert {o['cert']} obj {o['obj']:.6f} chol_fixes {o['chol_fixes']} {time.time() - t0:.0f}s", flush=True)
