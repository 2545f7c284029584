"""Writes tests/golden/c4_library_f<k>.npz: the ORACLE's MALP-A decode of config-4 frames
(n = 32,000, m = 16,000, 2.2 dB) with every LP solved by a library LP solver
(oracle/lp_library.py: Alg. 3 as in oracle/lp.py, the LP step by scipy HiGHS dual simplex).
The oracle's own dense IPM ends on its Newton-step cap on these frames after about an hour
each (tools/make_c4_golden.py), so its outputs cannot gate P1-P3; these can.  Calls only
oracle/ and synth/ (never the CUDA path).

  python tools/make_c4_golden_library.py FRAME [FRAME ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from oracle.certify import dual_certificate
from oracle.lp_library import malp_decode_library
from synth import config_code, config_frames

if __name__ == "__main__":
    code = config_code(4)
    frames = [int(a) for a in sys.argv[1:]] or [0, 1]
    fb = config_frames(4, frames=frames, code=code)
    for t, f in enumerate(frames):
        t0 = time.time()
        o = malp_decode_library(code, fb.llr[t])
        c = dual_certificate(code, fb.llr[t], o["u"], o["y"], o["masks"])
        out = os.path.join(ROOT, "tests", "golden", f"c4_library_f{f}.npz")
        # u as hard decision + the sparse set of fractional entries (a vertex: <= m of them, Cor. 5)
        frac = np.nonzero((o["u"] > 1e-9) & (o["u"] < 1 - 1e-9))[0].astype(np.int32)
        np.savez_compressed(out, frame=f, hard_u=np.packbits(o["u"] > 0.5), frac_idx=frac,
                            frac_val=o["u"][frac], masks=o["masks"],
                            obj=o["obj"], g_max=o["g_max"], cert=o["cert"], status=o["status"],
                            lp_solves=o["lp_solves"], simplex_iters=o["ipm_iters"], max_p=o["max_p"],
                            p6_ok=int(c["ok"]), llr_checksum=float(np.sum(fb.llr[t] ** 2)),
                            seconds=time.time() - t0)
        print(f"frame {f}: status {o['status']} lps {o['lp_solves']} simplex its {o['ipm_iters']} p {o['max_p']} "
              f"cert {o['cert']} g_max {o['g_max']:.3g} obj {o['obj']:.6f} nfrac {frac.size} P6 {c['ok']} "
              f"{time.time() - t0:.0f}s", flush=True)
