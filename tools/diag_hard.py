"""GPU diagnostics (run under gpurun): C2 frames at one Eb/N0 decoded under parameter variants;
per variant the capped / P4-failing frame counts, PCG iterations and time, and a per-Newton-step
trace (alp_debug_trace) of the first capped frames.  VARIANTS = JSON list of param dicts."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

REC = np.dtype([("frame", "<i4"), ("lp", "<i4"), ("it", "<i4"), ("p", "<i4"), ("status", "<i4"),
                ("iters", "<i4"), ("nLb", "<i4"), ("nLf", "<i4"), ("relres", "<f8"), ("rec", "<f8"), ("d2min", "<f8"), ("d2max", "<f8"),
                ("mu", "<f8"), ("rb", "<f8"), ("rc", "<f8"), ("gap", "<f8"), ("bP", "<f8"), ("bD", "<f8")])
snr = int(os.environ.get("SNR", "0"))
F = int(os.environ.get("NF", "256"))
variants = json.loads(os.environ.get("VARIANTS", "[{}]"))
ntrace = int(os.environ.get("NTRACE", "2"))
code = config_code(2)
fb = config_frames(2, snr, frames=range(F))
c = alp.Code.from_synth(code)
llr = torch.from_numpy(fb.llr).cuda()
cap = 400000
buf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device="cuda")
for v in variants:
    prm = alp.default_params(**v)
    alp.lib().alp_debug_trace(buf.data_ptr(), cap)
    torch.cuda.synchronize()
    t0 = time.time()
    res = alp.decode(c, llr, prm)
    torch.cuda.synchronize()
    dt = time.time() - t0
    alp.lib().alp_debug_trace(None, 0)
    st = res.status.cpu().numpy()
    s = res.stats_numpy()
    capped = np.nonzero(st & 19)[0]
    print(f"== variant {v}: {dt:.2f}s capped {capped.size} (ipm {int(((st & 2) != 0).sum())}, alp {int(((st & 1) != 0).sum())}) "
          f"p4-frames {int(((st & 12) != 0).sum())} pcg_iters {int(s['pcg_iters'].sum())} "
          f"p4 fails {int(s['pcg_p4_fail'].sum())}/{int(s['pcg_solves'].sum())} cert {int(res.certificate.sum())}")
    print("   capped frames", capped.tolist()[:40])
    order = np.argsort(-s["pcg_iters"])[:8]
    print("   top pcg frames", [(int(f), int(s['pcg_iters'][f]), int(s['ipm_iters'][f]), int(s['lp_solves'][f]), int(st[f])) for f in order])
    recs = buf.cpu().numpy().view(REC)
    recs = recs[recs["iters"] + recs["p"] > 0]
    for f in capped[:ntrace]:
        rr = np.sort(recs[recs["frame"] == f], order=["lp", "it"])
        print(f"   frame {f}: lp {s['lp_solves'][f]} ipm {s['ipm_iters'][f]} pcg {s['pcg_iters'][f]} status {st[f]}")
        last = rr["lp"].max() if rr.size else 0
        for r in rr:
            if r["lp"] >= last - 1:
                print("     lp %2d it %3d p %3d st %2d its %4d true %.1e rec %.1e d2 [%.0e %.0e] mu %.1e rb %.1e rc %.1e gap %.1e bP %.2e bD %.2e" % (
                    r["lp"], r["it"], r["p"], r["status"], r["iters"], r["relres"], r["rec"], r["d2min"], r["d2max"],
                    r["mu"], r["rb"], r["rc"], r["gap"], r["bP"], r["bD"]))
