"""Per-Newton-step trace of the GPU decode on C2 frames (alp_debug_trace)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

REC = np.dtype([("frame", "<i4"), ("lp", "<i4"), ("it", "<i4"), ("p", "<i4"), ("status", "<i4"),
                ("iters", "<i4"), ("nLb", "<i4"), ("nLf", "<i4"), ("relres", "<f8"), ("rec", "<f8"), ("d2min", "<f8"),
                ("d2max", "<f8"), ("mu", "<f8"), ("rb", "<f8"), ("rc", "<f8"), ("gap", "<f8"), ("bP", "<f8"), ("bD", "<f8")])
snr = int(os.environ.get("SNR", "0"))
frames = [int(a) for a in os.environ.get("FRAMES", "1,2,3").split(",")]
code = config_code(2)
fb = config_frames(2, snr, frames=frames)
c = alp.Code.from_synth(code)
cap = 200000
buf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device="cuda")
alp.lib().alp_debug_trace(buf.data_ptr(), cap)
res = alp.decode(c, torch.from_numpy(fb.llr).cuda())
torch.cuda.synchronize()
alp.lib().alp_debug_trace(None, 0)
recs = buf.cpu().numpy().view(REC)
recs = recs[recs["iters"] + recs["p"] > 0]
recs = np.sort(recs, order=["frame", "lp", "it"])
st = res.stats_numpy()
for fi, f in enumerate(frames):
    print(f"frame {f}: lp {st['lp_solves'][fi]} ipm {st['ipm_iters'][fi]} pcg {st['pcg_iters'][fi]} status {int(res.status[fi])}")
    for r in recs[recs["frame"] == fi]:
        if r["status"] != 0 or r["it"] < 1 or r["iters"] > 60:
            print("   lp %2d it %3d p %3d st %3d its %4d relres %.1e d2 [%.0e %.0e] mu %.1e rb %.1e rc %.1e gap %.1e" % (
                r["lp"], r["it"], r["p"], r["status"], r["iters"], r["relres"], r["d2min"], r["d2max"], r["mu"],
                r["rb"], r["rc"], r["gap"]))
