"""Why the slowest C2 frames are slow (they set the kernel time at 2.0 / 2.5 dB): decode a few
named frames alone with the per-Newton-step trace on and summarise, per frame, the PCG
iterations, sweep level counts (back / forward), p, and cycles per PCG iteration.
  SNR=0 FRAMES=1356,4061,2158 python tools/straggler_trace.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

REC = np.dtype([("frame", "<i4"), ("lp", "<i4"), ("it", "<i4"), ("p", "<i4"), ("status", "<i4"),
                ("iters", "<i4"), ("nLb", "<i4"), ("nLf", "<i4"), ("relres", "<f8"), ("rec", "<f8"), ("d2min", "<f8"),
                ("d2max", "<f8"), ("mu", "<f8"), ("rb", "<f8"), ("rc", "<f8"), ("gap", "<f8"), ("bP", "<f8"), ("bD", "<f8")])
snr = int(os.environ.get("SNR", "0"))
frames = [int(v) for v in os.environ.get("FRAMES", "1356,4061,2158").split(",")]
prm = alp.default_params(**eval(os.environ.get("PRM", "{}")))
code = config_code(2)
fb = config_frames(2, snr, frames=frames)
c = alp.Code.from_synth(code)
cap = 200000
buf = torch.zeros(cap * REC.itemsize, dtype=torch.uint8, device="cuda")
alp.lib().alp_debug_trace(buf.data_ptr(), cap)
torch.cuda.synchronize()
res = alp.decode(c, torch.from_numpy(fb.llr).cuda(), prm)
torch.cuda.synchronize()
alp.lib().alp_debug_trace(None, 0)
tr = np.frombuffer(buf.cpu().numpy().tobytes(), dtype=REC)
tr = tr[tr["p"] > 0]
st = res.stats_numpy()
for k, f in enumerate(frames):
    t = tr[tr["frame"] == k]
    cyc = {n: int(st[n][k]) for n in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other")}
    its = int(st["pcg_iters"][k])
    w = t["iters"].astype(np.float64)
    out = dict(frame=f, status=int(res.status.cpu().numpy()[k]), lps=int(st["lp_solves"][k]),
               ipm=int(st["ipm_iters"][k]), pcg=its, newton_steps=int(len(t)),
               capped_solves=int((t["iters"] >= prm.pcg_max_iter).sum()),
               p_mean=float(t["p"].mean()) if len(t) else 0,
               levels_back_mean_weighted=float((t["nLb"] * w).sum() / max(w.sum(), 1)),
               levels_fwd_mean_weighted=float((t["nLf"] * w).sum() / max(w.sum(), 1)),
               levels_back_max=int(t["nLb"].max()) if len(t) else 0,
               cyc_per_pcg_it={n: v / max(its, 1) for n, v in cyc.items()})
    print(json.dumps(out), flush=True)
