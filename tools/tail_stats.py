"""Per-frame work distribution of a C2 decode (which frames set the kernel time): the frames
with the most PCG iterations, their LP / IPM counts and status, and the share of all PCG
iterations they hold."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

F = int(os.environ.get("F", "4096"))
code = config_code(2)
c = alp.Code.from_synth(code)
out = {}
params = alp.default_params(**eval(os.environ.get("PRM", "{}")))
for si in [int(v) for v in os.environ.get("SNRS", "0,1,2").split(",")]:
    fb = config_frames(2, si, frames=range(F))
    llr = torch.from_numpy(fb.llr).cuda()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    res = alp.decode(c, llr, params)
    b.record()
    torch.cuda.synchronize()
    st = res.stats_numpy()
    pcg = st["pcg_iters"].astype(np.int64)
    order = np.argsort(-pcg)
    tot = pcg.sum()
    top = [dict(frame=int(f), pcg=int(pcg[f]), lps=int(st["lp_solves"][f]), ipm=int(st["ipm_iters"][f]),
                status=int(res.status.cpu().numpy()[f]), cyc=int(sum(int(st[k][f]) for k in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other"))))
           for f in order[:12]]
    q = np.quantile(pcg, [0.5, 0.9, 0.99, 0.999, 1.0]).tolist()
    out[si] = dict(ms=a.elapsed_time(b), frames=F, pcg_total=int(tot), pcg_quantiles=q,
                   top10_share=float(pcg[order[:10]].sum() / tot), top=top)
    print(si, json.dumps(out[si]), flush=True)
