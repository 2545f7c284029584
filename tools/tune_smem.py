"""Decode-time sweep over the shared-memory split (frames per SM) on C2 at 3.0 dB."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

F = int(os.environ.get("F", "4096"))
code = config_code(2)
fb = config_frames(2, 2, frames=range(F))
c = alp.Code.from_synth(code)
llr = torch.from_numpy(fb.llr).cuda()
ref = None
for cfg in os.environ.get("CFGS", "4:12").split(","):
    wpb, fps = (int(v) for v in cfg.split(":"))
    p = alp.default_params(smem_frames_per_sm=fps, warps_per_block=wpb)
    res = alp.decode(c, llr, p)
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = alp.decode(c, llr, p)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    st = res.stats_numpy()
    cyc = {k: float(st[k].sum()) for k in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other", "cyc_sort", "cyc_peel")}
    its = st["pcg_iters"].sum()
    obj = res.objective.cpu().numpy()
    same = "n/a" if ref is None else ("%.1e" % np.max(np.abs(obj - ref) / np.maximum(1, np.abs(ref))))
    ref = obj if ref is None else ref
    print("wpb %d fps %2d: %.3f s  %.0f frames/s | per PCG it: spmv %.0f sweep %.0f other %.0f cyc | per IPM it: build %.0f (sort %.0f peel %.0f) body %.0f, PCG its/IPM it %.1f | obj diff %s" % (
        wpb, fps, dt, F / dt, cyc["cyc_spmv"] / its, cyc["cyc_sweep"] / its, cyc["cyc_pcg_other"] / its,
        cyc["cyc_build"] / st["ipm_iters"].sum(), cyc["cyc_sort"] / st["ipm_iters"].sum(),
        cyc["cyc_peel"] / st["ipm_iters"].sum(), cyc["cyc_ipm"] / st["ipm_iters"].sum(),
        its / st["ipm_iters"].sum(), same), flush=True)
