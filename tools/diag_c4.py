"""Times the config-4 decode (n = 32,000) of a few frames on the GPU (large-n layout)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames
F = int(os.environ.get("NF", "1"))
code = config_code(4)
t0 = time.time()
fb = config_frames(4, frames=range(F), code=code)
print(f"frames generated in {time.time() - t0:.1f}s", flush=True)
c = alp.Code.from_synth(code)
t = time.time()
res = alp.decode(c, torch.from_numpy(fb.llr).cuda())
torch.cuda.synchronize()
dt = time.time() - t
st = res.stats_numpy()
print(f"{F} frames in {dt:.1f}s; status {res.status.cpu().numpy().tolist()} cert {res.certificate.cpu().numpy().tolist()}")
for k in ("lp_solves", "ipm_iters", "pcg_iters", "max_p", "pcg_p4_fail"):
    print(k, st[k].tolist())
for k in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other", "cyc_sort", "cyc_peel"):
    print(k, (st[k] / 1e6).round(1).tolist(), "Mcyc")
print("obj", res.objective.cpu().numpy().tolist())
