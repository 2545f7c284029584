"""Tiny decode for compute-sanitizer runs (C1, a few frames, and a small step solve)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames, c5_systems
F = int(os.environ.get("NF", "4"))
code = config_code(int(os.environ.get("CFG", "1")))
fb = config_frames(1, frames=range(F), code=code) if code.n == 120 else config_frames(2, 2, frames=range(F), code=code)
c = alp.Code.from_synth(code)
res = alp.decode(c, torch.from_numpy(fb.llr).cuda(), alp.default_params(**eval(os.environ.get("PRM", "{}"))))
torch.cuda.synchronize()
print("decode status", res.status.cpu().numpy().tolist(), "cert", res.certificate.cpu().numpy().tolist())
if os.environ.get("STEP", "1") == "1":
    sy = c5_systems(range(2), code, lo=-3, hi=3)
    st = alp.ipm_step_pcg(c, torch.from_numpy(sy.masks.view(np.int16)).cuda(), torch.from_numpy(sy.d).cuda(),
                          torch.from_numpy(sy.r).cuda())
    torch.cuda.synchronize()
    print("step status", st.status.cpu().numpy().tolist(), "iters", st.iters.cpu().numpy().tolist())
