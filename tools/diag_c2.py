"""Per-Newton-step log of the oracle IPM driven by the GPU step solve on hard C2 frames."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from oracle.lp import malp_decode, cholesky_solve, normal_matrix
from synth import config_code, config_frames
from tools.diag_decode import gpu_step_solver

code = config_code(2)
fb = config_frames(2, 0, frames=range(64))
c = alp.Code.from_synth(code)
res = alp.decode(c, torch.from_numpy(fb.llr).cuda())
torch.cuda.synchronize()
status = res.status.cpu().numpy()
st = res.stats_numpy()
bad = [f for f in range(64) if status[f] & 7]
print("bad frames", bad[:10], "statuses", status[bad[:10]].tolist())
for f in bad[:2]:
    ref = malp_decode(code, fb.llr[f], record=True)
    print(f"frame {f}: oracle lp {ref['lp_solves']} ipm {ref['ipm_iters']} obj {ref['obj']:.9g} cert {ref['cert']} | gpu lp {st['lp_solves'][f]} ipm {st['ipm_iters'][f]} pcg {st['pcg_iters'][f]}")
    solver, log = gpu_step_solver(code, c)
    o = malp_decode(code, fb.llr[f], step_solver=solver)
    print(f"   oracle+gpuPCG lp {o['lp_solves']} ipm {o['ipm_iters']} status {o['status']} obj {o['obj']:.9g}")
    for k, e in enumerate(log[:400]):
        if e[3] != 0 or k % 10 == 0:
            print("   step %d p=%d its=%d relres=%.2e st=%d err=%.2e tres=%.2e d2=[%.1e,%.1e]" % ((k,) + e))
