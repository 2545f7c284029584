"""Config-5 step-solve variants (window mode x refinement): systems/s over 65,536 systems and the
forward error vs the oracle's exact solve on a 64-system sample (oracle in a process pool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, c5_systems
from tests.helpers import dense_step_matrix
from tests.oracle_pool import oracle_step_exact

def main():
    code = config_code(5)
    S = int(os.environ.get("S", "65536"))
    sy = c5_systems(range(S), code)
    c = alp.Code.from_synth(code)
    masks = torch.from_numpy(sy.masks.view(np.int16)).cuda()
    d = torch.from_numpy(sy.d).cuda()
    r = torch.from_numpy(sy.r).cuda()
    sample = list(range(64))
    orc = oracle_step_exact(sample)
    for name, kw in (("sm refine2", dict(pcg_refine=2)), ("sm refine1", dict(pcg_refine=1)),
                     ("sm refine0", dict(pcg_refine=0)), ("gm8 refine1", dict(pcg_refine=1, smem_frames_per_sm=8)),
                     ("gm8 refine2", dict(pcg_refine=2, smem_frames_per_sm=8))):
        prm = alp.default_params(**kw)
        res = alp.ipm_step_pcg(c, masks, d, r, params=prm)
        torch.cuda.synchronize()
        t = time.time()
        res = alp.ipm_step_pcg(c, masks, d, r, params=prm)
        torch.cuda.synchronize()
        dt = time.time() - t
        dy = res.dy[:64].cpu().numpy()
        errs = []
        for k, s in enumerate(sample):
            A, rows = dense_step_matrix(code, sy.masks[s])
            errs.append(np.linalg.norm(dy[s][rows] - orc[k][0]) / np.linalg.norm(orc[k][0]))
        st = res.status.cpu().numpy()
        print(f"{name}: {S / dt:.0f} systems/s, mean its {res.iters.float().mean().item():.1f}, "
              f"max err {max(errs):.2e} median {np.median(errs):.2e}, status {dict(zip(*[a.tolist() for a in np.unique(st, return_counts=True)]))}", flush=True)


if __name__ == "__main__":
    main()
