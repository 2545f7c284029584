"""GPU ipm_step_pcg on captured late-IPM Newton systems (scratch/caps.pkl): status, iterations,
true residual and dual-step error vs the extended-precision exact solve."""
import sys, os, pickle
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from oracle.lp import normal_matrix, cholesky_solve, step_solve_exact
from synth import config_code

code = config_code(2)
c = alp.Code.from_synth(code)
caps = pickle.load(open(os.path.join(os.path.dirname(__file__), "..", "scratch", "caps.pkl"), "rb"))
key = {tuple(code.N(j)): j for j in range(code.m)}
n, m = code.n, code.m
for precond in (0, 1):
    for k, (A, d2, w) in enumerate(caps):
        A = A.astype(float)
        p = A.shape[0]
        masks = np.zeros((1, m), dtype=np.uint16); d = np.ones((1, n + m)); r = np.zeros((1, m)); rows = []
        for rr in range(p):
            j = key[tuple(np.nonzero(A[rr, :n])[0])]; rows.append(j)
            wd = 0x8000
            for t, i in enumerate(code.N(j)):
                if A[rr, i] > 0: wd |= 1 << t
            masks[0, j] = wd; r[0, j] = w[rr]; d[0, n + j] = np.sqrt(d2[n + rr])
        d[0, :n] = np.sqrt(d2[:n])
        res = alp.ipm_step_pcg(c, torch.from_numpy(masks.view(np.int16)).cuda(), torch.from_numpy(d).cuda(),
                               torch.from_numpy(r).cuda(), params=alp.default_params(precond=precond))
        torch.cuda.synchronize()
        y = res.dy.cpu().numpy()[0][rows]
        Q = normal_matrix(A, d2)
        ye = step_solve_exact(A, d2, w)
        yc = cholesky_solve(Q, w)
        dz = np.abs(A.T @ (y - ye)).max(); dzc = np.abs(A.T @ (yc - ye)).max()
        print("precond %d step %2d st %3d its %4d relres %.1e tres %.1e dz %.1e (chol dz %.1e)" % (
            precond, k, int(res.status[0]), int(res.iters[0]), float(res.relres[0]),
            np.linalg.norm(w - Q @ y) / np.linalg.norm(w), dz, dzc), flush=True)
