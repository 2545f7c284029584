"""E5-style PCG residual traces (§VI-B, Figs. 5-8; SURVEY f-1), qualitative.

The paper compares CG with MTS-preconditioned CG on Newton systems of an n=2000 (3,6) code at
IPM iterations 8 and 18 of a MALP-A LP, for an integral (1.5 dB) and a fractional (1.0 dB) frame.
Here: our seeded n=2000 (3,6) code (4-cycles kept, reading C-21), the first frame at each SNR whose
MALP-A decode has >= 3 LPs; the LP solved third is run by the ORACLE's IPM (direct Cholesky step)
to capture the Newton systems at IPM iterations 8 and 18; each system is then solved on the GPU by
ipm_step_pcg with the column-wise MTS preconditioner (precond=0, Alg. 7), the row-wise MTS with
diagonal expansion (precond=2, Alg. 8) and plain CG (precond=1), capped at k = 1..K iterations,
giving the TRUE relative residual ||w - Q dy||/||w|| after k iterations (the paper plots the
squared ratio, G15).  The incremental MTS (precond=3, Alg. 6 with the Triangulation Step; O(q)
triangulations per build) is traced on the coarse grid k = 10, 20, ..., K.  Output:
gpurun_out/e5_traces.json.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0902_0657_b200 as alp
import oracle.lp as L
from synth import awgn_frames, regular_code

K = int(os.environ.get("K", "80"))
code = regular_code(2000, 3, 6, seed=1005, name="e5")
c = alp.Code.from_synth(code)
key = {tuple(code.N(j)): j for j in range(code.m)}
out = {}
for label, snr in (("integral_1.5dB", 1.5), ("fractional_1.0dB", 1.0)):
    for f in range(12):
        fb = awgn_frames(code, snr, 2005, 9, [f], random_codeword=False)
        o = L.malp_decode(code, fb.llr[0])
        want_frac = label.startswith("fractional")
        if o["lp_solves"] >= 3 and (o["cert"] == 0) == want_frac:
            break
    # re-run the third LP's IPM with capture
    pool_trace = L.malp_decode(code, fb.llr[0], record=True)["trace"]
    lp_pool = pool_trace[2]["pool"]
    lp = L.augmented_lp(code, lp_pool, fb.llr[0])
    seen = []

    def cap_solver(A, d2, w, info):
        seen.append((np.asarray(A.todense()) if hasattr(A, "todense") else np.asarray(A), d2.copy(), w.copy()))
        return L.cholesky_solve(L.normal_matrix(A, d2), w, info)

    L.ipm_solve(lp["A"], lp["b"], lp["c"], L.DEFAULT_PARAMS, step_solver=cap_solver)
    n, m = code.n, code.m
    for it in (8, 18):
        if it >= len(seen):
            continue
        A, d2, w = seen[it]
        p = A.shape[0]
        masks = np.zeros((1, m), dtype=np.uint16)
        d = np.ones((1, n + m))
        r = np.zeros((1, m))
        rows = []
        for rr in range(p):
            j = key[tuple(np.nonzero(A[rr, :n])[0])]
            rows.append(j)
            wd = 0x8000
            for t, i in enumerate(code.N(j)):
                if A[rr, i] > 0:
                    wd |= 1 << t
            masks[0, j] = wd
            r[0, j] = w[rr]
            d[0, n + j] = np.sqrt(d2[n + rr])
        d[0, :n] = np.sqrt(d2[:n])
        Q = L.normal_matrix(A, d2)
        tm = torch.from_numpy(masks.view(np.int16)).cuda()
        td = torch.from_numpy(d).cuda()
        tr = torch.from_numpy(r).cuda()
        curves = {}
        for name, pc in (("column-wise MTS", 0), ("row-wise MTS", 2), ("CG", 1), ("incremental MTS", 3)):
            res = []
            for k in (range(1, K + 1) if pc != 3 else range(10, K + 1, 10)):
                prm = alp.default_params(precond=pc, pcg_max_iter=k, pcg_rel_tol=1e-14)
                sol = alp.ipm_step_pcg(c, tm, td, tr, params=prm)
                torch.cuda.synchronize()
                y = sol.dy.cpu().numpy()[0][rows]
                res.append(float(np.linalg.norm(w - Q @ y) / np.linalg.norm(w)))
            curves[name] = res
        ev = np.linalg.eigvalsh(Q)
        out[f"{label} frame {f} LP3 IPM iteration {it}"] = {
            "p": p, "q": n + p, "kappa_Q": float(ev[-1] / max(ev[0], 1e-300)),
            "true_relres_after_k": curves}
        print(label, "frame", f, "it", it, "p", p, "kappa %.2e" % (ev[-1] / max(ev[0], 1e-300)),
              {k: ["%.1e" % v for v in (vals[9::10] if len(vals) == K else vals)] for k, vals in curves.items()},
              flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/e5_traces.json", "w"), indent=1)
