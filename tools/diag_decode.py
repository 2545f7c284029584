"""GPU diagnostics (run under gpurun): per-frame decode counters vs the oracle, and the
oracle's IPM driven by the GPU's ipm_step_pcg as its step solver (every Newton system
compared with the oracle's Cholesky)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0902_0657_b200 as alp
from oracle.lp import malp_decode, cholesky_solve, normal_matrix
from synth import config_code, config_frames
from synth.codes import code_from_rows


def gpu_step_solver(code, c):
    key = {tuple(code.N(j)): j for j in range(code.m)}
    n, m = code.n, code.m
    log = []

    def solve(A, d2, w, info):
        A = np.asarray(A.todense()) if hasattr(A, "todense") else np.asarray(A)
        p = A.shape[0]
        masks = np.zeros((1, m), dtype=np.uint16)
        d = np.ones((1, n + m))
        r = np.zeros((1, m))
        rows = []
        for rr in range(p):
            nz = tuple(np.nonzero(A[rr, :n])[0])
            j = key[nz]
            rows.append(j)
            wd = 0x8000
            for t, i in enumerate(code.N(j)):
                if A[rr, i] > 0:
                    wd |= 1 << t
            masks[0, j] = wd
            r[0, j] = w[rr]
            d[0, n + j] = np.sqrt(d2[n + rr])
        d[0, :n] = np.sqrt(d2[:n])
        res = alp.ipm_step_pcg(c, torch.from_numpy(masks.view(np.int16)).cuda(), torch.from_numpy(d).cuda(),
                               torch.from_numpy(r).cuda())
        torch.cuda.synchronize()
        dy = res.dy.cpu().numpy()[0][rows]
        Q = normal_matrix(A, d2)
        ref = cholesky_solve(Q, w)
        err = np.linalg.norm(dy - ref) / max(1e-300, np.linalg.norm(ref))
        tres = np.linalg.norm(w - Q @ dy) / max(1e-300, np.linalg.norm(w))
        log.append((p, int(res.iters[0]), float(res.relres[0]), int(res.status[0]), err, tres,
                    float(d2.min()), float(d2.max())))
        info["pcg_iters"] = info.get("pcg_iters", 0) + int(res.iters[0])
        return dy

    return solve, log


def main():
    code = config_code(1)
    fb = config_frames(1, frames=range(12))
    c = alp.Code.from_synth(code)
    res = alp.decode(c, torch.from_numpy(fb.llr).cuda(), want_u=True)
    torch.cuda.synchronize()
    st = res.stats_numpy()
    status = res.status.cpu().numpy()
    obj = res.objective.cpu().numpy()
    print("frame | gpu status lp ipm pcg max_p obj | oracle lp ipm obj")
    for f in range(fb.F):
        o = malp_decode(code, fb.llr[f])
        print(f, "|", status[f], st["lp_solves"][f], st["ipm_iters"][f], st["pcg_iters"][f], st["max_p"][f],
              "%.9g" % obj[f], "|", o["lp_solves"], o["ipm_iters"], "%.9g" % o["obj"])
    # same with plain CG
    res2 = alp.decode(c, torch.from_numpy(fb.llr).cuda(), alp.default_params(precond=1))
    torch.cuda.synchronize()
    st2 = res2.stats_numpy()
    print("plain CG: status", res2.status.cpu().numpy().tolist())
    print("plain CG: obj", res2.objective.cpu().numpy().tolist())
    print("plain CG: ipm", st2["ipm_iters"].tolist(), "pcg", st2["pcg_iters"].tolist())
    # H1 example
    h1 = code_from_rows([[0, 1, 2], [1, 2, 3]], 4, "H1")
    llr = np.array([[-3.0, 1.0, 2.0, -1.0], [1.0, 1.0, 1.0, 1.0], [-1.0, -2.0, 3.0, 4.0]])
    r = alp.decode(alp.Code.from_synth(h1), torch.from_numpy(llr).cuda(), want_u=True)
    torch.cuda.synchronize()
    print("H1 gpu u", r.u.cpu().numpy().tolist(), "cert", r.certificate.cpu().tolist(), "status",
          r.status.cpu().tolist(), "stats", r.stats_numpy().tolist())
    for f in range(3):
        o = malp_decode(h1, llr[f])
        print("H1 oracle", o["u"].tolist(), o["cert"], o["lp_solves"], o["obj"])
    # oracle IPM with the GPU step solver, C1 frames 0..2
    for f in range(3):
        solver, log = gpu_step_solver(code, c)
        o = malp_decode(code, fb.llr[f], step_solver=solver)
        ref = malp_decode(code, fb.llr[f])
        print(f"frame {f}: oracle+gpuPCG obj {o['obj']:.9g} lp {o['lp_solves']} ipm {o['ipm_iters']} status {o['status']}"
              f" | oracle obj {ref['obj']:.9g} lp {ref['lp_solves']} ipm {ref['ipm_iters']}")
        print("   max pcg its %d, max true relres %.2e, statuses %s" % (max(e[1] for e in log), max(e[5] for e in log),
              sorted(set(e[3] for e in log))))


def corrected_newton(A, x, z, rb, rc, mu, step_solver=None, info=None):
    """Diagnostic twin of the GPU recovery (reading R-1): dz = r_c - A^T dy,
    dx_std = (r_e - x dz)/z, dx_slack = r_b - A_std dx_std."""
    import oracle.lp as L
    n = A.shape[1] - A.shape[0]
    re = mu - x * z
    d2 = x / z
    w = rb + A @ (d2 * rc - re / z)
    dy = step_solver(A, d2, w, info) if step_solver else L.cholesky_solve(L.normal_matrix(A, d2), w, info)
    dz = rc - A.T @ dy
    dx = (re - x * dz) / z
    Ad = np.asarray(A.todense()) if hasattr(A, "todense") else A
    dx[n:] = rb - Ad[:, :n] @ dx[:n]
    return dx, dy, dz


def c5_report():
    from synth import c5_systems
    from tests.helpers import dense_step_matrix, step_weights
    code = config_code(5)
    c = alp.Code.from_synth(code)
    for lo, hi in ((-6, 6), (-3, 3), (-1, 1), (-0.5, 0.5)):
        sy = c5_systems(range(8), code, lo=lo, hi=hi)
        res = alp.ipm_step_pcg(c, torch.from_numpy(sy.masks.view(np.int16)).cuda(), torch.from_numpy(sy.d).cuda(),
                               torch.from_numpy(sy.r).cuda())
        torch.cuda.synchronize()
        dy = res.dy.cpu().numpy()
        for s in range(sy.S):
            A, rows = dense_step_matrix(code, sy.masks[s])
            w2 = step_weights(code, sy.d[s], rows)
            Q = normal_matrix(A, w2)
            w = sy.r[s][rows]
            ref = cholesky_solve(Q, w)
            g = dy[s][rows]
            tres = np.linalg.norm(w - Q @ g) / np.linalg.norm(w)
            cres = np.linalg.norm(w - Q @ ref) / np.linalg.norm(w)
            floor = 8 * np.finfo(float).eps * np.linalg.norm(np.abs(A) @ (w2 * (np.abs(A).T @ np.abs(g)))) / np.linalg.norm(w)
            ev = np.linalg.eigvalsh(Q)
            bound = (np.linalg.norm(w - Q @ g) + np.linalg.norm(w - Q @ ref)) / ev[0] / np.linalg.norm(ref)
            err = np.linalg.norm(g - ref) / np.linalg.norm(ref)
            e = g - ref
            qerr = np.sqrt(abs(e @ Q @ e)) / np.sqrt(abs(ref @ Q @ ref))
            print("C5 d=10^U(%g,%g) s=%d its=%d relres=%.2e tres=%.2e chol_res=%.2e floor=%.2e err=%.2e bound=%.2e qerr=%.2e kappa=%.1e"
                  % (lo, hi, s, int(res.iters[s]), float(res.relres[s]), tres, cres, floor, err, bound, qerr, ev[-1] / ev[0]))


GAP = float(os.environ.get("GAP", "1e-9"))


def c2_sample(F=512, snr_idx=0, cfg=2):
    import time
    code = config_code(cfg)
    fb = config_frames(cfg, snr_idx, frames=range(F))
    c = alp.Code.from_synth(code)
    llr = torch.from_numpy(fb.llr).cuda()
    params = alp.default_params(gap_tol=GAP)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = alp.decode(c, llr, params)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    st = res.stats_numpy()
    status = res.status.cpu().numpy()
    vals, cnts = np.unique(status, return_counts=True)
    print(f"C{cfg} snr{snr_idx} F={F}: {dt*1e3:.1f} ms ({F/dt:.0f} frames/s); status counts {dict(zip(vals.tolist(), cnts.tolist()))}")
    print("   lp/frame %.2f ipm/frame %.1f pcg/frame %.0f pcg/ipm %.1f max_p mean %.0f; cert %d/%d" % (
        st["lp_solves"].mean(), st["ipm_iters"].mean(), st["pcg_iters"].mean(),
        st["pcg_iters"].sum() / max(1, st["ipm_iters"].sum()), st["max_p"].mean(), int(res.certificate.sum()), F))
    hard = res.hard.cpu().numpy()
    print("   frame errors vs tx:", int(np.any(hard != fb.codewords, axis=1).sum()))
    cyc = {k: float(st[k].sum()) for k in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other")}
    tot = sum(cyc.values())
    print("   phase shares:", {k: round(v / tot, 3) for k, v in cyc.items()},
          "cycles/PCG-iter %.0f (spmv %.0f sweep %.0f other %.0f)" % (
              (cyc["cyc_spmv"] + cyc["cyc_sweep"] + cyc["cyc_pcg_other"]) / st["pcg_iters"].sum(),
              cyc["cyc_spmv"] / st["pcg_iters"].sum(), cyc["cyc_sweep"] / st["pcg_iters"].sum(),
              cyc["cyc_pcg_other"] / st["pcg_iters"].sum()),
          "build cycles/IPM-iter %.0f" % (cyc["cyc_build"] / st["ipm_iters"].sum()))
    lat = np.argsort(-st["pcg_iters"])[:5]
    print("   slowest frames (pcg its):", [(int(f), int(st["pcg_iters"][f]), int(st["lp_solves"][f]), int(st["ipm_iters"][f]), int(status[f])) for f in lat])
    from oracle.lp import params_with
    obj = res.objective.cpu().numpy()
    worst = 0.0
    for f in range(8):
        o = malp_decode(code, fb.llr[f], params=params_with(gap_tol=GAP))
        worst = max(worst, abs(obj[f] - o["obj"]) / max(1.0, abs(o["obj"])))
        print("   frame %d gpu obj %.9f oracle %.9f | lp %d/%d ipm %d/%d status %d" % (
            f, obj[f], o["obj"], st["lp_solves"][f], o["lp_solves"], st["ipm_iters"][f], o["ipm_iters"], status[f]))
    print("   worst rel obj diff (8 frames): %.2e" % worst)


if __name__ == "__main__":
    if os.environ.get("MAIN", "1") == "1":
        main()
    c2_sample()
    c2_sample(F=2048, snr_idx=2)
    c2_sample(F=256, snr_idx=0, cfg=3)
