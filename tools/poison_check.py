"""Uninitialised-state check (stands in for compute-sanitizer initcheck, closed on this pool).

Runs the same decodes / step solves with the normal library and with the -DALP_POISON build
(libalp_poison.so: every frame's shared window and global slot are filled with NaN patterns
before the frame starts), each in its own process, plus a permuted-frame-order run of the normal
build, and requires every output to be bit-identical: a read of anything a frame did not write
first would change it.  Workloads: C1 all 100 frames (MALP-A and MALP-B), C2 128 frames at 2.0 dB,
C3 32 frames (generic window mode), C1 and C5 step systems.
  python tools/poison_check.py            (driver; needs paper_0902_0657_b200/libalp_poison.so)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np


def run(out_path, permute):
    import torch
    import paper_0902_0657_b200 as alp
    from synth import config_code, config_frames, c5_systems
    res = {}
    jobs = [("c1A", 1, None, dict(variant=0)), ("c1B", 1, None, dict(variant=1)),
            ("c2_2dB", 2, 0, {}), ("c3", 3, None, {})]
    for name, cfg, si, prm in jobs:
        code = config_code(cfg)
        F = {1: 100, 2: 128, 3: 32}[cfg]
        fb = config_frames(cfg, si, frames=range(F)) if si is not None else config_frames(cfg, frames=range(F))
        order = np.random.default_rng(5).permutation(F) if permute else np.arange(F)
        c = alp.Code.from_synth(code)
        r = alp.decode(c, torch.from_numpy(np.ascontiguousarray(fb.llr[order])).cuda(), alp.default_params(**prm),
                       want_u=True, want_y=True, want_masks=True)
        torch.cuda.synchronize()
        inv = np.argsort(order)
        for k, v in dict(hard=r.hard, obj=r.objective, cert=r.certificate, status=r.status, u=r.u, y=r.y,
                         masks=r.masks).items():
            res[f"{name}.{k}"] = v.cpu().numpy()[inv]
        st = r.stats_numpy()
        for k in ("lp_solves", "ipm_iters", "pcg_iters"):
            res[f"{name}.{k}"] = st[k][inv]
    for name, cfg, S in (("step_c1", 1, 64), ("step_c5", 5, 64)):
        code = config_code(cfg)
        sy = c5_systems(range(S), code, lo=-3, hi=3) if cfg == 1 else c5_systems(range(S), code)
        order = np.random.default_rng(6).permutation(S) if permute else np.arange(S)
        c = alp.Code.from_synth(code)
        st = alp.ipm_step_pcg(c, torch.from_numpy(np.ascontiguousarray(sy.masks[order]).view(np.int16)).cuda(),
                              torch.from_numpy(np.ascontiguousarray(sy.d[order])).cuda(),
                              torch.from_numpy(np.ascontiguousarray(sy.r[order])).cuda())
        torch.cuda.synchronize()
        inv = np.argsort(order)
        for k, v in dict(dy=st.dy, iters=st.iters, status=st.status, relres=st.relres).items():
            res[f"{name}.{k}"] = v.cpu().numpy()[inv]
    np.savez(out_path, **res)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--run":
        run(sys.argv[2], sys.argv[3] == "1")
        return 0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    outs = {}
    for tag, lib, perm in (("normal", None, "0"), ("poison", "libalp_poison.so", "0"), ("permuted", None, "1")):
        env = dict(os.environ)
        if lib:
            env["ALP_LIB"] = os.path.join(ROOT, "paper_0902_0657_b200", lib)
        path = os.path.join(ROOT, "gpurun_out", f"poison_{tag}.npz")
        subprocess.run([sys.executable, __file__, "--run", path, perm], check=True, env=env)
        outs[tag] = dict(np.load(path))
    bad = []
    for tag in ("poison", "permuted"):
        for k, v in outs["normal"].items():
            w = outs[tag][k]
            same = np.array_equal(v.view(np.uint8), w.view(np.uint8)) if v.dtype.kind == "f" else np.array_equal(v, w)
            if not same:
                bad.append((tag, k))
    n = len(outs["normal"])
    print(f"poison / permutation check: {n} output arrays x 2 comparisons, {len(bad)} differ", bad[:20])
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
