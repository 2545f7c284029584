"""Per-frame decode cost on C2 vs cheap difficulty predictors, and what frame ORDER does to the
persistent kernel's tail: list-scheduling simulation of the measured per-frame cycles on the
launch's concurrent frame slots (in-order vs sorted by a predictor vs ideal LPT).  Writes
gpurun_out/sched_<snr>.npz with the per-frame arrays."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import heapq
import numpy as np
import torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames

F = int(os.environ.get("F", "16384"))
code = config_code(2)
c = alp.Code.from_synth(code)
H = np.zeros((code.m, code.n), dtype=np.int32)
for j in range(code.m):
    H[j, code.N(j)] = 1


def makespan(cost, order, slots):
    h = [0.0] * slots
    for f in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + cost[f])
    return max(h)


for si in [int(v) for v in os.environ.get("SNRS", "0,1,2").split(",")]:
    fb = config_frames(2, si, frames=range(F))
    llr = torch.from_numpy(fb.llr).cuda()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    res = alp.decode(c, llr)
    b.record()
    torch.cuda.synchronize()
    st = res.stats_numpy()
    cyc = sum(st[k].astype(np.float64) for k in ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other"))
    hard = (fb.llr < 0).astype(np.int32)
    synd = ((hard @ H.T) & 1).sum(axis=1)
    weak = (np.abs(fb.llr) < 1.0).sum(axis=1)
    np.savez_compressed(f"gpurun_out/sched_{si}.npz", cyc=cyc, synd=synd, weak=weak,
                        pcg=st["pcg_iters"], status=res.status.cpu().numpy())
    info = alp.launch_info(c, F)
    slots = int(os.environ.get("SLOTS", "740"))
    ms = a.elapsed_time(b)
    base = makespan(cyc, range(F), slots)
    out = dict(snr=si, ms=ms, slots=slots, launch=str(info), in_order=1.0,
               sorted_synd=makespan(cyc, np.argsort(-synd, kind="stable"), slots) / base,
               sorted_weak=makespan(cyc, np.argsort(-weak, kind="stable"), slots) / base,
               lpt_ideal=makespan(cyc, np.argsort(-cyc, kind="stable"), slots) / base,
               mean_bound=cyc.sum() / slots / base,
               corr_synd=float(np.corrcoef(synd, np.log(cyc))[0, 1]),
               corr_weak=float(np.corrcoef(weak, np.log(cyc))[0, 1]))
    print(json.dumps(out), flush=True)
