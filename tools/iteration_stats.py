"""SURVEY f-3, the paper's §III-D experiment (E1/E2; Figs. 1-2 are missing): MALP-A
and MALP-B outer-iteration (LP) counts of random (3,6)-regular codes with 4-cycles removed
(reading C-21 option), AWGN at 2 dB, 1000 all-zero-codeword trials per length, decoded on the
GPU (alp_decode), split by integral (certified) / fractional outputs.
E1: the histograms at n = 480.  E2: mean, 95th percentile and the 95 % one-sided upper
confidence bound of the mean (mean + 1.645 s/sqrt(N)) versus n over 8 lengths.
Output: gpurun_out/iteration_stats.json (committed under profiles/)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_0902_0657_b200 as alp
from synth import awgn_frames
from synth.codes import regular_code

TRIALS = int(os.environ.get("TRIALS", "1000"))
LENGTHS = [int(v) for v in os.environ.get("LENGTHS", "120,240,360,480,720,960,1440,1920").split(",")]
SNR = float(os.environ.get("SNR", "2.0"))


def summary(x):
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        return None
    return dict(n=int(x.size), mean=float(x.mean()), p95=float(np.percentile(x, 95)),
                mean_ucb95=float(x.mean() + 1.645 * x.std(ddof=1) / np.sqrt(x.size)) if x.size > 1 else float(x.mean()),
                max=int(x.max()), hist={int(k): int(v) for k, v in zip(*np.unique(x.astype(int), return_counts=True))})


out = dict(snr_db=SNR, trials=TRIALS, code="random (3,6)-regular, 4-cycles removed, seed 3000+n",
           channel="all-zero codeword, BPSK/AWGN", lengths={})
for n in LENGTHS:
    code = regular_code(n, 3, 6, seed=3000 + n, girth6=True)
    c = alp.Code.from_synth(code)
    fb = awgn_frames(code, SNR, 4000 + n, 0, range(TRIALS), random_codeword=False)
    llr = torch.from_numpy(fb.llr).cuda()
    row = {}
    for name, variant in (("MALP-A", 0), ("MALP-B", 1)):
        t = time.time()
        res = alp.decode(c, llr, alp.default_params(variant=variant))
        torch.cuda.synchronize()
        st = res.stats_numpy()
        cert = res.certificate.cpu().numpy() == 1
        status = res.status.cpu().numpy()
        fin = (status & (1 | 2 | 16)) == 0
        lps = st["lp_solves"]
        row[name] = dict(integral=summary(lps[cert & fin]), fractional=summary(lps[~cert & fin]),
                         unfinished=int((~fin).sum()), max_p=summary(st["max_p"][fin]),
                         seconds=time.time() - t)
        print(n, name, "integral", row[name]["integral"] and {k: row[name]["integral"][k] for k in ("mean", "p95", "max")},
              "fractional", row[name]["fractional"] and {k: row[name]["fractional"][k] for k in ("mean", "p95", "max")},
              "unfinished", row[name]["unfinished"], flush=True)
    out["lengths"][n] = row
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/iteration_stats.json", "w"), indent=1)
