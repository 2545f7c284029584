"""Peel diagnostics on C2 (3.0 dB): libalp_split.so puts the Alg. 7 initialisation cycles into
cyc_cut (with the cut search's own), libalp_count.so the batch / pick counts of the batched peel
(in the sort / peel clocks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_0902_0657_b200 as alp
from synth import config_code, config_frames
F = int(os.environ.get("F", "2048"))
snr = int(os.environ.get("SNR", "2"))
code = config_code(2)
fb = config_frames(2, snr, frames=range(F))
c = alp.Code.from_synth(code)
res = alp.decode(c, torch.from_numpy(fb.llr).cuda())
torch.cuda.synchronize()
st = res.stats_numpy()
ipm = st["ipm_iters"].sum()
cut = st["cyc_cut"].astype(np.int64)
lib = os.environ.get("ALP_LIB", "")
if "count" in lib:
    nb = st["cyc_sort"].sum(); picks = st["cyc_peel"].sum()
    print(lib, "batches/IPM it %.1f picks/IPM it %.1f picks per batch %.3f" % (nb / ipm, picks / ipm, picks / nb))
else:
    print(lib, "per IPM it: peel %.0f (init %.0f) sort %.0f cyc" % (st["cyc_peel"].sum() / ipm, cut.sum() / ipm, st["cyc_sort"].sum() / ipm))
