"""Benchmark of the batched ALP decoder (libalp.so) — the driver's bench contract.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: launched by torch.distributed.run, one rank per GPU)

Workload = BASELINE.json configs[1] ("C2"): random (3,6)-regular LDPC code n=1000, m=500,
16,384 frames per rank of random codewords, BPSK/AWGN at Eb/N0 = 3.0 dB (--snr-idx 0/1 picks
2.0 / 2.5 dB; at 2.0 dB a fraction of frames ends on the IPM/PCG caps), fp64
LLR costs.  One STEP = one alp_decode
call over the whole batch: MALP-A cut search, every LP solved by the primal-dual IPM, every
Newton step by PCG with the column-wise triangular preconditioner.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the
launching stream; between timed steps a 256 MiB buffer is written to flush L2 (outside the
events).  Inputs (131 MB of LLRs) are device-resident for `value`; `e2e` repeats the step
through alp_decode_host from pinned host memory (H2D + D2H inside the timed region).
Frames shard across ranks (frame f -> rank f mod N, no data-path collective; counters are
all-reduced once at the end), so `scaling` is "weak" (16,384 frames per GPU).

The oracle (oracle/, fp64 numpy, dense Cholesky step solve) is timed on the host cores on
a bounded sample (cpu_baseline; and `--impl reference`).  It is never on the product path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np

METRIC = "LP-decoded frames/sec, (3,6) LDPC n=1000; PCG HBM GB/s vs ~8 TB/s peak"
UNIT = "frames/s"
FRAMES_PER_RANK = 16384
SNRS = [2.0, 2.5, 3.0]


CONFIG_DESC = {
    1: ("C1: random (3,6)-regular LDPC n=120 m=60", "rnd(3,6) n=120 m=60 seed 1001", [3.0], "all-zero codeword"),
    2: ("C2: random (3,6)-regular LDPC n=1000 m=500", "rnd(3,6) n=1000 m=500 seed 1002", [2.0, 2.5, 3.0],
        "random-codeword"),
    3: ("C3: random (3,12)-regular LDPC n=4000 m=1000", "rnd(3,12) n=4000 m=1000 seed 1003", [3.5], "all-zero codeword"),
    4: ("C4: random (3,6)-regular LDPC n=32000 m=16000", "rnd(3,6) n=32000 m=16000 seed 1004", [2.2],
        "random-codeword"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4],
                    help="BASELINE.json config of the decode workload (2 = the metric's; 1/3/4 = the "
                         "other decode configs, e.g. --config 4 --frames 1184 for the n=32,000 line)")
    ap.add_argument("--snr-idx", type=int, default=None, help="Eb/N0 index (config 2: 0/1/2 = 2.0/2.5/3.0 dB)")
    ap.add_argument("--frames", type=int, default=FRAMES_PER_RANK, help="frames per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle sample budget")
    ap.add_argument("--snr-sweep", type=int, default=1,
                    help="also decode the config's other SNRs (2.0, 2.5 dB) once each and report them")
    ap.add_argument("--step-systems", type=int, default=65536,
                    help="config-5 isolated step solves timed beside the decode (0 = skip)")
    a = ap.parse_args()
    if a.snr_idx is None:
        a.snr_idx = 2 if a.config == 2 else 0
    a.snrs = CONFIG_DESC[a.config][2]
    if a.config != 2:
        a.snr_sweep = 0
    return a


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_config(args, ws):
    desc, code_desc, snrs, kind = CONFIG_DESC[args.config]
    return {
        "workload": f"{desc}, {args.frames} {kind} "
                    f"frames per GPU, BPSK/AWGN Eb/N0={snrs[args.snr_idx]} dB, fp64 LLR, MALP-A + "
                    "primal-dual IPM + PCG (column-wise MTS preconditioner) to recursive rel. "
                    "residual 1e-8 (forcing term min(1e-8, 1e-2 mu)) with the basis-corrected "
                    "Newton recovery (DESIGN.md C-32)",
        "code": code_desc,
        "frames_per_gpu": args.frames,
        "global_frames": args.frames * ws,
        "ebn0_db": snrs[args.snr_idx],
        "parallelism": f"frame-sharded dp{ws}",
        "l2": "256 MiB L2 flush between timed steps (LLR input 131 MB also exceeds L2)",
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- oracle arm
def _oracle_worker(args_tuple):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)   # one BLAS thread per worker process
    cfg, snr_idx, frames = args_tuple
    from synth import config_code, config_frames
    from oracle.lp import malp_decode
    code = config_code(cfg)
    fb = config_frames(cfg, snr_idx, frames=frames, code=code)
    t0 = time.perf_counter()
    for f in range(fb.F):
        malp_decode(code, fb.llr[f])
    return fb.F, time.perf_counter() - t0


def time_oracle(snr_idx: int, budget_s: float, frame_offset: int = 0, cfg: int = 2):
    """Oracle MALP-A decode (fp64, dense Cholesky) on the host cores: one frame per worker
    process, frames taken in order from frame_offset, workers run until budget_s elapses.
    Returns (frames/s, cores, frames decoded)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    per = 2
    t0 = time.perf_counter()
    done, nxt = 0, frame_offset
    ctx = mp.get_context("fork")
    env_threads = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_threads:
        os.environ[k] = "1"
    try:
        with ctx.Pool(cores) as pool:
            while True:
                jobs = [(cfg, snr_idx, list(range(nxt + w * per, nxt + (w + 1) * per))) for w in range(cores)]
                nxt += cores * per
                for F, _ in pool.map(_oracle_worker, jobs):
                    done += F
                if time.perf_counter() - t0 >= budget_s:
                    break
    finally:
        for k, v in env_threads.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    wall = time.perf_counter() - t0
    return done / wall, cores, done, wall


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    times, frames = [], 0
    budget = max(2.0, min(args.cpu_seconds, 60.0))
    for s in range(args.warmup + args.steps):
        fps, cores, nf, wall = time_oracle(args.snr_idx, budget / 2, frame_offset=0, cfg=args.config)
        if s >= args.warmup:
            times.append(wall)
            frames += nf
    v = frames / sum(times)
    sample = (f"MALP-A oracle (fp64 numpy, dense Cholesky step solve) on the first frames of the "
              f"config, {cores} worker processes x 1 BLAS thread, ~{budget / 2:.0f} s per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, ws),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device (no CPU fallback)"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_0902_0657_b200 as alp
    from paper_0902_0657_b200.dist import shard_frame_ids, frame_counters, reduce_run, counters_dict
    from synth import config_code, config_frames

    code = config_code(args.config)
    # this rank's frames: global frame g = rank + ws * t (interleaved sharding)
    frame_ids = shard_frame_ids(args.frames, rank, ws)
    fb = config_frames(args.config, args.snr_idx, frames=frame_ids, code=code)
    llr_host = torch.from_numpy(fb.llr).pin_memory()
    llr = llr_host.to(dev)
    c = alp.Code.from_synth(code)
    stream = torch.cuda.current_stream(dev)
    F = args.frames

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = alp.decode(c, llr, stream=stream)      # allocates outputs + workspace once
    torch.cuda.synchronize(dev)

    def step():
        alp.decode(c, llr, stream=stream, out=out)
        return alp.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    launches = 0
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        ev[k][0].record(stream)
        launches += step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if ws > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    t_rank = sum(ms) / 1e3

    # per-frame counters of the last step (identical every step: deterministic decode)
    st = out.stats_numpy()
    counters = frame_counters(out.hard.cpu().numpy(), fb.codewords, out.certificate.cpu().numpy(),
                              out.status.cpu().numpy(), st)
    pcg_bytes = float(counters[7])

    # e2e through the host API (pinned host LLRs in, host outputs back, inside the timing)
    e2e_t = 0.0
    if not args.no_e2e:
        hout = dict(hard=torch.empty((F, code.n), dtype=torch.uint8, pin_memory=True),
                    objective=torch.empty(F, dtype=torch.float64, pin_memory=True),
                    certificate=torch.empty(F, dtype=torch.uint8, pin_memory=True),
                    status=torch.empty(F, dtype=torch.int32, pin_memory=True))
        alp.decode_host(c, llr_host, stream=stream, out=hout)
        torch.cuda.synchronize(dev)
        e2e_ms = []
        for k in range(args.steps):
            flush.fill_(k & 0xff)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            alp.decode_host(c, llr_host, stream=stream, out=hout)   # synchronises internally
            b.record(stream)
            torch.cuda.synchronize(dev)
            e2e_ms.append(a.elapsed_time(b))
        e2e_t = sum(e2e_ms) / 1e3
        h2d = F * code.n * 8
        d2h = F * code.n + F * 8 + F + F * 4
    allc, t_max = reduce_run(counters, t_rank, device=dev)
    _, e2e_max = reduce_run(counters[:1], e2e_t, device=dev)
    counters, pcg_bytes_all = allc, float(allc[7])

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    total_frames = F * ws * args.steps
    value = total_frames / t_max
    peak, peak_kind = measured_peak_hbm()
    # dominant (only) kernel: alp_decode_kernel, one launch per step on `stream`
    achieved = pcg_bytes / (t_rank / args.steps) / 1e9
    traffic, traffic_src = None, None
    try:   # DRAM bytes per frame from the committed ncu --set full capture (C2), scaled to this launch
        if args.config != 2:
            raise OSError("no capture for this config")
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tj = json.load(fh)
        traffic = float(tj["dram_bytes_per_frame"]) * F
        traffic_src = f"{tj['capture']}: {tj['frames']} frames, scaled per frame to {F}"
    except (OSError, KeyError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, ws),
        "gpu_launches": launches,
        "launch": alp.launch_info(c, F),
        "clocks": clk,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": pcg_bytes,
                     "kernel": "alp_decode_kernel",
                     "bytes": "sum over executed PCG iterations of B_min(p,n_act,m) (DESIGN.md §6)",
                     "peak_kind": peak_kind},
        "pcg_phase": pcg_phase(st, pcg_bytes, t_rank / args.steps),
        "pcg": {"iters_per_s": counters[5] / (t_max / args.steps),
                "iters_total_per_step": int(counters[5]),
                "gbs_all_ranks": pcg_bytes_all / (t_max / args.steps) / 1e9},
        "decode": counters_dict(counters),
        "step_ms": ms,
    }
    if not args.no_e2e:
        line["e2e"] = {"value": total_frames / e2e_max, "unit": UNIT,
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if args.snr_sweep and ws == 1:
        line["snr_sweep"] = {}
        for si in range(len(SNRS)):
            if si == args.snr_idx:
                continue
            fbs = config_frames(2, si, frames=frame_ids, code=code)
            llr_s = torch.from_numpy(fbs.llr).to(dev)
            alp.decode(c, llr_s, stream=stream, out=out)     # warm-up (same shapes)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(7)
            a.record(stream)
            alp.decode(c, llr_s, stream=stream, out=out)
            b.record(stream)
            torch.cuda.synchronize(dev)
            cs = frame_counters(out.hard.cpu().numpy(), fbs.codewords, out.certificate.cpu().numpy(),
                                out.status.cpu().numpy(), out.stats_numpy())
            line["snr_sweep"][f"{SNRS[si]} dB"] = dict(frames_per_s=F / (a.elapsed_time(b) / 1e3),
                                                      **counters_dict(cs))
    if args.step_systems > 0:
        line["step_solve"] = time_step_solve(args, dev, stream)
    if ws == 1 and not args.no_cpu_baseline and args.config != 4:
        fps, cores, nf, wall = time_oracle(args.snr_idx, args.cpu_seconds, cfg=args.config)
        line["cpu_baseline"] = {
            "value": fps, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {nf} frames of the same workload, MALP-A oracle (fp64 numpy, dense "
                      f"Cholesky), {cores} worker processes x 1 BLAS thread, {wall:.1f} s"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def pcg_phase(st, pcg_bytes, t_launch):
    """Share of the decode kernel's warp-cycles spent in the PCG loop (SpMV, sweeps, vector
    updates; alp_frame_stats.cyc_*) and the algorithmic PCG bytes per second of PCG-phase time
    (the kernel time scaled by that share)."""
    keys = ("cyc_cut", "cyc_ipm", "cyc_build", "cyc_spmv", "cyc_sweep", "cyc_pcg_other")
    tot = {k: float(st[k].sum()) for k in keys}
    allc = sum(tot.values())
    pcgc = tot["cyc_spmv"] + tot["cyc_sweep"] + tot["cyc_pcg_other"]
    share = pcgc / allc if allc > 0 else 0.0
    return {"share_of_warp_cycles": share,
            "shares": {k: v / allc for k, v in tot.items()} if allc > 0 else {},
            "algorithmic_gbs_in_pcg_phase": pcg_bytes / (t_launch * share) / 1e9 if share > 0 else None}


def time_step_solve(args, dev, stream):
    """BASELINE.json configs[4]: ipm_step_pcg on config-5 systems (n=2000 (3,6) code, one random
    odd cut per check, d log-uniform over 12 decades, r ~ N(0,1)), device-resident, timed with
    CUDA events over `steps` calls after `warmup` calls.  Algorithmic bytes per PCG iteration
    B_min(p=1000, n_act=2000, m=1000) = 79,000 B."""
    import torch
    import paper_0902_0657_b200 as alp
    from synth import config_code, c5_systems
    code = config_code(5)
    S = args.step_systems
    sy = c5_systems(range(S), code)
    c = alp.Code.from_synth(code)
    masks = torch.from_numpy(sy.masks.view(np.int16)).to(dev)
    d = torch.from_numpy(sy.d).to(dev)
    r = torch.from_numpy(sy.r).to(dev)
    res = None
    for _ in range(max(1, args.warmup)):
        res = alp.ipm_step_pcg(c, masks, d, r, stream=stream)
    torch.cuda.synchronize(dev)
    ms = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        res = alp.ipm_step_pcg(c, masks, d, r, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms.append(a.elapsed_time(b))
    t = sum(ms) / len(ms) / 1e3
    its = int(res.iters.sum().item())
    st = res.status.cpu().numpy()
    bmin = 8.0 * (code.n + code.m) + 48.0 * code.m + 5.0 * code.m + 2.0 * code.m
    peak, kind = measured_peak_hbm()
    gbs = its * bmin / t / 1e9
    return {"workload": f"C5: {S} systems A D^2 A^T dy = r, (3,6) n=2000 m=1000, d = 10^U(-6,6), "
                        "column-wise MTS PCG to recursive rel. residual 1e-8, then refined until the "
                        "TRUE residual meets 1e-8 or the fp64 evaluation floor (PCG_FLOOR)",
            "systems_per_s": S / t, "ms_per_call": 1e3 * t, "pcg_iters_per_s": its / t,
            "mean_pcg_iters": its / S, "status_counts": {int(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))},
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "bytes": "PCG iterations x B_min(1000, 2000, 1000) = 79 KB", "peak_kind": kind}}


def maybe_launch_ranks(args):
    """`--gpus N` (N > 1) without a torch.distributed environment: launch the N ranks here
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1) and return their exit
    code; under torchrun check that WORLD_SIZE matches --gpus."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if args.gpus > 1 and int(ws_env) != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws_env}")
        return None
    if args.gpus <= 1:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    rc = maybe_launch_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
