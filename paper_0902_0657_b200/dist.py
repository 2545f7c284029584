"""Frame sharding across ranks.

Frames are independent LP-decoding problems, so the multi-GPU path has no data-path
collective: global frame g belongs to rank g mod world_size (interleaved, which spreads
the rare hard — fractional — frames evenly), each rank regenerates its own frames from
the per-frame-keyed RNG, decodes them with one alp_decode call, and the run ends with
one SUM all-reduce of the integer counters and one MAX all-reduce of the timed duration.
Works on any torch.distributed backend (nccl on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

# order of the counter vector reduced at the end of a run
STATUS_BITS = {"alp_maxiter": 1, "ipm_maxiter": 2, "pcg_maxiter": 4, "pcg_breakdown": 8, "numeric": 16}
COUNTERS = ("frames", "frame_errors", "not_certified", "lp_solves", "ipm_iters", "pcg_iters",
            "frames_capped", "pcg_bytes", "pcg_solves", "pcg_p4_failed_solves",
            "pcg_true_failed_solves") + tuple("frames_" + k for k in STATUS_BITS)
CAP_BITS = 1 | 2 | 16


def shard_frame_ids(frames_per_rank: int, rank: int, world_size: int) -> np.ndarray:
    """Global frame ids owned by `rank` when every rank decodes frames_per_rank frames."""
    if not (0 <= rank < world_size):
        raise ValueError("rank out of range")
    return np.arange(frames_per_rank, dtype=np.int64) * world_size + rank


def frame_counters(hard, codewords, certificate, status, stats) -> np.ndarray:
    """Per-rank counter vector (COUNTERS order) from one decode's host-side outputs.
    frames_capped = frames whose decode ended on a cap / cycle / non-finite status; the
    frames_<bit> entries count the frames carrying each alp_frame_status bit."""
    hard = np.asarray(hard)
    status = np.asarray(status)
    errs = int(np.any(hard != np.asarray(codewords), axis=1).sum())
    bits = [int(((status & b) != 0).sum()) for b in STATUS_BITS.values()]
    return np.array([hard.shape[0], errs, int((np.asarray(certificate) == 0).sum()),
                     int(stats["lp_solves"].sum()), int(stats["ipm_iters"].sum()),
                     int(stats["pcg_iters"].sum()), int(((status & CAP_BITS) != 0).sum()),
                     float(stats["pcg_bytes"].sum()), int(stats["pcg_solves"].sum()),
                     int(stats["pcg_p4_fail"].sum()), int(stats["pcg_true_fail"].sum())] + bits,
                    dtype=np.float64)


def counters_dict(c) -> dict:
    return {k: (float(v) if k == "pcg_bytes" else int(v)) for k, v in zip(COUNTERS, c)}


def reduce_run(counters: np.ndarray, seconds: float, device=None) -> tuple[np.ndarray, float]:
    """SUM of the counters and MAX of the timed duration over all ranks (identity when
    torch.distributed is not initialised)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return np.asarray(counters, dtype=np.float64), float(seconds)
    dev = device if device is not None else torch.device("cpu")
    c = torch.tensor(np.asarray(counters, dtype=np.float64), device=dev)
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return c.cpu().numpy(), float(t.item())
