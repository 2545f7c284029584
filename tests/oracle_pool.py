"""Runs the oracle (test infrastructure) over many frames / systems in a process pool.

Spawned worker processes import only `oracle/` and `synth/` (never the product, never CUDA),
one BLAS thread each, so the SURVEY §8(c) c.5 sample sizes (C1 all frames, C2 256 per SNR,
C3 128, C5 1024 systems) finish in about a minute on the GPU box's host cores.
"""
from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_KEEP = ("u", "hard", "obj", "g_max", "cert", "status", "lp_solves", "ipm_iters", "max_p",
         "masks", "y", "chol_fixes")


def _init():
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _decode_job(job):
    cfg, snr_idx, frames, variant, llr_scale, library = job
    from synth import config_code, config_frames
    if library:     # Alg. 3 with the LP step by HiGHS (oracle/lp_library.py): never ends on an IPM cap
        from oracle.lp_library import malp_decode_library as malp_decode
    else:
        from oracle.lp import malp_decode
    code = config_code(cfg)
    fb = config_frames(cfg, snr_idx, frames=frames, code=code) if cfg == 2 else \
        config_frames(cfg, frames=frames, code=code)
    out = []
    for f in range(fb.F):
        o = malp_decode(code, fb.llr[f] * llr_scale, variant)
        out.append({k: o[k] for k in _KEEP})
    return out


def _exact_job(job):
    idx, lo, hi = job
    from synth import config_code, c5_systems
    from oracle.lp import step_solve_exact
    from oracle.precond import mts_columnwise
    from tests.helpers import dense_step_matrix, step_weights
    code = config_code(5)
    sy = c5_systems(idx, code, lo=lo, hi=hi)
    out = []
    for s in range(sy.S):
        A, rows = dense_step_matrix(code, sy.masks[s])
        w2 = step_weights(code, sy.d[s], rows)
        col, row = mts_columnwise(A, w2)
        out.append((step_solve_exact(A, w2, sy.r[s][rows]), col, row))
    return out


def _pool(n_jobs):
    workers = max(1, min(os.cpu_count() or 1, n_jobs))
    return ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn"),
                               initializer=_init)


def oracle_decode(cfg: int, frames, snr_idx: int = 0, variant: str = "A", llr_scale: float = 1.0,
                  chunk: int = 2, library: bool = False) -> list:
    """malp_decode (library=True: malp_decode_library) on config `cfg` frames (same seeded inputs
    as the GPU tests), in order."""
    frames = list(frames)
    jobs = [(cfg, snr_idx, frames[i:i + chunk], variant, llr_scale, library)
            for i in range(0, len(frames), chunk)]
    with _pool(len(jobs)) as ex:
        return [o for part in ex.map(_decode_job, jobs) for o in part]


def oracle_step_exact(systems, lo: float = -6, hi: float = 6, chunk: int = 2) -> list:
    """step_solve_exact (extended-precision Cholesky + refinement) and the Alg. 7 heap pivot
    sequence on config-5 systems: list of (dy, pivot cols, pivot rows)."""
    systems = list(systems)
    jobs = [(systems[i:i + chunk], lo, hi) for i in range(0, len(systems), chunk)]
    with _pool(len(jobs)) as ex:
        return [y for part in ex.map(_exact_job, jobs) for y in part]
