"""Binary symmetric channel frames with LLR jitter (SURVEY f-4; §III-B).

The BSC has discrete outputs, so intermediate MALP LPs can have non-unique optima (the
uniqueness assumption of P:258-261 fails; reading C-12's cycles).  The paper's remedy is "adding
a very small continuous-domain noise to their output (or LLR vector)": here
gamma_i = (1 - 2 y_i) log((1 - p)/p) + U(-jitter, +jitter) for the received bit y_i
(eq.`def gamma` P:97-101 for the BSC).  Input generation only: no decoding arithmetic.
Per-frame stream default_rng([frame_seed, 7, frame]) draws the info bits (random codewords),
then the crossover pattern, then the jitter.
"""
from __future__ import annotations

import numpy as np

from .codes import Code
from .frames import FrameBatch, _encoder


def bsc_llr(bits: np.ndarray, p: float, jitter: np.ndarray | float = 0.0) -> np.ndarray:
    """gamma = +-log((1-p)/p) by received bit (0 -> +), plus the given jitter."""
    if not (0.0 < p < 0.5):
        raise ValueError("crossover must lie in (0, 1/2)")
    L = float(np.log((1.0 - p) / p))
    return (1.0 - 2.0 * np.asarray(bits, dtype=np.float64)) * L + jitter


def bsc_frames(code: Code, p: float, jitter: float, frame_seed: int, frames,
               random_codeword: bool = True) -> FrameBatch:
    frames = np.asarray(list(frames) if not isinstance(frames, np.ndarray) else frames, dtype=np.int64)
    n = code.n
    F = frames.size
    enc = _encoder(code) if random_codeword else None
    info = np.empty((F, enc.k), dtype=np.uint8) if random_codeword else None
    flips = np.empty((F, n), dtype=np.uint8)
    jit = np.empty((F, n))
    for t, f in enumerate(frames):
        rng = np.random.default_rng([frame_seed, 7, int(f)])
        if random_codeword:
            info[t] = rng.integers(0, 2, enc.k)
        flips[t] = (rng.random(n) < p).astype(np.uint8)
        jit[t] = rng.uniform(-jitter, jitter, n) if jitter > 0 else 0.0
    cw = enc.encode(info) if random_codeword else np.zeros((F, n), dtype=np.uint8)
    y = cw ^ flips
    llr = bsc_llr(y, p, jit)
    return FrameBatch(code, float("nan"), float("nan"), frames, cw, llr)
