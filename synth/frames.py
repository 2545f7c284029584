"""Received frames: random (or all-zero) codewords sent BPSK over AWGN.

Channel and LLR convention (PAPER.md eq.`def gamma`
l.97-101): bit 0 -> +1, y = (1 - 2c) + sigma * N(0,1), gamma = 2 y / sigma^2,
sigma^2 = 1 / (2 R 10^(EbN0/10)), R = 1 - m/n (design rate).

Every frame has its own RNG stream default_rng([frame_seed, snr_idx, frame])
so any shard (rank) can regenerate exactly its own frames.  For random
codewords the info bits are drawn first (k = n - rank(H)), then the noise.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

from .codes import Code, config_code


def sigma2_for(code: Code, ebn0_db: float) -> float:
    R = 1.0 - code.m / code.n
    return 1.0 / (2.0 * R * 10.0 ** (ebn0_db / 10.0))


class GF2Encoder:
    """Systematic encoder from a deterministic GF(2) reduced row-echelon form of H.

    Column pivoting takes the lowest-index column with a usable 1 (SURVEY.md
    d.1).  Pivot columns P are computed from the free columns F (info bits).
    """

    def __init__(self, code: Code):
        n, m = code.n, code.m
        W = (n + 63) // 64
        rows = np.zeros((m, W), dtype=np.uint64)
        for j in range(m):
            for i in code.N(j):
                rows[j, i >> 6] |= np.uint64(1) << np.uint64(i & 63)
        rank = 0
        pivots = []
        for c in range(n):
            if rank == m:
                break
            w, b = c >> 6, np.uint64(c & 63)
            col_bits = (rows[rank:, w] >> b) & np.uint64(1)
            nz = np.nonzero(col_bits)[0]
            if nz.size == 0:
                continue
            r = rank + int(nz[0])
            if r != rank:
                rows[[rank, r]] = rows[[r, rank]]
            has = ((rows[:, w] >> b) & np.uint64(1)).astype(bool)
            has[rank] = False
            rows[has] ^= rows[rank]
            pivots.append(c)
            rank += 1
        self.n, self.rank = n, rank
        self.pivots = np.array(pivots, dtype=np.int64)
        mask = np.ones(n, dtype=bool)
        mask[self.pivots] = False
        self.free = np.nonzero(mask)[0]
        self.k = n - rank
        # dense 0/1 matrix R[r, f] restricted to free columns (rank x k), as float32 for batched matmul
        Rf = np.zeros((rank, self.k), dtype=np.float32)
        for t, f in enumerate(self.free):
            Rf[:, t] = ((rows[:rank, f >> 6] >> np.uint64(f & 63)) & np.uint64(1)).astype(np.float32)
        self.Rf = Rf

    def encode(self, info: np.ndarray) -> np.ndarray:
        """info [F, k] 0/1 -> codewords [F, n] uint8."""
        info = np.atleast_2d(info).astype(np.float32)
        cw = np.zeros((info.shape[0], self.n), dtype=np.uint8)
        cw[:, self.free] = info.astype(np.uint8)
        par = (info @ self.Rf.T)  # exact: sums <= k < 2^24
        cw[:, self.pivots] = (np.rint(par).astype(np.int64) & 1).astype(np.uint8)
        return cw


@dataclass
class FrameBatch:
    code: Code
    ebn0_db: float
    sigma2: float
    frame_ids: np.ndarray      # global frame indices
    codewords: np.ndarray      # [F, n] uint8 transmitted
    llr: np.ndarray            # [F, n] float64 gamma

    @property
    def F(self) -> int:
        return int(self.llr.shape[0])


_ENC_CACHE: dict = {}


def _encoder(code: Code) -> GF2Encoder:
    key = (code.name, code.n, code.m, code.E, int(code.col_idx[:64].sum()))
    enc = _ENC_CACHE.get(key)
    if enc is None:
        enc = GF2Encoder(code)
        _ENC_CACHE[key] = enc
    return enc


def awgn_frames(code: Code, ebn0_db: float, frame_seed: int, snr_idx: int,
                frames, random_codeword: bool) -> FrameBatch:
    frames = np.asarray(list(frames) if not isinstance(frames, np.ndarray) else frames,
                        dtype=np.int64)
    n = code.n
    s2 = sigma2_for(code, ebn0_db)
    sig = np.sqrt(s2)
    F = frames.size
    noise = np.empty((F, n))
    info = None
    enc = _encoder(code) if random_codeword else None
    if random_codeword:
        info = np.empty((F, enc.k), dtype=np.uint8)
    for t, f in enumerate(frames):
        rng = np.random.default_rng([frame_seed, snr_idx, int(f)])
        if random_codeword:
            info[t] = rng.integers(0, 2, enc.k)
        noise[t] = rng.standard_normal(n)
    cw = enc.encode(info) if random_codeword else np.zeros((F, n), dtype=np.uint8)
    y = (1.0 - 2.0 * cw) + sig * noise
    llr = 2.0 * y / s2
    return FrameBatch(code, ebn0_db, s2, frames, cw, llr)


# BASELINE.json configs 1-4
CONFIGS = {
    1: dict(frame_seed=2001, snrs=[3.0], frames=100, random_codeword=False),
    2: dict(frame_seed=2002, snrs=[2.0, 2.5, 3.0], frames=16384, random_codeword=True),
    3: dict(frame_seed=2003, snrs=[3.5], frames=8192, random_codeword=False),
    4: dict(frame_seed=2004, snrs=[2.2], frames=4096, random_codeword=True),
}


def config_frames(cfg: int, snr_idx: int = 0, frames=None, code: Code | None = None) -> FrameBatch:
    p = CONFIGS[cfg]
    code = code or config_code(cfg)
    if frames is None:
        frames = range(p["frames"])
    return awgn_frames(code, p["snrs"][snr_idx], p["frame_seed"], snr_idx, frames,
                       p["random_codeword"])
