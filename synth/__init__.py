"""Seeded synthetic inputs shared by the oracle, the tests and the benchmark.

This package holds INPUT generation only (codes, codewords, channel noise,
isolated step-solve systems).  It contains none of the decoding method's
arithmetic: no cut search, no LP, no interior point, no preconditioner.
Both `oracle/` and the CUDA path consume what it produces; neither imports
the other.

Recipes follow SURVEY.md §8(d) d.1 and are restated in DESIGN.md §4.
"""
from .codes import Code, regular_code, code_from_rows, CONFIG_CODES, config_code
from .frames import (sigma2_for, awgn_frames, FrameBatch, CONFIGS, config_frames,
                     GF2Encoder)
from .systems import StepSystems, c5_systems, odd_masks
from .bsc import bsc_llr, bsc_frames

__all__ = [
    "Code", "regular_code", "code_from_rows", "CONFIG_CODES", "config_code",
    "sigma2_for", "awgn_frames", "FrameBatch", "CONFIGS", "config_frames",
    "GF2Encoder", "StepSystems", "c5_systems", "odd_masks", "bsc_llr", "bsc_frames",
]
