"""Thin Python binding of libalp.so (include/alp.h).

Argument marshalling only: torch supplies device memory and the stream; every step of
the decoder runs inside libalp's CUDA kernels.  There is no CPU fallback — if the
library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _ffi
from ._ffi import AlpParams, STATS_FIELDS, STATS_BYTES

STATUS_NAMES = {0: "ALP_OK", -1: "ALP_ERR_INVALID_ARG", -2: "ALP_ERR_BAD_CODE",
                -3: "ALP_ERR_UNSUPPORTED", -4: "ALP_ERR_CUDA", -5: "ALP_ERR_WORKSPACE"}
FRAME_ALP_MAXITER, FRAME_IPM_MAXITER, FRAME_PCG_MAXITER, FRAME_PCG_BREAKDOWN, FRAME_NUMERIC = 1, 2, 4, 8, 16
FRAME_PCG_FLOOR = 32   # informational (include/alp.h; ipm_step_pcg only)
STATS_DTYPE = np.dtype(STATS_FIELDS)


class AlpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    return _ffi.load()


def _check(st: int):
    if st != 0:
        raise AlpError(st, lib().alp_last_error().decode())


def default_params(**kw) -> AlpParams:
    p = AlpParams()
    lib().alp_default_params(C.byref(p))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    return p


def _sizing_error() -> AlpError:
    """Error of a *_workspace_bytes query that returned 0: the library's own failing status
    (e.g. ALP_ERR_UNSUPPORTED), never a generic one."""
    st = int(lib().alp_last_status())
    return AlpError(st if st != 0 else -1, lib().alp_last_error().decode())


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Code:
    """A parity-check matrix H (m x n) uploaded once to the device (alp_code)."""

    def __init__(self, n: int, m: int, row_ptr, col_idx):
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().alp_code_create(int(n), int(m), rp.ctypes.data, ci.ctypes.data, C.byref(h)))
        self.handle = h
        self.n, self.m = int(n), int(m)

    @classmethod
    def from_synth(cls, code) -> "Code":
        return cls(code.n, code.m, code.row_ptr, code.col_idx)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            lib().alp_code_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Workspace:
    """Caller-owned device scratch, grown on demand (torch allocations are 512 B aligned)."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws: dict = {}


def _ws(key, device) -> Workspace:
    w = _default_ws.get((key, str(device)))
    if w is None:
        w = Workspace(device)
        _default_ws[(key, str(device))] = w
    return w


@dataclass
class DecodeResult:
    hard: torch.Tensor        # [F, n] uint8
    objective: torch.Tensor   # [F] float64
    certificate: torch.Tensor  # [F] uint8
    status: torch.Tensor      # [F] int32
    stats: torch.Tensor       # [F, 128] uint8 (alp_frame_stats); see stats_numpy()
    u: torch.Tensor | None = None
    y: torch.Tensor | None = None
    masks: torch.Tensor | None = None

    def stats_numpy(self) -> np.ndarray:
        return self.stats.cpu().numpy().view(STATS_DTYPE).reshape(-1)


def decode(code: Code, llr: torch.Tensor, params: AlpParams | None = None, want_u=False,
           want_y=False, want_masks=False, stream=None, workspace: Workspace | None = None,
           out: DecodeResult | None = None) -> DecodeResult:
    """alp_decode on device-resident LLRs [F, n] (float64, CUDA)."""
    if llr.dtype != torch.float64 or not llr.is_cuda or llr.dim() != 2 or llr.shape[1] != code.n:
        raise ValueError("llr must be a CUDA float64 tensor of shape [F, n]")
    llr = llr.contiguous()
    F = llr.shape[0]
    dev = llr.device
    if out is None:
        out = DecodeResult(
            hard=torch.empty((F, code.n), dtype=torch.uint8, device=dev),
            objective=torch.empty(F, dtype=torch.float64, device=dev),
            certificate=torch.empty(F, dtype=torch.uint8, device=dev),
            status=torch.empty(F, dtype=torch.int32, device=dev),
            stats=torch.empty((F, STATS_BYTES), dtype=torch.uint8, device=dev),
            u=torch.empty((F, code.n), dtype=torch.float64, device=dev) if want_u else None,
            y=torch.empty((F, code.m), dtype=torch.float64, device=dev) if want_y else None,
            masks=torch.empty((F, code.m), dtype=torch.int16, device=dev) if want_masks else None,
        )
    pp = C.byref(params) if params is not None else None
    nbytes = lib().alp_decode_workspace_bytes(code.handle, F, pp)
    if nbytes == 0 and F > 0:
        raise _sizing_error()
    ws = (workspace or _ws("decode", dev)).get(nbytes)
    _check(lib().alp_decode(code.handle, F, _ptr(llr), _ptr(out.hard), _ptr(out.objective),
                            _ptr(out.certificate), _ptr(out.status), _ptr(out.stats), _ptr(out.u),
                            _ptr(out.y), _ptr(out.masks), ws.data_ptr(), ws.numel(), pp,
                            _stream_ptr(stream)))
    return out


def decode_host(code: Code, llr_host: torch.Tensor, params: AlpParams | None = None, stream=None,
                workspace: Workspace | None = None, out: dict | None = None) -> dict:
    """alp_decode_host: host LLRs in, host outputs back (copies inside the call)."""
    if llr_host.dtype != torch.float64 or llr_host.is_cuda or llr_host.shape[1] != code.n:
        raise ValueError("llr_host must be a CPU float64 tensor of shape [F, n]")
    llr_host = llr_host.contiguous()
    F = llr_host.shape[0]
    pin = llr_host.is_pinned()
    if out is None:
        out = dict(hard=torch.empty((F, code.n), dtype=torch.uint8, pin_memory=pin),
                   objective=torch.empty(F, dtype=torch.float64, pin_memory=pin),
                   certificate=torch.empty(F, dtype=torch.uint8, pin_memory=pin),
                   status=torch.empty(F, dtype=torch.int32, pin_memory=pin))
    pp = C.byref(params) if params is not None else None
    nbytes = lib().alp_decode_host_workspace_bytes(code.handle, F, pp)
    if nbytes == 0 and F > 0:
        raise _sizing_error()
    ws = (workspace or _ws("decode_host", "cuda")).get(nbytes)
    _check(lib().alp_decode_host(code.handle, F, _ptr(llr_host), _ptr(out["hard"]),
                                 _ptr(out["objective"]), _ptr(out["certificate"]), _ptr(out["status"]),
                                 None, ws.data_ptr(), ws.numel(), pp, _stream_ptr(stream)))
    return out


@dataclass
class StepResult:
    dy: torch.Tensor
    iters: torch.Tensor
    relres: torch.Tensor
    status: torch.Tensor
    pivot_rows: torch.Tensor | None = None
    pivot_cols: torch.Tensor | None = None


def ipm_step_pcg(code: Code, masks: torch.Tensor, d: torch.Tensor, r: torch.Tensor,
                 flip: torch.Tensor | None = None, params: AlpParams | None = None,
                 want_pivots=False, stream=None, workspace: Workspace | None = None) -> StepResult:
    """Isolated step-direction solve A D^2 A^T dy = r for [S] systems (device tensors)."""
    S = masks.shape[0]
    dev = masks.device
    if masks.dtype not in (torch.int16, torch.uint16) or masks.shape != (S, code.m):
        raise ValueError("masks must be int16/uint16 [S, m]")
    if d.dtype != torch.float64 or d.shape != (S, code.n + code.m):
        raise ValueError("d must be float64 [S, n+m]")
    if r.dtype != torch.float64 or r.shape != (S, code.m):
        raise ValueError("r must be float64 [S, m]")
    if flip is not None and (flip.dtype != torch.uint8 or flip.shape != (S, code.n)):
        raise ValueError("flip must be uint8 [S, n]")
    for t in (masks, d, r) + ((flip,) if flip is not None else ()):
        if not t.is_cuda:
            raise ValueError("inputs must be CUDA tensors")
    masks, d, r = masks.contiguous(), d.contiguous(), r.contiguous()
    res = StepResult(dy=torch.empty((S, code.m), dtype=torch.float64, device=dev),
                     iters=torch.empty(S, dtype=torch.int32, device=dev),
                     relres=torch.empty(S, dtype=torch.float64, device=dev),
                     status=torch.empty(S, dtype=torch.int32, device=dev))
    if want_pivots:
        res.pivot_rows = torch.empty((S, code.m), dtype=torch.int32, device=dev)
        res.pivot_cols = torch.empty((S, code.m), dtype=torch.int32, device=dev)
    pp = C.byref(params) if params is not None else None
    nbytes = lib().alp_pcg_workspace_bytes(code.handle, S, pp)
    if nbytes == 0 and S > 0:
        raise _sizing_error()
    ws = (workspace or _ws("pcg", dev)).get(nbytes)
    _check(lib().ipm_step_pcg(code.handle, S, _ptr(masks), _ptr(flip), _ptr(d), _ptr(r), _ptr(res.dy),
                              _ptr(res.iters), _ptr(res.relres), _ptr(res.status), _ptr(res.pivot_rows),
                              _ptr(res.pivot_cols), ws.data_ptr(), ws.numel(), pp, _stream_ptr(stream)))
    return res


def last_launch_count() -> int:
    return int(lib().alp_last_launch_count())


def launch_info(code: "Code", units: int, params=None, step: bool = False) -> dict:
    """Launch plan the library would use (alp_launch_info): window mode, frames per CTA, grid,
    shared-memory bytes per frame / per CTA, slot bytes per warp."""
    info = (C.c_int32 * 6)()
    pp = C.byref(params) if params is not None else None
    _check(lib().alp_launch_info(code.handle, int(units), pp, 1 if step else 0, C.addressof(info)))
    return dict(smem_mode=bool(info[0]), frames_per_cta=info[1], grid=info[2], smem_per_frame=info[3],
                smem_per_cta=info[4], slot_bytes=info[5])
