"""ORACLE (test infrastructure only — see oracle/__init__.py).

O(E) LP-duality certificate of a decode output, needing no
LP solve.  Inputs are a decoder's final u, the duals y of its final pool LP (per check,
0 on absent checks) and the pool masks.

  (i)   u lies in the fundamental polytope: Alg. 2 finds no cut with
        lhs < 1 - tol_cut on any check, and -tol <= u <= 1 + tol;
  (ii)  (y, z = c - A^T y) is dual feasible for the final pool LP in augmented form
        (dual LP P:418-428 read as "maximize b^T y", G4): z_std >= -tol_z (1 + ||c||),
        and the slack columns give z_{n+j} = -y_j >= -tol_z (1 + ||c||), i.e. y <= tol_z (1 + ||c||)
        (the same relative scale as the IPM's dual-feasibility stop, reading C-8);
  (iii) weak duality: for every x feasible for the full LP (which satisfies the pool rows
        and 0 <= x_aug <= ub, ub = 1 on standard and d_j on slack columns)
        c^T x = b^T y + z^T x_aug >= LB := b^T y + sum_i min(0, z_i) ub_i,
        while UB := c^T x(u) >= OPT because u is feasible.  Require UB - LB <= tol_gap (1+|UB|).
Then |gamma^T u - OPT| <= UB - LB.
"""
from __future__ import annotations

import numpy as np

from .lp import find_violated_cut


def dual_certificate(code, gamma, u, y, masks, tol_cut=1.001e-6, tol_box=1.001e-6, tol_z=1e-7,
                     tol_gap=1e-6):
    gamma = np.asarray(gamma, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n, m = code.n, code.m
    flip = gamma < 0
    c = np.abs(gamma)
    cn = float(np.max(c)) if n else 0.0
    out = dict(ok=True, reasons=[])
    # (i) primal feasibility in the full polytope
    min_lhs = np.inf
    for j in range(m):
        _, lhs, _ = find_violated_cut(u[code.N(j)])
        min_lhs = min(min_lhs, lhs)
    out["min_lhs"] = float(min_lhs)
    if m and min_lhs < 1.0 - tol_cut:
        out["ok"] = False
        out["reasons"].append(f"cut violated: min lhs {min_lhs}")
    if np.any(u < -tol_box) or np.any(u > 1.0 + tol_box):
        out["ok"] = False
        out["reasons"].append("box")
    # (ii) dual feasibility of (y, c - A^T y) on the final pool LP
    x = np.where(flip, 1.0 - u, u)
    z = c.copy()
    LB = 0.0
    slack_terms = 0.0
    for j in range(m):
        w = int(masks[j])
        if not (w >> 15) & 1:
            continue
        Nj = code.N(j)
        d = len(Nj)
        inV = np.array([(w >> t) & 1 for t in range(d)], dtype=bool)
        a = np.where(inV, 1.0, -1.0)
        s = np.where(flip[Nj], -1.0, 1.0)
        coef = a * s
        b = inV.sum() - 1.0 - np.sum(a[flip[Nj]])
        z[Nj] -= coef * y[j]
        LB += b * y[j]
        if y[j] > tol_z * (1.0 + cn):
            out["ok"] = False
            out["reasons"].append(f"y[{j}] = {y[j]} > 0")
        slack_terms += min(0.0, -y[j]) * d
    if np.any(z < -tol_z * (1.0 + cn)):
        out["ok"] = False
        out["reasons"].append(f"z min {float(np.min(z))}")
    # (iii) weak duality gap
    UB = float(c @ x)
    LB += float(np.sum(np.minimum(0.0, z))) + slack_terms
    out.update(UB=UB, LB=LB, gap=UB - LB, opt_lo=LB + float(np.sum(gamma[flip])),
               opt_hi=UB + float(np.sum(gamma[flip])))
    if UB - LB > tol_gap * (1.0 + abs(UB)):
        out["ok"] = False
        out["reasons"].append(f"duality gap {UB - LB}")
    return out


def dual_certificate_batch(code, gamma, u, y, masks, tol_cut=1.001e-6, tol_box=1.001e-6, tol_z=1e-7,
                           tol_gap=1e-6):
    """dual_certificate over a batch of frames ([F, n] / [F, m] arrays), vectorised with numpy
    (same three checks, same tolerances).  Returns a dict of per-frame arrays incl. ok."""
    gamma = np.asarray(gamma, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    masks = np.asarray(masks).astype(np.int64) & 0xFFFF
    Fn, n = u.shape
    m = code.m
    deg = np.diff(code.row_ptr).astype(np.int64)
    dc = int(deg.max())
    Nb = np.zeros((m, dc), dtype=np.int64)
    valid = np.arange(dc)[None, :] < deg[:, None]
    for j in range(m):
        Nb[j, :deg[j]] = code.N(j)
    un = u[:, Nb]                                         # [F, m, dc]
    # (i) Alg. 2 on every check
    S = (un > 0.5) & valid
    cntS = S.sum(axis=2)
    dist = np.where(valid, np.abs(un - 0.5), np.inf)
    istar = np.argmin(dist, axis=2)                       # first minimum = lowest position
    toggle = (cntS % 2 == 0)[..., None] & (np.arange(dc)[None, None, :] == istar[..., None])
    V = S ^ toggle
    lhs = np.where(valid, np.where(V, 1.0 - un, un), 0.0).sum(axis=2)
    min_lhs = lhs.min(axis=1)
    ok = min_lhs >= 1.0 - tol_cut
    ok &= np.all((u >= -tol_box) & (u <= 1.0 + tol_box), axis=1)
    # (ii) dual feasibility on the final pool LP
    flip = gamma < 0
    c = np.abs(gamma)
    cn = c.max(axis=1)
    present = ((masks >> 15) & 1).astype(bool)            # [F, m]
    inV = ((masks[..., None] >> np.arange(dc)[None, None, :]) & 1).astype(bool) & valid
    a = np.where(inV, 1.0, -1.0)
    fl = flip[:, Nb]                                      # [F, m, dc]
    coef = np.where(valid, a * np.where(fl, -1.0, 1.0), 0.0)
    yp = np.where(present, y, 0.0)
    z = c.copy()
    contrib = (coef * yp[..., None])                      # [F, m, dc]
    flat = (np.arange(Fn)[:, None, None] * n + Nb[None, :, :])
    np.subtract.at(z.reshape(-1), flat[:, valid].reshape(-1), contrib[:, valid].reshape(-1))
    b = inV.sum(axis=2) - 1.0 - np.where(valid & fl, a, 0.0).sum(axis=2)
    ok &= np.all(~present | (y <= tol_z * (1.0 + cn)[:, None]), axis=1)
    ok &= z.min(axis=1) >= -tol_z * (1.0 + cn)
    x = np.where(flip, 1.0 - u, u)
    UB = (c * x).sum(axis=1)
    LB = (np.where(present, b * y, 0.0)).sum(axis=1) + np.minimum(0.0, z).sum(axis=1) \
        + np.where(present, np.minimum(0.0, -y) * deg[None, :], 0.0).sum(axis=1)
    gap = UB - LB
    ok &= gap <= tol_gap * (1.0 + np.abs(UB))
    return dict(ok=ok, min_lhs=min_lhs, gap=gap, UB=UB, LB=LB)
