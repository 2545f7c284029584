"""ORACLE (test infrastructure only — see oracle/__init__.py).

Adaptive LP decoding written out step by step from PAPER.md:

  hard_decision        eq.`initial constraints` P:147-155
  cut_lhs              eq.`constraints2` P:114-118 (left-hand side)
  find_violated_cut    Alg. 2 P:185-201 (ties: reading C-2)
  augmented_lp         §IV-B P:404-416 (flip to x_i >= 0, slack per row), eq.`MALP matrix form` P:246-257
  ipm_solve            §IV-B infeasible primal-dual path following P:401-504:
                       residuals eq.`matrix equation` P:455-474, normal equations
                       eq.`Delta y` P:479, recovery eq.`Delta x`/`Delta z` P:480-481,
                       D^2 = X Z^-1 eq.`definition of D2` P:484-487, mu eq.`update mu`
                       P:496-500 with sigma (C-5), ratio test (C-6), start (C-7),
                       stopping rule (C-8).  The step solve is DIRECT (Cholesky of
                       the dense A D^2 A^T; safeguard C-29) — no PCG.
  step_solve_exact     dy = (A D^2 A^T)^-1 w in extended precision (reference for PCG parity)
  malp_decode          Alg. 3 MALP-A P:220-240; MALP-B P:242; plain ALP Alg. 1
  decode_outputs       hard decision, objective gamma^T u, ML certificate (C-11, C-14)

All arithmetic is fp64.  Constants are those of DESIGN.md §3
and are identical to the CUDA path's alp_default_params().
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

PRESENT = 1 << 15
SPARSE_Q = 8192     # LPs with more columns keep A in sparse storage (config 4; same products)

# DESIGN.md §3 / SURVEY.md §8(c) c.3 constants (C-3, C-4, C-5, C-6, C-8, C-9, C-11, C-12)
DEFAULT_PARAMS = dict(
    sigma=0.1, eta=0.99,
    gap_tol=1e-9, feas_tol=1e-8,
    pcg_rel_tol=1e-8,
    tau_viol=1e-6, tau_act=1e-6, tau_cert=1e-2,
    alp_max_iter=200, ipm_max_iter=100, pcg_max_iter=1000,
    stop_on_lp_failure=1,
)

# per-frame status bits (mirrors include/alp.h alp_frame_status)
ST_OK, ST_ALP_MAXITER, ST_IPM_MAXITER, ST_PCG_MAXITER, ST_PCG_BREAKDOWN, ST_NUMERIC = 0, 1, 2, 4, 8, 16


def params_with(**kw):
    p = dict(DEFAULT_PARAMS)
    p.update(kw)
    return p


# --------------------------------------------------------------------------- cut search
def hard_decision(gamma: np.ndarray) -> np.ndarray:
    """u_i = 0 if gamma_i >= 0 else 1: the optimum of LP^0 (eq.`initial constraints`)."""
    return (np.asarray(gamma) < 0).astype(np.float64)


def cut_lhs(u_nb: np.ndarray, inV: np.ndarray) -> float:
    """LHS of eq.`constraints2`: sum_{i in V}(1 - u_i) + sum_{i in N(j)\\V} u_i."""
    u_nb = np.asarray(u_nb, dtype=np.float64)
    inV = np.asarray(inV, dtype=bool)
    return float(np.sum(1.0 - u_nb[inV]) + np.sum(u_nb[~inV]))


def find_violated_cut(u_nb: np.ndarray, tau_viol: float = 0.0):
    """Alg. 2 for one check, given u restricted to N(j) (sorted).

    Returns (inV, lhs, violated): inV marks V within N(j).  Line 1: S = {u_i > 1/2}
    (strict, C-2).  Lines 2-6: if |S| is even toggle i* = argmin |u_i - 1/2|, ties to
    the lowest position (C-2).  Line 8: violated iff eq.`constraints2` fails, read as
    lhs < 1 - tau_viol (C-3).
    """
    u_nb = np.asarray(u_nb, dtype=np.float64)
    S = u_nb > 0.5
    V = S.copy()
    if int(S.sum()) % 2 == 0:
        istar = int(np.argmin(np.abs(u_nb - 0.5)))   # argmin returns the first (lowest) index on ties
        V[istar] = not V[istar]
    lhs = cut_lhs(u_nb, V)
    return V, lhs, lhs < 1.0 - tau_viol


def mask_word(inV: np.ndarray) -> int:
    """Pack V (bit t <-> N(j)[t]) with the present bit, as in include/alp.h."""
    w = PRESENT
    for t, b in enumerate(inV):
        if b:
            w |= 1 << t
    return w


def mask_bits(word: int, d: int) -> np.ndarray:
    return np.array([(int(word) >> t) & 1 for t in range(d)], dtype=bool)


# --------------------------------------------------------------------------- augmented LP
def augmented_lp(code, pool: dict, gamma: np.ndarray):
    """Primal LP in augmented form (eq.`primal LP`).

    Rows: present checks in ascending order (MALP pool: one cut per check, Thm 3).
    For check j with cut V, the parity inequality sum_V u - sum_{N\\V} u <= |V| - 1
    (eq.`constraints`) with u_i = x_i (gamma_i >= 0) or u_i = 1 - x_i
    (gamma_i < 0) becomes sum_i a_ji s_i x_i + x_{n+r} = |V| - 1 - sum_{i flipped} a_ji,
    a_ji = +1 on V, -1 off V, s_i = -1 if flipped.  Cost c_i = |gamma_i|, slack cost 0.
    Returns dict with A (p x q; dense, or scipy.sparse CSR when q > SPARSE_Q — storage only,
    for config 4), b (p), c (q), rows (check ids), flip, const
    (= sum_{gamma_i<0} gamma_i so that gamma^T u = c^T x + const).
    """
    gamma = np.asarray(gamma, dtype=np.float64)
    n = code.n
    flip = gamma < 0
    rows = sorted(pool.keys())
    p = len(rows)
    q = n + p
    ri, ci, vals = [], [], []
    b = np.zeros(p)
    for r, j in enumerate(rows):
        Nj = code.N(j)
        inV = np.asarray(pool[j], dtype=bool)
        a = np.where(inV, 1.0, -1.0)
        s = np.where(flip[Nj], -1.0, 1.0)
        ri += [r] * (len(Nj) + 1)
        ci += list(Nj) + [n + r]
        vals += list(a * s) + [1.0]
        b[r] = inV.sum() - 1.0 - np.sum(a[flip[Nj]])
    A = sp.csr_matrix((vals, (ri, ci)), shape=(p, q))
    if q <= SPARSE_Q:
        A = A.toarray()
    c = np.concatenate([np.abs(gamma), np.zeros(p)])
    const = float(np.sum(gamma[flip]))
    return dict(A=A, b=b, c=c, rows=rows, flip=flip, n=n, p=p, q=q, const=const)


# --------------------------------------------------------------------------- step solve
def cholesky_solve(Q: np.ndarray, w: np.ndarray, info: dict | None = None) -> np.ndarray:
    """dy = Q^-1 w by Cholesky (Q = A D^2 A^T is SPD).

    Safeguard C-29: a pivot <= 1e-30 * max_k Q_kk (or non-positive) is replaced by 1e64,
    which drives that direction's component of dy to ~0.  LAPACK is used when it
    succeeds with no tiny pivot; otherwise the plain column Cholesky below runs.
    """
    p = Q.shape[0]
    if p == 0:
        return np.zeros(0)
    qmax = float(np.max(np.diag(Q)))
    thresh = 1e-30 * qmax
    L = None
    try:
        L = np.linalg.cholesky(Q)
        if np.any(np.diag(L) ** 2 <= thresh):
            L = None
    except np.linalg.LinAlgError:
        L = None
    if L is None:
        L = np.zeros_like(Q)
        nfix = 0
        for k in range(p):
            dkk = Q[k, k] - L[k, :k] @ L[k, :k]
            if not (dkk > thresh):
                dkk = 1e64
                nfix += 1
            L[k, k] = np.sqrt(dkk)
            L[k + 1:, k] = (Q[k + 1:, k] - L[k + 1:, :k] @ L[k, :k]) / L[k, k]
        if info is not None:
            info["chol_fixes"] = info.get("chol_fixes", 0) + nfix
    t = sla.solve_triangular(L, w, lower=True)
    return sla.solve_triangular(L.T, t, lower=False)


def step_solve_exact(A, d2: np.ndarray, w: np.ndarray, refine: int = 12) -> np.ndarray:
    """dy = Q^-1 w, Q = A D^2 A^T (eq.`Delta y`), to full fp64 accuracy even when
    kappa(Q) ~ 1e18 (config 5, d^2 over 24 decades; SURVEY C-27).

    The plain definition, solved by iterative refinement whose residuals are EXACT: every input
    is a dyadic rational (A is +-1/0, d2 and w are fp64), so r = w - A D^2 A^T y is computed in
    exact rational arithmetic (fractions.Fraction over A's nonzeros), y itself is kept exact as
    the sum of its corrections, and each correction solves Q delta = r with a long-double
    (x87, eps 1.1e-19) column Cholesky of Q.  The error contracts by ~kappa * eps_longdouble per
    step, so for kappa < ~1e18 the result is the correctly rounded solution after a few steps
    (stop when a correction is below 1e-22 of |y|, at most `refine` steps).  (Refining with
    long-double residuals alone, as round 1 did, stalls at kappa * eps_longdouble, ~1e-7 on some
    config-5 systems — measured against this.)  Reference for the GPU PCG parity of
    ipm_step_pcg; fp64 Cholesky (cholesky_solve) cannot serve there."""
    from fractions import Fraction
    A = np.asarray(A.todense()) if sp.issparse(A) else np.asarray(A)
    ld = np.longdouble
    p = A.shape[0]
    if p == 0:
        return np.zeros(0)
    d2 = np.asarray(d2, dtype=np.float64)
    # Q = sum_i d2_i a_i a_i^T over the columns a_i of A (the definition, summed column by
    # column) — only the nonzeros of a_i touch Q
    Q = np.zeros((p, p), dtype=ld)
    d2l = d2.astype(ld)
    cols = []
    for i in range(A.shape[1]):
        nz = np.nonzero(A[:, i])[0]
        if nz.size:
            a = A[nz, i]
            cols.append((i, nz.tolist(), [int(v) for v in a]))
            al = a.astype(ld)
            Q[np.ix_(nz, nz)] += d2l[i] * np.outer(al, al)
    L = np.zeros_like(Q)
    for k in range(p):
        dkk = Q[k, k] - L[k, :k] @ L[k, :k]
        if not dkk > 0:
            raise np.linalg.LinAlgError("Q not numerically SPD in extended precision")
        L[k, k] = np.sqrt(dkk)
        L[k + 1:, k] = (Q[k + 1:, k] - L[k + 1:, :k] @ L[k, :k]) / L[k, k]

    def solve(b):
        t = np.zeros(p, dtype=ld)
        for k in range(p):
            t[k] = (b[k] - L[k, :k] @ t[:k]) / L[k, k]
        y = np.zeros(p, dtype=ld)
        for k in range(p - 1, -1, -1):
            y[k] = (t[k] - L[k + 1:, k] @ y[k + 1:]) / L[k, k]
        return y

    def exact(v):   # a long double as an exact rational (its fp64 head + fp64 tail)
        h = float(v)
        return Fraction(h) + Fraction(float(v - ld(h)))

    d2f = [Fraction(float(v)) for v in d2]
    wf = [Fraction(float(v)) for v in np.asarray(w, dtype=np.float64)]

    def residual(yf):   # w - A (D^2 (A^T y)), exact
        l = [Fraction(0)] * p
        for i, nz, a in cols:
            t = Fraction(0)
            for r, av in zip(nz, a):
                t = t + yf[r] if av > 0 else t - yf[r]
            t *= d2f[i]
            for r, av in zip(nz, a):
                l[r] = l[r] + t if av > 0 else l[r] - t
        return [wf[r] - l[r] for r in range(p)]

    y = solve(np.asarray(w, dtype=np.float64).astype(ld))
    yf = [exact(v) for v in y]
    ynorm = float(np.linalg.norm(y.astype(np.float64)))
    for _ in range(refine):
        r = residual(yf)
        dl = solve(np.array([float(v) for v in r], dtype=np.float64).astype(ld))
        yf = [a + exact(b) for a, b in zip(yf, dl)]
        if not float(np.linalg.norm(dl.astype(np.float64))) > 1e-22 * ynorm:
            break
    return np.array([float(v) for v in yf])


def normal_matrix(A, d2: np.ndarray) -> np.ndarray:
    """Q = A D^2 A^T (eq.`Delta y` left-hand side), returned dense.

    A may be dense or scipy.sparse (a storage choice only: same products)."""
    if sp.issparse(A):
        return np.asarray((A @ sp.diags(d2) @ A.T).todense())
    return (A * d2) @ A.T


# --------------------------------------------------------------------------- IPM
def newton_direction(A, x, z, rb, rc, mu, step_solver=None, info=None):
    """Newton direction of eq.`matrix equation` via the normal equations:
    r_e = mu e - X Z e, D^2 = X Z^-1 (eq.`definition of D2`),
    (A D^2 A^T) dy = r_b + A D^2 r_c - A Z^-1 r_e   (eq.`Delta y`)
    dx = D^2 A^T dy - D^2 r_c + Z^-1 r_e              (eq.`Delta x`)
    dz = X^-1 (r_e - Z dx)                           (eq.`Delta z`)
    The step solve is Cholesky unless a step_solver(A, d2, w, info) is supplied."""
    re = mu - x * z
    d2 = x / z
    w = rb + A @ (d2 * rc - re / z)
    if step_solver is None:
        dy = cholesky_solve(normal_matrix(A, d2), w, info)
    else:
        dy = step_solver(A, d2, w, info)
    dx = d2 * (A.T @ dy) - d2 * rc + re / z
    dz = (re - z * dx) / x
    return dx, dy, dz


def step_lengths(x, z, dx, dz, eta):
    """beta_P = min(1, eta * min_{dx_i<0} -x_i/dx_i), beta_D likewise on z (C-6)."""
    neg = dx < 0
    bP = min(1.0, eta * float(np.min(-x[neg] / dx[neg]))) if np.any(neg) else 1.0
    neg = dz < 0
    bD = min(1.0, eta * float(np.min(-z[neg] / dz[neg]))) if np.any(neg) else 1.0
    return bP, bD


def ipm_solve(A, b, c, params=None, step_solver=None, record=False):
    """Infeasible primal-dual path-following IPM (§IV-B) on
    min c^T x s.t. A x = b, x >= 0.

    Start x = z = s0 e, y = 0 with s0 = max(1, ||b||_inf, ||c||_inf) (C-7).
    Each iteration: r_b = b - A x, r_c = c - A^T y - z, gap = x^T z;
    stop if gap <= gap_tol (1 + |c^T x|), ||r_b||_inf <= feas_tol (1 + ||b||_inf),
    ||r_c||_inf <= feas_tol (1 + ||c||_inf) (C-8); else mu = sigma gap / q
    (eq.`update mu` with C-5), r_e = mu e - X Z e, D^2 = X Z^-1, solve
    (A D^2 A^T) dy = r_b + A D^2 r_c - A Z^-1 r_e (eq.`Delta y`),
    dx = D^2 A^T dy - D^2 r_c + Z^-1 r_e (eq.`Delta x`), dz = X^-1 (r_e - Z dx)
    (eq.`Delta z`); beta_P = min(1, eta min_{dx_i<0} -x_i/dx_i), beta_D likewise on z
    (C-6); x += beta_P dx, y += beta_D dy, z += beta_D dz.
    At most ipm_max_iter Newton steps.
    """
    P = dict(DEFAULT_PARAMS) if params is None else params
    A = sp.csr_matrix(A, dtype=np.float64) if sp.issparse(A) else np.asarray(A, dtype=np.float64)
    p, q = A.shape
    if q > 256 and not sp.issparse(A):
        A = sp.csr_matrix(A)   # storage only; every product below is unchanged
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    bnorm = float(np.max(np.abs(b))) if p else 0.0
    cnorm = float(np.max(np.abs(c))) if q else 0.0
    s0 = max(1.0, bnorm, cnorm)
    x = np.full(q, s0)
    z = np.full(q, s0)
    y = np.zeros(p)
    hist = []
    info: dict = {}
    status = ST_OK
    it = 0
    while True:
        rb = b - A @ x
        rc = c - A.T @ y - z
        gap = float(x @ z)
        cx = float(c @ x)
        rbn = float(np.max(np.abs(rb))) if p else 0.0
        rcn = float(np.max(np.abs(rc)))
        if record:
            hist.append(dict(it=it, gap=gap, rb=rbn, rc=rcn, cx=cx))
        if (gap <= P["gap_tol"] * (1.0 + abs(cx)) and rbn <= P["feas_tol"] * (1.0 + bnorm)
                and rcn <= P["feas_tol"] * (1.0 + cnorm)):
            break
        if it >= P["ipm_max_iter"]:
            status |= ST_IPM_MAXITER
            break
        mu = P["sigma"] * gap / q
        dx, dy, dz = newton_direction(A, x, z, rb, rc, mu, step_solver, info)
        bP, bD = step_lengths(x, z, dx, dz, P["eta"])
        x = x + bP * dx
        y = y + bD * dy
        z = z + bD * dz
        it += 1
        if not (np.all(np.isfinite(x)) and np.all(np.isfinite(z)) and np.all(np.isfinite(y))):
            status |= ST_NUMERIC
            break
    return dict(x=x, y=y, z=z, iters=it, status=status, hist=hist,
                chol_fixes=info.get("chol_fixes", 0), pcg_iters=info.get("pcg_iters", 0),
                pcg_status=info.get("pcg_status", 0))


# --------------------------------------------------------------------------- decode
def slack_of(code, j: int, inV, u: np.ndarray) -> float:
    """Slack of check j's cut at u: lhs - 1 (eq.`constraints2`; active iff ~0, C-4)."""
    return cut_lhs(u[code.N(j)], inV) - 1.0


def decode_outputs(code, gamma, u, tau_cert, lp_converged=True):
    """Hard decision [u_i > 1/2] (C-14), objective gamma^T u (C-13), g_max and the
    ML certificate: integral (g_max <= tau_cert, C-11) and H hard = 0 mod 2.
    The certificate claims u is the LP optimum; when the last LP's IPM did not converge
    (Newton-step cap or non-finite iterate) u is not, and it never certifies (C-31)."""
    gamma = np.asarray(gamma, dtype=np.float64)
    hard = (u > 0.5).astype(np.uint8)
    obj = float(gamma @ u)
    g_max = float(np.max(np.minimum(u, 1.0 - u))) if u.size else 0.0
    parity_ok = all(int(hard[code.N(j)].sum()) % 2 == 0 for j in range(code.m))
    cert = int(g_max <= tau_cert and parity_ok and lp_converged)
    return hard, obj, g_max, cert


def malp_decode(code, gamma, variant: str = "A", params=None, step_solver=None, record=False,
                lp_solver=None):
    """Adaptive LP decoding of one frame.

    variant "A": MALP-A, Alg. 3.  For every check j (all read u^{k-1}):
      skip j if its pool cut is active (slack <= tau_act; line 6, Cor. 2 P:208-213);
      else run Alg. 2; if violated, replace j's cut (lines 8-9).  If nothing changed,
      stop and output the last solved u (G2); else solve the LP (line 13).
    variant "B": MALP-B: first remove every inactive pool cut, then as "A".
    variant "ALP": Alg. 1: add every violated cut found at u^{k-1}; never
      remove (several cuts per check may accumulate).
    At most alp_max_iter LPs (C-12); a frame that would need more gets ST_ALP_MAXITER, and
    so does a MALP frame whose new pool equals the pool of an LP it already solved (the
    deterministic cycle C-12 describes; detected before solving the repeat).
    lp_solver: the LP step of line 13 (default: ipm_solve, this module's IPM); oracle/lp_library.py
    passes a library LP solver with the same call shape (large n, where the dense IPM is too slow).
    """
    P = dict(DEFAULT_PARAMS) if params is None else params
    gamma = np.asarray(gamma, dtype=np.float64)
    n, m = code.n, code.m
    u = hard_decision(gamma)
    pool: dict = {}          # MALP: j -> inV ; ALP: list of (j, inV)
    alp_rows: list = []
    status = ST_OK
    lp_solves = ipm_iters = max_p = chol_fixes = pcg_iters = 0
    y_check = np.zeros(m)
    trace = []
    objs = []
    seen_pools = set()      # reading C-12: a repeated pool is a deterministic cycle
    last_lp_ok = True       # the last solved LP converged (C-31)
    for k in range(P["alp_max_iter"] + 1):
        changed = False
        if variant == "B":
            for j in list(pool.keys()):
                if slack_of(code, j, pool[j], u) > P["tau_act"]:
                    del pool[j]
        for j in range(m):
            if variant in ("A", "B") and j in pool and slack_of(code, j, pool[j], u) <= P["tau_act"]:
                continue
            inV, lhs, viol = find_violated_cut(u[code.N(j)], P["tau_viol"])
            if viol:
                if variant == "ALP":
                    alp_rows.append((j, inV))
                else:
                    pool[j] = inV
                changed = True
        if not changed:
            break
        if k == P["alp_max_iter"]:
            status |= ST_ALP_MAXITER
            break
        if variant != "ALP":
            # The LP, hence u^k and the next cut search, are functions of the pool alone:
            # a pool equal to an earlier LP's pool repeats forever (C-12).  Stop with the
            # last solved u (G2) and the cap status.
            key = frozenset((j, int(mask_word(v))) for j, v in pool.items())
            if key in seen_pools:
                status |= ST_ALP_MAXITER
                break
            seen_pools.add(key)
        if variant == "ALP":
            lp = _augmented_multi(code, alp_rows, gamma)
        else:
            lp = augmented_lp(code, pool, gamma)
        res = (lp_solver or ipm_solve)(lp["A"], lp["b"], lp["c"], P, step_solver=step_solver)
        lp_solves += 1
        ipm_iters += res["iters"]
        max_p = max(max_p, lp["p"])
        chol_fixes += res["chol_fixes"]
        pcg_iters += res["pcg_iters"]
        status |= res["status"] & (ST_IPM_MAXITER | ST_NUMERIC | ST_PCG_MAXITER | ST_PCG_BREAKDOWN)
        last_lp_ok = not (res["status"] & (ST_IPM_MAXITER | ST_NUMERIC))
        xs = res["x"][:n]
        u = np.where(lp["flip"], 1.0 - xs, xs)
        y_check = np.zeros(m)
        if variant != "ALP":
            for r, j in enumerate(lp["rows"]):
                y_check[j] = res["y"][r]
        objs.append(float(gamma @ u))
        if record:
            trace.append(dict(pool={j: np.array(v) for j, v in pool.items()} if variant != "ALP"
                              else list(alp_rows), u=u.copy(), obj=objs[-1], p=lp["p"],
                              ipm_iters=res["iters"]))
        if (status & ST_NUMERIC) or (P.get("stop_on_lp_failure", 1) and (res["status"] & ST_IPM_MAXITER)):
            # reading C-30: an LP that did not converge gives no trustworthy u for the next
            # cut search; the frame stops with its status bits and the last u
            break
    hard, obj, g_max, cert = decode_outputs(code, gamma, u, P["tau_cert"], last_lp_ok)
    masks = np.zeros(m, dtype=np.uint16)
    if variant != "ALP":
        for j, inV in pool.items():
            masks[j] = mask_word(inV)
    return dict(u=u, hard=hard, obj=obj, g_max=g_max, cert=cert, status=status,
                lp_solves=lp_solves, ipm_iters=ipm_iters, max_p=max_p, masks=masks,
                y=y_check, trace=trace, objs=objs, chol_fixes=chol_fixes,
                pcg_iters=pcg_iters, pool=pool if variant != "ALP" else alp_rows)


def _augmented_multi(code, rows_list, gamma):
    """Augmented LP for plain ALP (Alg. 1), whose pool may hold several cuts per check."""
    gamma = np.asarray(gamma, dtype=np.float64)
    n = code.n
    flip = gamma < 0
    p = len(rows_list)
    q = n + p
    A = np.zeros((p, q))
    b = np.zeros(p)
    for r, (j, inV) in enumerate(rows_list):
        Nj = code.N(j)
        inV = np.asarray(inV, dtype=bool)
        a = np.where(inV, 1.0, -1.0)
        s = np.where(flip[Nj], -1.0, 1.0)
        A[r, Nj] = a * s
        A[r, n + r] = 1.0
        b[r] = inV.sum() - 1.0 - np.sum(a[flip[Nj]])
    c = np.concatenate([np.abs(gamma), np.zeros(p)])
    return dict(A=A, b=b, c=c, rows=[j for j, _ in rows_list], flip=flip, n=n, p=p, q=q,
                const=float(np.sum(gamma[flip])))
