"""ORACLE (test infrastructure only — see oracle/__init__.py).

MALP decoding with every LP of Alg. 3 line 13 handed to a LIBRARY LP solver
(scipy's HiGHS dual simplex) in place of the oracle's own dense interior-point method.

Why it exists: at config 4 (n = 32,000; p ~ 1e4 cut rows) `oracle.lp.ipm_solve` spends
about an hour per frame in dense Cholesky factorisations of A D^2 A^T and ends on its
Newton-step cap (tools/make_c4_golden.py: status IPM_MAXITER on both committed frames), so
it proves nothing there.  The LP itself has a plain definition — eq.`primal LP` P:404-416:
min c^T x s.t. A x = b, x >= 0 on the augmented form of the current cut pool — and what
Alg. 3 outputs depends on the LP optimum alone (unique for continuous LLRs), not
on how it was reached (Thm 2c).  A library primitive may serve as that step.

  library_lp_solve     min c^T x s.t. A x = b, x >= 0 by scipy.optimize.linprog (HiGHS dual
                       simplex); returns the same fields as oracle.lp.ipm_solve
                       (y = dual of A x = b under G4 / C-25: max b^T y, A^T y + z = c)
  malp_decode_library  oracle.lp.malp_decode (Alg. 3 / P:242, same cut search, pool update,
                       cycle rule C-12 and outputs) with that LP step

Pinned in tests/test_oracle_library_lp.py: against oracle.lp.malp_decode (the IPM path)
frame by frame on config 1, against the Bland-rule simplex on the FULL Feldman relaxation
and brute-force ML on tiny codes, and by the LP-duality certificate of oracle/certify.py
on its own (u, y, pool).  Iteration counts: the LP count is the IPM path's whenever both
reach the same vertices; `ipm_iters` reports HiGHS's simplex iterations (not comparable,
"parity unpinned" like every count).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog

from .lp import ST_NUMERIC, ST_OK, malp_decode


def library_lp_solve(A, b, c, params=None, step_solver=None, record=False):
    """min c^T x s.t. A x = b, x >= 0 (eq.`primal LP` P:404-416) by HiGHS dual simplex.

    Same call shape and result fields as oracle.lp.ipm_solve so that malp_decode can take
    either.  y is the equality-constraint multiplier d(obj)/d(b), i.e. the dual variable of
    max b^T y s.t. A^T y + z = c, z >= 0 (G4 / C-25); z = c - A^T y.
    """
    A = sp.csr_matrix(A, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)
    res = linprog(c, A_eq=A, b_eq=b, bounds=(0, None), method="highs-ds",
                  options=dict(presolve=True, primal_feasibility_tolerance=1e-9,
                               dual_feasibility_tolerance=1e-9))
    if res.status != 0:
        q = c.size
        return dict(x=np.full(q, np.nan), y=np.zeros(b.size), z=np.full(q, np.nan), iters=int(getattr(res, "nit", 0)),
                    status=ST_NUMERIC, hist=[], chol_fixes=0, pcg_iters=0, pcg_status=0)
    x = np.asarray(res.x, dtype=np.float64)
    y = np.asarray(res.eqlin.marginals, dtype=np.float64)
    z = c - A.T @ y
    return dict(x=x, y=y, z=z, iters=int(res.nit), status=ST_OK, hist=[], chol_fixes=0,
                pcg_iters=0, pcg_status=0)


def malp_decode_library(code, gamma, variant: str = "A", params=None, record=False):
    """Alg. 3 MALP-A / MALP-B with the LP step solved by HiGHS."""
    return malp_decode(code, gamma, variant=variant, params=params, record=record,
                       lp_solver=library_lp_solve)
