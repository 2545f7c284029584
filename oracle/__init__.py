"""ORACLE — plain, slow, obviously-correct CPU reference.  TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_0902_0657_b200`, `libalp.so`) never imports, links or calls it,
and this package never imports the product.  The two share no code; only the
seeded input generators in `synth/` (which hold none of the method's
arithmetic) serve both.

Everything is fp64 numpy/scipy written in the paper's order and notation.
Citations are PAPER.md line numbers (P:n) with the section / algorithm /
equation label, and the readings C-n of SURVEY.md §8(c) restated in DESIGN.md.

Modules
  lp        Alg. 2 cut search, MALP-A / MALP-B (Alg. 3), plain ALP (Alg. 1),
            augmented form (§IV-B), infeasible primal-dual IPM with a direct
            (Cholesky) step solve, decode outputs and ML certificate.
  lp_library  Alg. 3 with the LP step (line 13) handed to a library LP solver (scipy HiGHS)
            instead of the dense IPM — the oracle for config 4 (n = 32,000), where the dense
            Cholesky IPM takes an hour per frame and ends on its cap.
  precond   Alg. 5 Triangulation Step, Alg. 6 incremental / Alg. 7 column-wise /
            Alg. 8 row-wise greedy MTS, the 3-stage preconditioner apply,
            PCG (Alg. 4).
  full_lp   dense Bland-rule simplex on the full Feldman relaxation
            (eq.`LP decoding`), brute-force ML decoding for tiny codes.
  certify   O(E) LP-duality certificate of a decode output (weak duality).
  peeling   erasure peeling and stopping sets (Thm 4, Lemma 2).

Pinning status (details in DESIGN.md §3 and tests/test_oracle_*.py):
every public function is pinned by a `-m "not gpu"` test against a worked
example, a closed form, an independent solver or brute force, except the
iteration COUNTS (ALP / IPM / PCG), which the paper gives only qualitatively
and which are therefore "parity unpinned" (reported, not gated).
"""
