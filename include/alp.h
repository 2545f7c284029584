/*
 * alp.h — C ABI of libalp.so: batched adaptive-LP decoding of LDPC codes on B200 (sm_100a).
 *
 * Method: Taghavi, Shokrollahi, Siegel, "Efficient Implementation of Linear Programming
 * Decoding" (arXiv 0902.0657).  Citations "P:n" are lines of that paper's text
 * with the section / algorithm / equation label.
 *
 * Two product calls, plus code handles, sizing and diagnostics:
 *
 *   alp_decode    — LP decoding of a batch of received frames by MALP-A / MALP-B
 *                   (Alg. 3), every LP solved by the infeasible
 *                   primal-dual path-following IPM (§IV-B) whose Newton step
 *                   (eq.`Delta y` P:479) is solved by PCG (Alg. 4) with the
 *                   column-wise greedy triangular preconditioner (Alg. 7 P:662-678,
 *                   M = A_M D_M^2 A_M^T).  Outputs per frame: hard decisions,
 *                   the LP objective gamma^T u, the ML-certificate flag.
 *   ipm_step_pcg  — the isolated step-direction solve A D^2 A^T dy = r (eq.`Delta y`)
 *                   for a batch of independent systems, same kernels as inside alp_decode.
 *
 * Conventions (all calls):
 *  - Pointers marked DEVICE must be device memory of the current CUDA device; HOST must be
 *    host memory (pinned for speed).  Work is enqueued on `stream` (a cudaStream_t passed
 *    as void*, NULL = legacy default stream) and is stream-ordered: outputs are valid after
 *    the stream is synchronised.  alp_decode_host synchronises `stream` before returning.
 *  - Ownership: the caller owns every buffer; the library never frees caller memory.
 *    An alp_code owns only its device copy of the Tanner graph.  All per-frame scratch
 *    comes from the caller's `workspace` (DEVICE, >= 256-byte aligned), sized by the
 *    matching *_workspace_bytes query.
 *  - Errors: argument / shape errors are returned synchronously before any launch
 *    (ALP_ERR_INVALID_ARG / ALP_ERR_BAD_CODE / ALP_ERR_UNSUPPORTED / ALP_ERR_WORKSPACE);
 *    CUDA launch or runtime errors map to ALP_ERR_CUDA; alp_last_error() gives a
 *    thread-local message for the last non-OK return.  Numerical outcomes of a frame
 *    (iteration caps, PCG breakdown, non-finite values) are VALUES in frame_status, never
 *    errors.  A fractional LP output is not an error either: certificate = 0 is the
 *    decoder's "failure" declaration.
 *  - Thread safety: an alp_code may be shared by concurrent calls; concurrent calls need
 *    distinct workspaces (and normally distinct streams).
 *  - Layouts are row-major with the frame (system) index slowest: [n_frames][n] etc.,
 *    i.e. each frame's vector is contiguous.  n_frames = 0 is valid and does nothing.
 *
 * Cut-mask word (uint16, one per check and frame/system): bit t (t < d_j <= 15) set <=>
 * N(j)[t] (the t-th smallest variable of check j) is in the odd set V of that check's
 * parity inequality sum_{V} u - sum_{N(j)\V} u <= |V| - 1 (eq.`constraints` P:107-110),
 * i.e. its coefficient is +1 (else -1) before the flip of §IV-B; bit 15 set <=> the
 * check's row is present in the LP.  At most one row per check (Thm 3).
 */
#ifndef ALP_H
#define ALP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ALP_OK = 0,
  ALP_ERR_INVALID_ARG = -1,  /* null pointer where required, negative size, bad params   */
  ALP_ERR_BAD_CODE = -2,     /* Tanner graph invalid: index out of range, duplicate, ... */
  ALP_ERR_UNSUPPORTED = -3,  /* valid but beyond this build: d_c > 15, d_v > 4,
                                n + m > 65535, m > 32767                                      */
  ALP_ERR_CUDA = -4,         /* a CUDA call failed (no device, launch failure, fault)    */
  ALP_ERR_WORKSPACE = -5     /* workspace NULL, misaligned or smaller than required      */
} alp_status;

/* Per-frame status bits (values, not errors). */
typedef enum {
  ALP_FRAME_OK = 0,
  ALP_FRAME_ALP_MAXITER = 1,     /* alp_max_iter LPs solved and cuts still change, or the cut
                                    pool repeated that of an LP already solved (a
                                    deterministic MALP cycle; C-12)                        */
  ALP_FRAME_IPM_MAXITER = 2,     /* some LP hit ipm_max_iter Newton steps                   */
  ALP_FRAME_PCG_MAXITER = 4,     /* some PCG recursion ended with ||r|| > pcg_rel_tol ||w||:
                                    at pcg_max_iter, or stalled (no new residual minimum in
                                    200 iterations; R-1).  The Newton step still
                                    proceeds with that dy (reading C-32)                   */
  ALP_FRAME_PCG_BREAKDOWN = 8,   /* some PCG solve met h^T Q h or z^T r = 0 / non-finite      */
  ALP_FRAME_NUMERIC = 16,        /* non-finite IPM iterate; decoding of the frame stopped   */
  ALP_FRAME_PCG_FLOOR = 32       /* informational, ipm_step_pcg only: the solve stopped with
                                    its TRUE residual above pcg_rel_tol ||w|| at the fp64
                                    attainable accuracy: at most the evaluation floor
                                    f = 16 eps || |A| D^2 |A|^T |dy| ||_2, or within 1e3 f with
                                    restarts (iterative refinement) no longer halving it    */
} alp_frame_status;

typedef struct alp_code alp_code;   /* opaque, immutable after creation */

/* Per-frame counters (alp_decode) — 128 bytes.  cyc_* are SM clock cycles (clock64) the
 * frame's warp spent per phase: cut search + sign tables, IPM body (residuals, rhs,
 * Newton recovery, update), preconditioner build (sort, Alg. 7 peel, level schedule),
 * PCG SpMV, PCG preconditioner sweeps, remaining PCG work (axpys, dots, true residual). */
typedef struct {
  int32_t lp_solves;   /* LPs solved (MALP outer iterations that added a cut)            */
  int32_t ipm_iters;   /* Newton steps summed over all LPs                                */
  int32_t pcg_iters;   /* PCG iterations summed over all Newton steps (all runs)          */
  int32_t max_p;       /* largest number of LP rows p (<= m, Cor. 3 P:289-292)             */
  int32_t pcg_solves;  /* Newton-step solves (one per Newton step)                         */
  int32_t pcg_p4_fail; /* solves whose final recursive residual ||r||/||w|| > pcg_rel_tol
                          (the failure count, 0 on a fully converged frame)     */
  int32_t pcg_true_fail; /* solves whose TRUE residual ||w - Q dy||/||w|| > pcg_rel_tol
                          (reported, not gated: the recovery tolerates it, C-32)         */
  int32_t reserved;
  double g_max;        /* max_i min(u_i, 1 - u_i) of the output (integrality, C-11)       */
  double pcg_bytes;    /* sum over PCG iterations of B_min(p, n_act, m)    */
  double max_rec_relres;  /* max over the frame's solves of the recursive ||r||/||w|| at exit */
  double max_true_relres; /* max over the frame's solves of the TRUE ||w - Q dy||/||w||     */
  int64_t cyc_cut, cyc_ipm, cyc_build, cyc_spmv, cyc_sweep, cyc_pcg_other;
  int64_t cyc_sort, cyc_peel;   /* parts of cyc_build: column sort, Alg. 7 peel */
} alp_frame_stats;

typedef struct {
  int32_t variant;        /* 0 = MALP-A (Alg. 3), 1 = MALP-B                         */
  int32_t precond;        /* 0 = column-wise greedy MTS (Alg. 7, default), 1 = none (plain CG,
                             P:511), 2 = row-wise greedy MTS with diagonal expansion (Alg. 8),
                             3 = incremental greedy MTS (Alg. 6 with the Triangulation Step,
                             Alg. 5; O(q) triangulations per build: a reference variant)  */
  double sigma;           /* centering: mu = sigma * x^T z / q (eq.`update mu`, C-5)   0.1    */
  double eta;             /* step damping of the ratio test (C-6)                0.99   */
  double gap_tol;         /* stop: x^T z <= gap_tol * (1 + |c^T x|) (C-8)               1e-9   */
  double feas_tol;        /* stop: ||r_b||, ||r_c|| <= feas_tol * (1 + ||b||, ||c||)    1e-8   */
  double pcg_rel_tol;     /* PCG acceptance (C-9, G15): the recursive residual
                             ||r||_2 <= pcg_rel_tol ||w||_2 at exit.  Inside the IPM the
                             recursion aims at the forcing term min(pcg_rel_tol, 1e-2 mu)
                             (>= 1e-14, at most 50 iterations past acceptance; DESIGN.md
                             R-1).  ipm_step_pcg additionally refines until the TRUE
                             residual meets it or reaches the fp64 floor          1e-8   */
  double tau_viol;        /* cut violated iff lhs < 1 - tau_viol (C-3)                  1e-6   */
  double tau_act;         /* cut active iff slack <= tau_act (C-4)                      1e-6   */
  double tau_cert;        /* certificate needs g_max <= tau_cert (C-11)                 1e-2   */
  int32_t alp_max_iter;   /* LP cap per frame (C-12), <= 255                            200    */
  int32_t ipm_max_iter;   /* Newton steps per LP (C-8)                                  100    */
  int32_t pcg_max_iter;   /* PCG iterations per Newton step (C-9)                       1000   */
  int32_t warps_per_block;/* tuning: frames (one warp each) per CTA; 0 = automatic             */
  int32_t smem_frames_per_sm; /* tuning: resident frames per SM the shared-memory budget is split
                             over; hot PCG arrays move into shared memory while they fit;
                             0 = automatic (8: measured best, tools/tune_smem.py)          */
  int32_t stop_on_lp_failure; /* 1: a frame stops decoding after an LP whose IPM hit
                             ipm_max_iter (reading C-30; status bit set, last u output)  1      */
  int32_t basis_correction; /* 1: after each Newton step the primal residual rho = r_b - A dx
                             left by an inexact PCG dy is removed on the preconditioner's
                             basis columns (A_M f = rho, dx_M += f; reading C-32)        1      */
  double pcg_forcing;     /* inexact-Newton forcing factor: inside the IPM the PCG recursion
                             aims at min(pcg_rel_tol, pcg_forcing * mu) (R-1); 0 =
                             plain pcg_rel_tol                                         1e-2   */
  int32_t pcg_refine;     /* ipm_step_pcg only: 0 = the PCG recursion alone; 1 = fp64 iterative
                             refinement from the true residual down to the fp64 evaluation floor
                             (round 1); 2 = refinement with double-double residuals until the
                             correction stops shrinking (forward error ~1e-16 vs ~3e-11
                             for 1 at config 5, 1.7x the iterations)                      1      */
} alp_params;

/* Fills the defaults listed above (identical to the oracle's constants). */
void alp_default_params(alp_params* params);

/* Creates a code from its parity-check matrix H (m x n) in check-major CSR:
 * row_ptr (HOST, m+1 entries, row_ptr[0] = 0, nondecreasing), col_idx (HOST, row_ptr[m]
 * entries, 0-based, strictly increasing within each row).  Validation happens on the host
 * before any CUDA call: ALP_ERR_BAD_CODE for range / order / duplicate errors,
 * ALP_ERR_UNSUPPORTED for d_c > 15, d_v > 4 or n + m > 65535, ALP_ERR_CUDA if the device
 * copy cannot be made.  On success *out receives a handle owned by the caller. */
alp_status alp_code_create(int32_t n, int32_t m, const int32_t* row_ptr, const int32_t* col_idx,
                           alp_code** out);
alp_status alp_code_destroy(alp_code* code);

/* Scratch bytes alp_decode needs for n_frames frames with these params (NULL = defaults).
 * Depends on the device's SM count and occupancy (persistent warps), so it queries the
 * current device; returns 0 on error (see alp_last_error). */
size_t alp_decode_workspace_bytes(const alp_code* code, int64_t n_frames, const alp_params* params);

/* Batched LP decoding (Alg. 3).  Inputs: llr (DEVICE, [n_frames][n] fp64),
 * gamma_i = log Pr(r_i | 0) / Pr(r_i | 1) (eq.`def gamma` P:97-101).  Outputs (DEVICE):
 *   hard        [n_frames][n] uint8   u_i > 1/2 of the final LP point u (C-14)
 *   objective   [n_frames] fp64       gamma^T u (C-13)
 *   certificate [n_frames] uint8      1 iff g_max <= tau_cert and H*hard = 0 mod 2 (C-11)
 * Optional outputs (DEVICE, NULL to skip):
 *   frame_status [n_frames] int32 (alp_frame_status bits), stats [n_frames] alp_frame_stats,
 *   u_out [n_frames][n] fp64 final u, y_out [n_frames][m] fp64 duals of the final LP per check
 *   (0 on absent checks), mask_out [n_frames][m] uint16 final cut pool (mask word above).
 * Everything runs on the device in one persistent kernel (no host round trips). */
alp_status alp_decode(const alp_code* code, int64_t n_frames, const double* llr, uint8_t* hard,
                      double* objective, uint8_t* certificate, int32_t* frame_status,
                      alp_frame_stats* stats, double* u_out, double* y_out, uint16_t* mask_out,
                      void* workspace, size_t workspace_bytes, const alp_params* params,
                      void* stream);

/* As alp_decode with HOST buffers (pinned recommended): copies llr to the device, decodes,
 * copies hard / objective / certificate (and frame_status, stats if non-NULL) back, and
 * synchronises `stream`.  Workspace (DEVICE) sized by alp_decode_host_workspace_bytes. */
size_t alp_decode_host_workspace_bytes(const alp_code* code, int64_t n_frames,
                                       const alp_params* params);
alp_status alp_decode_host(const alp_code* code, int64_t n_frames, const double* llr_host,
                           uint8_t* hard_host, double* objective_host, uint8_t* certificate_host,
                           int32_t* frame_status_host, alp_frame_stats* stats_host,
                           void* workspace, size_t workspace_bytes, const alp_params* params,
                           void* stream);

/* Scratch bytes for ipm_step_pcg on n_sys systems (queries the current device). */
size_t alp_pcg_workspace_bytes(const alp_code* code, int64_t n_sys, const alp_params* params);

/* Isolated step-direction solve (eq.`Delta y` P:479) for n_sys independent systems sharing
 * the code's Tanner graph.  For system s: A (p x q, q = n + m) has row j iff masks[s][j]
 * bit 15 is set, with A[j, N(j)[t]] = (bit t ? +1 : -1) * (flip[s][N(j)[t]] ? -1 : +1) and
 * slack A[j, n + j] = +1; Q = A diag(d)^2 A^T.  Inputs (DEVICE):
 *   masks [n_sys][m] uint16; flip [n_sys][n] uint8 or NULL (no flips);
 *   d [n_sys][n + m] fp64 > 0, the diagonal of D (entries of absent slack columns ignored);
 *   r [n_sys][m] fp64 right-hand side (absent rows ignored).
 * Outputs (DEVICE): dy [n_sys][m] (0 on absent rows); optional (NULL to skip):
 *   pcg_iters [n_sys] int32, rel_res [n_sys] fp64 (TRUE ||w - Q dy|| / ||w|| at exit),
 *   sys_status [n_sys] int32 (ALP_FRAME_PCG_* bits),
 *   pivot_rows / pivot_cols [n_sys][m] int32: the preconditioner's pivot sequence
 *   (Alg. 7 pick k: row pivot_rows[s][k], column pivot_cols[s][k] in 0..n+m-1, slack of
 *   row j = n + j), entries k >= p set to -1.  params->precond = 1 runs plain CG. */
alp_status ipm_step_pcg(const alp_code* code, int64_t n_sys, const uint16_t* masks,
                        const uint8_t* flip, const double* d, const double* r, double* dy,
                        int32_t* pcg_iters, double* rel_res, int32_t* sys_status,
                        int32_t* pivot_rows, int32_t* pivot_cols, void* workspace,
                        size_t workspace_bytes, const alp_params* params, void* stream);

/* Diagnostics: when `records` (DEVICE, capacity x 112-byte records {int32 frame, lp, ipm_it,
 * p, status, pcg_iters, back-sweep levels, forward-sweep levels; fp64 true relres, recursive relres, d2_min, d2_max, mu, ||r_b||inf,
 * ||r_c||inf, gap, beta_P, beta_D}) is non-NULL, every subsequent
 * alp_decode appends one record per Newton-step solve (order unspecified, records beyond
 * capacity dropped).  NULL disables.  Process-wide; not thread safe; not for production. */
alp_status alp_debug_trace(void* records, int32_t capacity);

/* Launch plan of alp_decode (step = 0) or ipm_step_pcg (step = 1) for `units` frames / systems
 * on the current device (engineering introspection, used by bench.py to report the residency).
 * info[0] = 1 for the shared-memory window mode, 0 for the generic mode; info[1] = frames
 * (warps) per CTA; info[2] = grid (CTAs); info[3] = shared-memory bytes per frame window;
 * info[4] = shared-memory bytes per CTA; info[5] = global slot bytes per warp.  info: HOST
 * pointer to 6 int32, owned by the caller.  Errors as for alp_decode_workspace_bytes. */
alp_status alp_launch_info(const alp_code* code, int64_t units, const alp_params* params, int32_t step,
                           int32_t* info);

/* Kernel launches enqueued by the last successful alp_decode / ipm_step_pcg on this thread. */
int32_t alp_last_launch_count(void);

const char* alp_status_string(alp_status s);
const char* alp_last_error(void);
/* Thread-local status of the last failing library call (the reason a *_workspace_bytes query
 * returned 0, e.g. ALP_ERR_UNSUPPORTED); ALP_OK after a successful sizing query. */
alp_status alp_last_status(void);
const char* alp_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* ALP_H */
