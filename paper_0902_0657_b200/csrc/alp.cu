// alp.cu — kernels and C ABI of libalp.so (see include/alp.h).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
// One persistent kernel per call: each warp repeatedly claims a frame (atomic counter),
// runs the whole adaptive-LP decode of that frame (Alg. 3 with the IPM of §IV-B and the
// PCG of Alg. 4 preconditioned by Alg. 7) and writes its outputs; no host round trips.
#include <algorithm>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "alp.h"
#include "alp_device.cuh"

namespace alp {

// Optional per-Newton-step trace (alp_debug_trace): one record per step solve.
struct TraceRec {
  int frame, lp, ipm_it, p, status, iters;
  double relres, rec_relres, d2min, d2max, mu, rb, rc, gap, beta_p, beta_d;
};
__device__ TraceRec* g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ int g_trace_n = 0;

struct IpmOut {
  int iters, status, pcg_iters, solves, p4_fail, true_fail;
  double pcg_bytes, max_rec, max_true;
};

// =====================================================================================
// Infeasible primal-dual path-following IPM (§IV-B) on the current pool LP
// min c^T x, A x = b, x >= 0 (q = n + p columns; absent slack columns excluded).
// Start x = z = s0 e, y = 0, s0 = max(1, ||b||, ||c||) (C-7).  Per iteration:
// r_b = b - A x, r_c = c - A^T y - z, gap = x^T z; stop per C-8; mu = sigma gap / q
// (eq.`update mu`, C-5); D^2 = X Z^-1, r_e = mu e - XZe; w = r_b + A (D^2 r_c - Z^-1 r_e)
// (eq.`Delta y`); PCG for dy; dx = D^2 A^T dy - D^2 r_c + Z^-1 r_e (eq.`Delta x`);
// dz = X^-1 (r_e - Z dx) (eq.`Delta z`); ratio test with eta (C-6); update.
// Arrays: v holds r_c then D^2 r_c - Z^-1 r_e then dx; d2 holds D^2 then dz; w holds r_b
// then the PCG right-hand side.
// =====================================================================================
__device__ ALP_HEAVY IpmOut ipm_solve(const Frame& F, const Params& P, const double* g, int p, int nact,
                            double bmax, double cmax, long long frame_id, int lp_id) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const int n = C.n, m = C.m, Q = C.Q, lane = F.lane;
  const double q = (double)(n + p);
  // restrict-qualified views: the arrays never alias, which lets the unrolled loops below
  // issue the next lane-iterations' loads before this one's stores
  double* __restrict__ X = F.x;
  double* __restrict__ Z = F.z;
  double* __restrict__ Y = F.y;
  double* __restrict__ V = F.v;
  const double* __restrict__ B = F.b;
  // (d2, w and dy are shared with build_precond / pcg_solve: plain pointers)
  double* D2 = F.d2;
  double* W = F.w;
  const double* DY = F.dy;
  const uint16_t* __restrict__ SC = F.sgnC;
  const uint8_t* __restrict__ SV = F.sgnV;
  double* __restrict__ RBv = F.rb;   // r_b and r_c of the current iterate (kept for the recovery)
  double* __restrict__ RCv = F.rc;
  const double s0 = fmax(1.0, fmax(bmax, cmax));
  for (int c = lane; c < Q; c += 32) {
    bool valid = (c < n) || (SC[c - n] & PRESENT);
    X[c] = valid ? s0 : 0.0;
    Z[c] = valid ? s0 : 0.0;
  }
  for (int j = lane; j < m; j += 32) Y[j] = 0.0;
  __syncwarp();
  IpmOut out{0, 0, 0, 0, 0, 0, 0.0, 0.0, 0.0};
  long long tk = clock64();
  // algorithmic bytes per PCG iteration of this LP
  const double Bmin = 8.0 * (nact + p) + 48.0 * p + 5.0 * p + 2.0 * m;
  int it = 0;
  while (true) {
    double rbn = 0.0, rcn = 0.0, gap = 0.0, cx = 0.0;
#pragma unroll 4
    for (int j = lane; j < m; j += 32) {
      uint16_t s = SC[j];
      if (!(s & PRESENT)) continue;
      int deg = C.chk_deg[j];
      double acc = B[j] - X[n + j];
      for (int t = 0; t < deg; ++t) {
        double xi = X[chk_nb(C, j, t)];
        acc = ((s >> t) & 1) ? acc + xi : acc - xi;
      }
      W[j] = acc;
      RBv[j] = acc;
      rbn = fmax(rbn, fabs(acc));
      double rc = -Y[j] - Z[n + j];
      V[n + j] = rc;
      RCv[n + j] = rc;
      rcn = fmax(rcn, fabs(rc));
      gap += X[n + j] * Z[n + j];
    }
#pragma unroll 4
    for (int i = lane; i < n; i += 32) {
      double ci = fabs(g[i]);
      uint8_t s = SV[i];
      int dv = C.var_deg[i];
      double acc = ci - Z[i];
      for (int k = 0; k < dv; ++k) {
        if (!((s >> k) & 1)) continue;
        double yj = Y[var_ck(C, i, k)];
        acc = ((s >> (4 + k)) & 1) ? acc + yj : acc - yj;
      }
      V[i] = acc;
      RCv[i] = acc;
      rcn = fmax(rcn, fabs(acc));
      double xi = X[i];
      gap += xi * Z[i];
      cx += ci * xi;
    }
    __syncwarp();
    rbn = wmax(rbn);
    rcn = wmax(rcn);
    gap = wsum(gap);
    cx = wsum(cx);
    if (gap <= P.gap_tol * (1.0 + fabs(cx)) && rbn <= P.feas_tol * (1.0 + bmax) &&
        rcn <= P.feas_tol * (1.0 + cmax))
      break;
    if (it >= P.ipm_max_iter) {
      out.status |= ST_IPM_MAXITER;
      break;
    }
    const double mu = P.sigma * gap / q;
#pragma unroll 4
    for (int c = lane; c < Q; c += 32) {
      if (c >= n && !(SC[c - n] & PRESENT)) continue;
      double xc = X[c], zc = Z[c];
      const double iz = 1.0 / zc;   // one division for D^2 = X Z^-1 and Z^-1 r_e
      double d2 = xc * iz;
      double re = mu - xc * zc;
      D2[c] = d2;
      V[c] = d2 * V[c] - re * iz;
    }
    __syncwarp();
#pragma unroll 4
    for (int j = lane; j < m; j += 32) {
      uint16_t s = SC[j];
      if (!(s & PRESENT)) continue;
      int deg = C.chk_deg[j];
      double acc = W[j] + V[n + j];
      for (int t = 0; t < deg; ++t) {
        double vi = V[chk_nb(C, j, t)];
        acc = ((s >> t) & 1) ? acc - vi : acc + vi;
      }
      W[j] = acc;
    }
    __syncwarp();
    int nLb = 0, nLf = 0;
    const bool mtm = (P.precond == 0);
    ALP_TICK(F, CY_IPM, tk);
    // the Alg. 7 triangular set is both the PCG preconditioner (precond = 0) and the basis of
    // the step's feasibility correction (C-32), so plain CG builds it too when that is on
    if (mtm || P.basis_correction) build_precond(F, p, nLb, nLf);
    ALP_TICK(F, CY_BUILD, tk);
    // inexact-Newton forcing term (R-1): the dual step needs A^T dy accurate to well
    // below z ~ mu on the basic columns, so late in the IPM the recursion aims at
    // min(pcg_rel_tol, 1e-2 mu) (floored at 1e-14); P4 acceptance is pcg_rel_tol.  An inexact
    // dy is admissible because the recovery below keeps every KKT row but the complementarity
    // of the basis columns exact (C-32).
    const double inner = fmin(P.pcg_rel_tol, fmax(1e-14, P.pcg_forcing * mu));
    PcgResult pr = pcg_solve(F, P, mtm ? PC_MTS : PC_NONE, nLb, nLf, inner, false);
    tk = clock64();
    out.status |= pr.status;
    out.solves += 1;
    out.p4_fail += (pr.status != 0) ? 1 : 0;
    out.true_fail += (pr.relres > P.pcg_rel_tol) ? 1 : 0;
    out.max_rec = fmax(out.max_rec, pr.rec_relres);
    out.max_true = fmax(out.max_true, pr.relres);
    double dmn = 1e308, dmx = 0.0;
    if (g_trace) {
      for (int c = lane; c < Q; c += 32) {
        if (c >= n && !(SC[c - n] & PRESENT)) continue;
        dmn = fmin(dmn, D2[c]);
        dmx = fmax(dmx, D2[c]);
      }
      dmn = wmin(dmn);
      dmx = wmax(dmx);
    }
    out.pcg_iters += pr.iters;
    out.pcg_bytes += (double)pr.iters * Bmin;
    // Newton recovery (eq.`Delta x`, eq.`Delta z` P:480-481).  dz is taken in the algebraically
    // identical form dz = r_c - A^T dy (eliminate dx from eq.`Delta z`), which keeps the dual
    // equation A^T(y+dy) + z + dz = c exact for ANY dy; with dx from eq.`Delta x` the
    // complementarity row Z dx + X dz = r_e is then exact too, so an inexact PCG dy only leaves
    // the primal row off by the step residual rho = r_b - A dx = w - Q dy.  That residual is
    // moved onto the preconditioner's basis columns: A_M f = rho (the back sweep of P:585),
    // dx_M += f, so A dx = r_b holds to rounding (reading C-32; R-1).
#pragma unroll 4
    for (int i = lane; i < n; i += 32) {
      uint8_t s = SV[i];
      int dv = C.var_deg[i];
      double atdy = 0.0;
      for (int k = 0; k < dv; ++k) {
        if (!((s >> k) & 1)) continue;
        double d = DY[var_ck(C, i, k)];
        atdy = ((s >> (4 + k)) & 1) ? atdy - d : atdy + d;
      }
      const double dx = D2[i] * atdy - V[i];
      V[i] = dx;
      D2[i] = RCv[i] - atdy;   // dz
    }
    for (int j = lane; j < m; j += 32) {
      if (!(SC[j] & PRESENT)) continue;
      const int c = n + j;
      const double dx = D2[c] * DY[j] - V[c];
      V[c] = dx;
      D2[c] = RCv[c] - DY[j];
    }
    __syncwarp();
    if (P.basis_correction && nLb > 0) {
      double* rS = F.S<double>(F.L->s_r);
      const double* fS = F.S<double>(F.L->s_f);
      for (int j = lane; j < m; j += 32) {
        uint16_t s = SC[j];
        double rho = 0.0;
        if (s & PRESENT) {
          int deg = C.chk_deg[j];
          double acc = RBv[j] - V[n + j];
          for (int t = 0; t < deg; ++t) {
            double xi = V[chk_nb(C, j, t)];
            acc = ((s >> t) & 1) ? acc + xi : acc - xi;
          }
          rho = acc;
        }
        rS[j] = rho;
      }
      __syncwarp();
      back_sweep(F, nLb);   // f = A_M^-1 rho, f_R = component of row R's pivot column
      __syncwarp();
      for (int j = lane; j < m; j += 32) {
        const uint16_t c = F.pcolR[j];
        if (c != NONE16) V[c] += fS[j];
      }
      __syncwarp();
    }
    // ratio test (C-6)
    double ax = 1e308, az = 1e308;
#pragma unroll 4
    for (int c = lane; c < Q; c += 32) {
      if (c >= n && !(SC[c - n] & PRESENT)) continue;
      const double dx = V[c], dz = D2[c];
      if (dx < 0.0) ax = fmin(ax, -X[c] / dx);
      if (dz < 0.0) az = fmin(az, -Z[c] / dz);
    }
    ax = wmin(ax);
    az = wmin(az);
    const double bP = fmin(1.0, P.eta * ax);
    const double bD = fmin(1.0, P.eta * az);
    if (g_trace) {
      if (lane == 0) {
        int slot = atomicAdd(&g_trace_n, 1);
        if (slot < g_trace_cap)
          g_trace[slot] = TraceRec{(int)frame_id, lp_id, it, p, pr.status, pr.iters, pr.relres, pr.rec_relres, dmn, dmx, mu, rbn, rcn, gap, bP, bD};
      }
    }
    bool bad = false;
#pragma unroll 4
    for (int c = lane; c < Q; c += 32) {
      if (c >= n && !(SC[c - n] & PRESENT)) continue;
      double xn = X[c] + bP * V[c];
      double zn = Z[c] + bD * D2[c];
      X[c] = xn;
      Z[c] = zn;
      bad |= !isfinite(xn) || !isfinite(zn);
    }
    for (int j = lane; j < m; j += 32) {
      if (!(SC[j] & PRESENT)) continue;
      double yn = Y[j] + bD * DY[j];
      Y[j] = yn;
      bad |= !isfinite(yn);
    }
    __syncwarp();
    ++it;
    if (__any_sync(FULL, bad)) {
      out.status |= ST_NUMERIC;
      break;
    }
  }
  ALP_TICK(F, CY_IPM, tk);
  out.iters = it;
  return out;
}

struct DecodeOut {
  uint8_t* hard;
  double* objective;
  uint8_t* cert;
  int* status;
  alp_frame_stats* stats;
  double* u_out;
  double* y_out;
  uint16_t* mask_out;
};

// MALP-A / MALP-B decode of one frame (Alg. 3; outputs P:143, C-11..C-15).
__device__ void decode_frame(Frame& F, const Params& P, const double* g, long long f,
                             const DecodeOut& O) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const int n = C.n, m = C.m, lane = F.lane;
  double cm = 0.0;
  for (int i = lane; i < n; i += 32) {
    double gi = g[i];
    uint8_t fl = gi < 0.0;  // eq.`initial constraints` P:147-155: u^0 = hard decision
    F.flip[i] = fl;
    F.u[i] = fl ? 1.0 : 0.0;
    cm = fmax(cm, fabs(gi));
  }
  for (int j = lane; j < m; j += 32) {
    F.mask[j] = 0;
    F.y[j] = 0.0;
  }
  const double cmax = wmax(cm);
  __syncwarp();
  int status = 0, lp_solves = 0, ipm_iters = 0, pcg_iters = 0, max_p = 0;
  int solves = 0, p4_fail = 0, true_fail = 0;
  double max_rec = 0.0, max_true = 0.0;
  bool last_lp_bad = false;   // the last solved LP did not converge (IPM cap / non-finite)
  double pcg_bytes = 0.0;
  if (lane < 8) F.cyc[lane] = 0;
  __syncwarp();
  long long tk = clock64();
  for (int k = 0;; ++k) {
    bool changed = cut_search(F, P);
    if (!changed) break;
    if (k == P.alp_max_iter) {
      status |= ST_ALP_MAXITER;
      break;
    }
    // Reading C-12: the LP (hence u^k and the next cut search) is a function of the pool, so
    // a pool equal to that of an LP already solved repeats forever: stop with the last solved
    // u (G2) and the cap status.  Pools are compared by a 64-bit order-independent hash.
    {
      unsigned long long hsh = 0ull;
      for (int j = lane; j < m; j += 32) {
        unsigned long long v = ((unsigned long long)(unsigned)j << 16) | F.mask[j];
        v *= 0x9E3779B97F4A7C15ull;
        v ^= v >> 29;
        v *= 0xBF58476D1CE4E5B9ull;
        v ^= v >> 32;
        hsh += (F.mask[j] & PRESENT) ? v : 0ull;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) hsh += __shfl_xor_sync(FULL, hsh, o);
      bool seen = false;
      for (int t = lane; t < k; t += 32) seen |= (F.hist[t] == hsh);
      if (__any_sync(FULL, seen)) {
        status |= ST_ALP_MAXITER;
        break;
      }
      if (lane == 0) F.hist[k] = hsh;
      __syncwarp();
    }
    int p, nact;
    double bmax;
    build_signs(F, true, p, nact, bmax);
    ALP_TICK(F, CY_CUT, tk);
    ++lp_solves;
    max_p = max(max_p, p);
    IpmOut o = ipm_solve(F, P, g, p, nact, bmax, cmax, f, lp_solves);
    status |= o.status;
    last_lp_bad = (o.status & (ST_IPM_MAXITER | ST_NUMERIC)) != 0;
    ipm_iters += o.iters;
    pcg_iters += o.pcg_iters;
    pcg_bytes += o.pcg_bytes;
    solves += o.solves;
    p4_fail += o.p4_fail;
    true_fail += o.true_fail;
    max_rec = fmax(max_rec, o.max_rec);
    max_true = fmax(max_true, o.max_true);
    for (int i = lane; i < n; i += 32) {
      double xi = F.x[i];
      F.u[i] = F.flip[i] ? 1.0 - xi : xi;
    }
    __syncwarp();
    tk = clock64();
    // Reading C-30: an LP whose IPM ended on a non-finite iterate or at the Newton-step cap
    // gives no trustworthy u for the next cut search, so the frame's decode stops there
    // (status bits set, last u output; `stop_on_lp_failure = 0` keeps going).
    if ((o.status & ST_NUMERIC) || (P.stop_on_lp_failure && (o.status & ST_IPM_MAXITER))) break;
  }
  ALP_TICK(F, CY_CUT, tk);
  // outputs: hard decision, objective gamma^T u, g_max, ML certificate
  double obj = 0.0, gm = 0.0;
  for (int i = lane; i < n; i += 32) {
    double ui = F.u[i];
    obj += g[i] * ui;
    gm = fmax(gm, fmin(ui, 1.0 - ui));
    O.hard[f * n + i] = (ui > 0.5) ? 1 : 0;
    if (O.u_out) O.u_out[f * n + i] = ui;
  }
  bool parity_bad = false;
  for (int j = lane; j < m; j += 32) {
    int deg = C.chk_deg[j];
    int par = 0;
    for (int t = 0; t < deg; ++t) par ^= (F.u[chk_nb(C, j, t)] > 0.5) ? 1 : 0;
    parity_bad |= (par != 0);
    uint16_t mk = F.mask[j];
    if (O.y_out) O.y_out[f * m + j] = (mk & PRESENT) ? F.y[j] : 0.0;
    if (O.mask_out) O.mask_out[f * m + j] = mk;
  }
  obj = wsum(obj);
  gm = wmax(gm);
  bool pbad = __any_sync(FULL, parity_bad);
  if (lane == 0) {
    O.objective[f] = obj;
    // ML certificate (C-11): an integral codeword that is the optimum of the LP; an LP
    // whose IPM did not converge proves nothing, so its u never certifies (C-31)
    O.cert[f] = (gm <= P.tau_cert && !pbad && !last_lp_bad) ? 1 : 0;
    if (O.status) O.status[f] = status;
    if (O.stats) {
      alp_frame_stats st;
      st.lp_solves = lp_solves;
      st.ipm_iters = ipm_iters;
      st.pcg_iters = pcg_iters;
      st.max_p = max_p;
      st.pcg_solves = solves;
      st.pcg_p4_fail = p4_fail;
      st.pcg_true_fail = true_fail;
      st.reserved = 0;
      st.max_rec_relres = max_rec;
      st.max_true_relres = max_true;
      st.g_max = gm;
      st.pcg_bytes = pcg_bytes;
      st.cyc_cut = F.cyc[CY_CUT];
      st.cyc_ipm = F.cyc[CY_IPM];
      st.cyc_build = F.cyc[CY_BUILD];
      st.cyc_spmv = F.cyc[CY_SPMV];
      st.cyc_sweep = F.cyc[CY_SWEEP];
      st.cyc_pcg_other = F.cyc[CY_PCG];
      st.cyc_sort = F.cyc[CY_SORT];
      st.cyc_peel = F.cyc[CY_PEEL];
      O.stats[f] = st;
    }
  }
  __syncwarp();
}

#ifndef ALP_MINB
#define ALP_MINB 1
#endif
__global__ void __launch_bounds__(128, ALP_MINB) alp_decode_kernel(DCode C, Params P, Layout L, GraphSmem G,
                                                        char* slots,
                                                        const double* __restrict__ llr,
                                                        long long n_frames, DecodeOut O,
                                                        unsigned long long* counter) {
  extern __shared__ __align__(16) char smem[];
  __shared__ DCode sC;    // code / layout descriptors in shared memory: the Frame's pointers to
  __shared__ Layout sL;   // them must not land in local memory
  if (threadIdx.x == 0) sL = L;
  DCode Cs;
  stage_graph(C, G, smem, Cs);
  if (threadIdx.x == 0) sC = Cs;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  Frame F;
  char* slot = slots + gw * L.slot_bytes;
  frame_bind(F, &sC, &sL, slot, L.win_global ? slot + L.g_win : smem + G.bytes + warp * L.smem_bytes, lane);
  __shared__ long long s_cyc[4][8];   // phase clocks in shared memory (a global RMW per tick
  F.cyc = s_cyc[warp];                // would stall the warp on an L2 round trip)
  while (true) {
    long long f = 0;
    if (lane == 0) f = (long long)atomicAdd(counter, 1ull);   // 64-bit: no wrap at any n_frames
    f = __shfl_sync(FULL, f, 0);
    if (f >= n_frames) break;
    decode_frame(F, P, llr + f * C.n, f, O);
  }
}

struct StepIO {
  const uint16_t* masks;
  const uint8_t* flip;
  const double* d;
  const double* r;
  double* dy;
  int* iters;
  double* relres;
  int* status;
  int* prow;
  int* pcol;
};

// Isolated step solve (eq.`Delta y` P:479) per system: signs, D^2, Alg. 7, PCG.
__global__ void __launch_bounds__(128) pcg_step_kernel(DCode C, Params P, Layout L, GraphSmem G,
                                                      char* slots, long long n_sys, StepIO io,
                                                      unsigned long long* counter) {
  extern __shared__ __align__(16) char smem[];
  __shared__ DCode sC;
  __shared__ Layout sL;
  if (threadIdx.x == 0) sL = L;
  DCode Cs;
  stage_graph(C, G, smem, Cs);
  if (threadIdx.x == 0) sC = Cs;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  Frame F;
  char* slot = slots + gw * L.slot_bytes;
  frame_bind(F, &sC, &sL, slot, L.win_global ? slot + L.g_win : smem + G.bytes + warp * L.smem_bytes, lane);
  const int n = C.n, m = C.m, Q = C.Q;
  while (true) {
    long long s = 0;
    if (lane == 0) s = (long long)atomicAdd(counter, 1ull);
    s = __shfl_sync(FULL, s, 0);
    if (s >= n_sys) break;
    for (int j = lane; j < m; j += 32) F.mask[j] = io.masks[s * m + j];
    for (int i = lane; i < n; i += 32) F.flip[i] = io.flip ? (io.flip[s * n + i] ? 1 : 0) : 0;
    __syncwarp();
    int p, nact;
    double bmax;
    build_signs(F, false, p, nact, bmax);
    for (int c = lane; c < Q; c += 32) {
      double dd = io.d[s * Q + c];
      F.d2[c] = dd * dd;
    }
    for (int j = lane; j < m; j += 32) F.w[j] = (F.sgnC[j] & PRESENT) ? io.r[s * m + j] : 0.0;
    __syncwarp();
    int nLb = 0, nLf = 0;
    const bool mtm = (P.precond == 0) && p > 0;
    if (mtm) build_precond(F, p, nLb, nLf);
    if ((io.prow || io.pcol)) {
      if (mtm) write_pivots(F, p, io.prow ? io.prow + s * m : nullptr, io.pcol ? io.pcol + s * m : nullptr);
      else
        for (int k = lane; k < m; k += 32) {
          if (io.prow) io.prow[s * m + k] = -1;
          if (io.pcol) io.pcol[s * m + k] = -1;
        }
    }
    PcgResult pr = pcg_solve(F, P, mtm ? PC_MTS : PC_NONE, nLb, nLf, P.pcg_rel_tol, true);
    for (int j = lane; j < m; j += 32) io.dy[s * m + j] = (F.sgnC[j] & PRESENT) ? F.dy[j] : 0.0;
    if (lane == 0) {
      if (io.iters) io.iters[s] = pr.iters;
      if (io.relres) io.relres[s] = pr.relres;
      if (io.status) io.status[s] = pr.status;
    }
    __syncwarp();
  }
}

}  // namespace alp

// =====================================================================================
// Host side
// =====================================================================================
using namespace alp;

struct alp_code {
  int n, m, dc, dv, E;
  uint16_t* d_chk_var;
  uint8_t* d_chk_deg;
  uint16_t* d_var_chk;
  uint8_t* d_var_slot;
  uint8_t* d_var_deg;
};

namespace {
thread_local std::string g_last_error;
thread_local alp_status g_last_status = ALP_OK;
thread_local int g_last_launches = 0;

alp_status fail(alp_status s, const std::string& msg) {
  g_last_error = msg;
  g_last_status = s;
  return s;
}
alp_status cuda_fail(cudaError_t e, const char* what) {
  return fail(ALP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
size_t al(size_t x, size_t a = 16) { return (x + a - 1) / a * a; }

DCode make_dcode(const alp_code* c) {
  DCode C;
  C.n = c->n;
  C.m = c->m;
  C.dc = c->dc;
  C.dv = c->dv;
  C.Q = c->n + c->m;
  C.W = (C.Q + 63) / 64;
  C.RB = (c->dc + 1 <= 8) ? 8 : 16;   // back-record u16 words: head + <= d_c - 1 deps
  C.chk_var = c->d_chk_var;
  C.chk_deg = c->d_chk_deg;
  C.var_chk = c->d_var_chk;
  C.var_slot = c->d_var_slot;
  C.var_deg = c->d_var_deg;
  return C;
}

Layout make_layout(const DCode& C, int smem_budget) {
  Layout L;
  const size_t n = C.n, m = C.m, Q = C.Q;
  size_t o = 0;
  auto g = [&](size_t bytes) {
    size_t r = o;
    o += al(bytes, 128);
    return (long long)r;
  };
  L.g_cyc = g(8 * 8);
  L.g_x = g(8 * Q);
  L.g_z = g(8 * Q);
  L.g_d2 = g(8 * Q);
  L.g_v = g(8 * Q);
  L.g_y = g(8 * m);
  L.g_dy = g(8 * m);
  L.g_l = g(8 * m);
  L.g_w = g(8 * m);
  L.g_u = g(8 * n);
  L.g_b = g(8 * m);
  L.g_dinvF = g(8 * m);
  L.g_recB = g(2 * m * C.RB);
  L.g_recF = g(2 * m * RF);
  L.g_offB = g(4 * (m + 2));
  L.g_offF = g(4 * (m + 2));
  L.g_sgnC = g(2 * m);
  L.g_mask = g(2 * m);
  L.g_hist = g(8 * 256);
  L.g_sgnV = g(n);
  L.g_flip = g(n);
  L.g_rb = g(8 * m);
  L.g_rc = g(8 * Q);
  L.g_pcol = g(2 * m);
  L.slot_bytes = (long long)al(o, 256);
  // shared window
  size_t a = 0;
  auto s = [&](size_t bytes) {
    size_t r = a;
    a += al(bytes, 16);
    return (int)r;
  };
  L.s_order = s(2 * Q);
  // sort phase (radix buffers kA/kB u32[Q], cA/cB u16[Q], 256-bin histogram) after `order`
  const size_t sort_base = a;
  L.s_sortk = (int)sort_base;
  L.s_sorth = (int)(sort_base + al(12 * Q, 16));
  const size_t s_sort = sort_base + al(12 * Q, 16) + 2048;
  a = sort_base;
  L.s_rank = s(2 * Q);
  L.s_cnt = s(Q);
  L.s_xr = s(2 * Q);
  L.s_bm = s(8 * (size_t)C.W);
  L.RS = (C.dc + 1 <= 8) ? 8 : 16;
  L.s_rrank = s(2 * (size_t)m * L.RS);
  L.s_pos = s(2 * m);
  L.s_pcol = s(2 * m);
  L.s_prow = s(2 * m);
  L.s_lvB = s(2 * m);
  L.s_lvF = s(2 * m);
  size_t end_peel = a;
  L.s_poc = L.s_order;  // order/rank are dead after the peel
  // hist/cur over cnt/xr/bm if they fit there, else after the peel arrays
  size_t need = 2 * al(4 * (m + 2), 16);
  if ((size_t)L.s_cnt + need <= (size_t)L.s_pos) {
    L.s_hist = L.s_cnt;
    L.s_cur = L.s_cnt + (int)al(4 * (m + 2), 16);
  } else {
    L.s_hist = (int)end_peel;
    L.s_cur = (int)(end_peel + al(4 * (m + 2), 16));
    end_peel += need;
  }
  // PCG phase
  a = 0;
  L.s_h = s(8 * m);
  L.s_r = s(8 * m);
  L.s_f = s(8 * m);
  L.s_z = s(8 * m);
  size_t end_pcg = a;
  if (8 * n <= end_pcg - L.s_f) {
    L.s_t = L.s_f;  // t (per variable) aliases f and z (dead during the SpMV)
  } else {
    L.s_t = s(8 * n);
    end_pcg = a;
  }
  size_t tot = al(std::max(s_sort, std::max(end_peel, end_pcg)), 16);
  L.win_global = 0;
  L.g_win = 0;
  if ((long long)tot > 200 * 1024) {
    // large code: the whole phase window goes to the slot (global memory, L2-cached), nothing
    // is relocated, and the kernel needs no per-frame shared memory
    L.win_global = 1;
    L.g_win = (long long)al(o, 256);
    L.slot_bytes = (long long)al(L.g_win + tot, 256);
    L.smask = 0;
    L.smem_bytes = 0;
    return L;
  }
  // Relocate the arrays the PCG loop touches every iteration into the shared window, by
  // priority (sign tables, l, dy, sweep program, D^2, w), while the window fits the budget.
  L.smask = 0;
  size_t rel_bytes[RL_N];
  rel_bytes[RL_SGNC] = 2 * m;
  rel_bytes[RL_SGNV] = n;
  rel_bytes[RL_L] = 8 * m;
  rel_bytes[RL_DY] = 8 * m;
  rel_bytes[RL_DINVF] = 8 * m;
  rel_bytes[RL_OFFB] = 4 * (m + 2);
  rel_bytes[RL_OFFF] = 4 * (m + 2);
  rel_bytes[RL_RECF] = 2 * m * (size_t)RF;
  rel_bytes[RL_RECB] = 2 * m * (size_t)C.RB;
  rel_bytes[RL_D2] = 8 * Q;
  rel_bytes[RL_W] = 8 * m;
  for (int k = 0; k < RL_N; ++k) {
    size_t need = al(rel_bytes[k], 16);
    if ((long long)(tot + need) > (long long)smem_budget) continue;
    L.smask |= 1u << k;
    L.soff[k] = (int)tot;
    tot += need;
  }
  L.smem_bytes = (int)al(tot, 128);
  return L;
}

GraphSmem make_graph_smem(const DCode& C) {
  GraphSmem G;
  size_t o = 0;
  auto a = [&](size_t bytes) {
    size_t r = o;
    o += al(bytes, 16);
    return (int)r;
  };
  G.o_chk_var = a(2 * (size_t)C.m * C.dc);
  G.o_chk_deg = a(C.m);
  G.o_var_chk = a(2 * (size_t)C.n * C.dv);
  G.o_var_slot = a((size_t)C.n * C.dv);
  G.o_var_deg = a(C.n);
  G.bytes = (int)al(o, 128);
  if (G.bytes > 48 * 1024) G = GraphSmem{0, 0, 0, 0, 0, 0};   // large codes: graph stays global
  return G;
}

// Shared-memory budget per warp (frame): the device's per-block opt-in limit split over
// `frames_per_sm` resident frames.
int smem_budget_for(const alp_params* p) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
    optin = 227 * 1024;
  // measured (tools/tune_smem.py, C2 3.0 dB, round 2): 8 beats 11 by ~25 % — the PCG vectors
  // and sweep programs then live in shared memory, worth more than the L1 the window takes
  int fps = (p && p->smem_frames_per_sm > 0) ? p->smem_frames_per_sm : 8;
  return (optin / fps) & ~127;
}

Params make_params(const alp_params* p) {
  alp_params d;
  alp_default_params(&d);
  if (!p) p = &d;
  Params P;
  P.variant = p->variant;
  P.precond = p->precond;
  P.sigma = p->sigma;
  P.eta = p->eta;
  P.gap_tol = p->gap_tol;
  P.feas_tol = p->feas_tol;
  P.pcg_rel_tol = p->pcg_rel_tol;
  P.stop_on_lp_failure = p->stop_on_lp_failure;
  P.basis_correction = p->basis_correction;
  P.pcg_forcing = p->pcg_forcing;
  P.tau_viol = p->tau_viol;
  P.tau_act = p->tau_act;
  P.tau_cert = p->tau_cert;
  P.alp_max_iter = p->alp_max_iter;
  P.ipm_max_iter = p->ipm_max_iter;
  P.pcg_max_iter = p->pcg_max_iter;
  return P;
}

alp_status check_params(const alp_params* p) {
  if (!p) return ALP_OK;
  if (p->variant < 0 || p->variant > 1) return fail(ALP_ERR_INVALID_ARG, "params.variant must be 0 or 1");
  if (p->precond < 0 || p->precond > 1) return fail(ALP_ERR_INVALID_ARG, "params.precond must be 0 or 1");
  if (!(p->sigma > 0 && p->sigma < 1) || !(p->eta > 0 && p->eta < 1))
    return fail(ALP_ERR_INVALID_ARG, "params.sigma and params.eta must lie in (0,1)");
  if (p->alp_max_iter < 0 || p->alp_max_iter > 255 || p->ipm_max_iter < 0 || p->pcg_max_iter < 1)
    return fail(ALP_ERR_INVALID_ARG, "iteration caps: 0 <= alp_max_iter <= 255, ipm >= 0, pcg >= 1");
  if (p->warps_per_block < 0 || p->warps_per_block > 4 || p->smem_frames_per_sm < 0 || p->smem_frames_per_sm > 32)
    return fail(ALP_ERR_INVALID_ARG, "params.warps_per_block must be 0..4, smem_frames_per_sm 0..32");
  return ALP_OK;
}

template <class K>
cudaError_t raise_smem_optin(K kernel, int dev, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;   // (kernel, device) pairs already set
  std::lock_guard<std::mutex> lk(mu);
  const void* key = reinterpret_cast<const void*>(kernel);
  for (auto& d : done)
    if (d.first == key && d.second == dev) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(key, dev);
  return e;
}

struct LaunchCfg {
  int wpb, grid, smem_block;
  long long slots;
};

template <class K>
alp_status plan_launch(K kernel, const Layout& L, int graph_bytes, long long units, const alp_params* p,
                       LaunchCfg& cfg) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int sms = 0, smem_optin = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  smem_optin -= 1024;   // static shared memory of the kernels (code / layout descriptors)
  int wpb = (p && p->warps_per_block > 0) ? p->warps_per_block : 4;
  while (wpb > 1 && (long long)wpb * L.smem_bytes + graph_bytes > smem_optin) --wpb;
  if ((long long)wpb * L.smem_bytes + graph_bytes > smem_optin)
    return fail(ALP_ERR_UNSUPPORTED, "per-frame shared memory " + std::to_string(L.smem_bytes) +
                                         " B exceeds the device limit");
  int smem_block = wpb * L.smem_bytes + graph_bytes;
  // The dynamic shared-memory opt-in is raised once per (kernel, device) to the device maximum,
  // never lowered per call: concurrent calls with different tuning params then cannot undo
  // each other's attribute between set and launch (include/alp.h thread-safety note).
  e = raise_smem_optin(kernel, dev, smem_optin);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  int nb = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, 32 * wpb, smem_block);
  if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  if (nb < 1) return fail(ALP_ERR_UNSUPPORTED, "kernel cannot be resident with this shared memory");
  long long blocks = (long long)nb * sms;
  long long need = (units + wpb - 1) / wpb;
  if (need < 1) need = 1;
  cfg.wpb = wpb;
  cfg.grid = (int)std::min(blocks, need);
  cfg.smem_block = smem_block;
  cfg.slots = (long long)cfg.grid * wpb;
  return ALP_OK;
}

const size_t kCounterBytes = 256;

}  // namespace

extern "C" {

void alp_default_params(alp_params* p) {
  if (!p) return;
  p->variant = 0;
  p->precond = 0;
  p->sigma = 0.1;
  p->eta = 0.99;
  p->gap_tol = 1e-9;
  p->feas_tol = 1e-8;
  p->pcg_rel_tol = 1e-8;
  p->tau_viol = 1e-6;
  p->tau_act = 1e-6;
  p->tau_cert = 1e-2;
  p->alp_max_iter = 200;
  p->ipm_max_iter = 100;
  p->pcg_max_iter = 1000;
  p->warps_per_block = 0;
  p->smem_frames_per_sm = 0;
  p->stop_on_lp_failure = 1;
  p->basis_correction = 1;
  p->pcg_forcing = 1e-2;
}

const char* alp_status_string(alp_status s) {
  switch (s) {
    case ALP_OK: return "ALP_OK";
    case ALP_ERR_INVALID_ARG: return "ALP_ERR_INVALID_ARG";
    case ALP_ERR_BAD_CODE: return "ALP_ERR_BAD_CODE";
    case ALP_ERR_UNSUPPORTED: return "ALP_ERR_UNSUPPORTED";
    case ALP_ERR_CUDA: return "ALP_ERR_CUDA";
    case ALP_ERR_WORKSPACE: return "ALP_ERR_WORKSPACE";
  }
  return "ALP_ERR_UNKNOWN";
}

const char* alp_last_error(void) { return g_last_error.c_str(); }

alp_status alp_last_status(void) { return g_last_status; }

const char* alp_build_info(void) {
  return "libalp: sm_100a, warp-per-frame persistent kernels, fp64";
}

int32_t alp_last_launch_count(void) { return g_last_launches; }

alp_status alp_debug_trace(void* records, int32_t capacity) {
  void* ptr = records;
  int cap = records ? capacity : 0, zero = 0;
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &ptr, sizeof(ptr));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_n, &zero, sizeof(zero));
  return e == cudaSuccess ? ALP_OK : cuda_fail(e, "alp_debug_trace");
}

alp_status alp_code_create(int32_t n, int32_t m, const int32_t* row_ptr, const int32_t* col_idx,
                           alp_code** out) {
  if (!out) return fail(ALP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n <= 0 || m <= 0) return fail(ALP_ERR_INVALID_ARG, "n and m must be positive");
  if (!row_ptr || !col_idx) return fail(ALP_ERR_INVALID_ARG, "row_ptr / col_idx is NULL");
  if (row_ptr[0] != 0) return fail(ALP_ERR_BAD_CODE, "row_ptr[0] must be 0");
  int dc = 0;
  for (int j = 0; j < m; ++j) {
    int a = row_ptr[j], b = row_ptr[j + 1];
    if (b < a) return fail(ALP_ERR_BAD_CODE, "row_ptr must be nondecreasing");
    if (b - a == 0) return fail(ALP_ERR_BAD_CODE, "check " + std::to_string(j) + " has no variable");
    dc = std::max(dc, b - a);
    for (int t = a; t < b; ++t) {
      if (col_idx[t] < 0 || col_idx[t] >= n)
        return fail(ALP_ERR_BAD_CODE, "col_idx out of range in check " + std::to_string(j));
      if (t > a && col_idx[t] <= col_idx[t - 1])
        return fail(ALP_ERR_BAD_CODE, "col_idx not strictly increasing in check " + std::to_string(j));
    }
  }
  const int E = row_ptr[m];
  std::vector<int> vdeg(n, 0);
  for (int t = 0; t < E; ++t) vdeg[col_idx[t]]++;
  int dv = 0;
  for (int i = 0; i < n; ++i) dv = std::max(dv, vdeg[i]);
  if (dc > DCMAX) return fail(ALP_ERR_UNSUPPORTED, "check degree > 15");
  if (dv > DVMAX) return fail(ALP_ERR_UNSUPPORTED, "variable degree > 4");
  if ((long long)n + m > 65535) return fail(ALP_ERR_UNSUPPORTED, "n + m > 65535");
  if (m > 32767) return fail(ALP_ERR_UNSUPPORTED, "m > 32767 (15-bit row ids in the sweep records)");
  if (dv == 0) dv = 1;
  std::vector<uint16_t> chk_var((size_t)m * dc, 0xffff), var_chk((size_t)n * dv, 0xffff);
  std::vector<uint8_t> chk_deg(m), var_slot((size_t)n * dv, 0), var_deg(n, 0);
  for (int j = 0; j < m; ++j) {
    int a = row_ptr[j], b = row_ptr[j + 1];
    chk_deg[j] = (uint8_t)(b - a);
    for (int t = a; t < b; ++t) {
      int i = col_idx[t];
      chk_var[(size_t)j * dc + (t - a)] = (uint16_t)i;
      int k = var_deg[i]++;
      var_chk[(size_t)i * dv + k] = (uint16_t)j;
      var_slot[(size_t)i * dv + k] = (uint8_t)(t - a);
    }
  }
  alp_code* c = new alp_code();
  c->n = n;
  c->m = m;
  c->dc = dc;
  c->dv = dv;
  c->E = E;
  cudaError_t e;
  auto up = [&](void** dst, const void* src, size_t bytes) -> bool {
    const size_t padded = al(bytes, 16);   // the kernels stage these arrays with 4-byte loads
    e = cudaMalloc(dst, padded);
    if (e != cudaSuccess) return false;
    e = cudaMemset(*dst, 0, padded);
    if (e != cudaSuccess) return false;
    e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    return e == cudaSuccess;
  };
  c->d_chk_var = nullptr;
  c->d_chk_deg = c->d_var_slot = c->d_var_deg = nullptr;
  c->d_var_chk = nullptr;
  bool ok = up((void**)&c->d_chk_var, chk_var.data(), chk_var.size() * 2) &&
            up((void**)&c->d_chk_deg, chk_deg.data(), chk_deg.size()) &&
            up((void**)&c->d_var_chk, var_chk.data(), var_chk.size() * 2) &&
            up((void**)&c->d_var_slot, var_slot.data(), var_slot.size()) &&
            up((void**)&c->d_var_deg, var_deg.data(), var_deg.size());
  if (!ok) {
    alp_status st = cuda_fail(e, "alp_code_create device copy");
    alp_code_destroy(c);
    return st;
  }
  *out = c;
  return ALP_OK;
}

alp_status alp_code_destroy(alp_code* c) {
  if (!c) return ALP_OK;
  cudaFree(c->d_chk_var);
  cudaFree(c->d_chk_deg);
  cudaFree(c->d_var_chk);
  cudaFree(c->d_var_slot);
  cudaFree(c->d_var_deg);
  delete c;
  return ALP_OK;
}

size_t alp_decode_workspace_bytes(const alp_code* code, int64_t n_frames, const alp_params* params) {
  g_last_status = ALP_OK;
  if (!code || n_frames < 0 || check_params(params) != ALP_OK) {
    if (!code || n_frames < 0) fail(ALP_ERR_INVALID_ARG, "bad code or n_frames");
    return 0;
  }
  DCode C = make_dcode(code);
  Layout L = make_layout(C, smem_budget_for(params));
  LaunchCfg cfg;
  if (plan_launch(alp_decode_kernel, L, make_graph_smem(C).bytes, std::max<int64_t>(n_frames, 1), params, cfg) != ALP_OK) return 0;
  return kCounterBytes + (size_t)cfg.slots * (size_t)L.slot_bytes;
}

size_t alp_pcg_workspace_bytes(const alp_code* code, int64_t n_sys, const alp_params* params) {
  g_last_status = ALP_OK;
  if (!code || n_sys < 0 || check_params(params) != ALP_OK) {
    if (!code || n_sys < 0) fail(ALP_ERR_INVALID_ARG, "bad code or n_sys");
    return 0;
  }
  DCode C = make_dcode(code);
  Layout L = make_layout(C, smem_budget_for(params));
  LaunchCfg cfg;
  if (plan_launch(pcg_step_kernel, L, make_graph_smem(C).bytes, std::max<int64_t>(n_sys, 1), params, cfg) != ALP_OK) return 0;
  return kCounterBytes + (size_t)cfg.slots * (size_t)L.slot_bytes;
}

alp_status alp_decode(const alp_code* code, int64_t n_frames, const double* llr, uint8_t* hard,
                      double* objective, uint8_t* certificate, int32_t* frame_status,
                      alp_frame_stats* stats, double* u_out, double* y_out, uint16_t* mask_out,
                      void* workspace, size_t workspace_bytes, const alp_params* params,
                      void* stream) {
  g_last_launches = 0;
  if (!code) return fail(ALP_ERR_INVALID_ARG, "code is NULL");
  if (n_frames < 0) return fail(ALP_ERR_INVALID_ARG, "n_frames < 0");
  alp_status ps = check_params(params);
  if (ps != ALP_OK) return ps;
  if (n_frames == 0) return ALP_OK;
  if (!llr || !hard || !objective || !certificate)
    return fail(ALP_ERR_INVALID_ARG, "llr, hard, objective and certificate are required");
  if (!workspace || ((uintptr_t)workspace & 255))
    return fail(ALP_ERR_WORKSPACE, "workspace NULL or not 256-byte aligned");
  DCode C = make_dcode(code);
  Layout L = make_layout(C, smem_budget_for(params));
  LaunchCfg cfg;
  const GraphSmem G = make_graph_smem(C);
  alp_status st = plan_launch(alp_decode_kernel, L, G.bytes, n_frames, params, cfg);
  if (st != ALP_OK) return st;
  size_t need = kCounterBytes + (size_t)cfg.slots * (size_t)L.slot_bytes;
  if (workspace_bytes < need)
    return fail(ALP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* counter = (unsigned long long*)workspace;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  DecodeOut O{hard, objective, certificate, frame_status, stats, u_out, y_out, mask_out};
  alp_decode_kernel<<<cfg.grid, 32 * cfg.wpb, cfg.smem_block, s>>>(
      C, make_params(params), L, G, (char*)workspace + kCounterBytes, llr, (long long)n_frames, O, counter);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "alp_decode_kernel launch");
  g_last_launches = 1;
  return ALP_OK;
}

size_t alp_decode_host_workspace_bytes(const alp_code* code, int64_t n_frames, const alp_params* params) {
  size_t base = alp_decode_workspace_bytes(code, n_frames, params);
  if (!base) return 0;
  size_t n = code->n;
  size_t F = (size_t)n_frames;
  return base + al(8 * F * n, 256) + al(F * n, 256) + al(8 * F, 256) + al(F, 256) + al(4 * F, 256) +
         al(sizeof(alp_frame_stats) * F, 256);
}

alp_status alp_decode_host(const alp_code* code, int64_t n_frames, const double* llr_host,
                           uint8_t* hard_host, double* objective_host, uint8_t* certificate_host,
                           int32_t* frame_status_host, alp_frame_stats* stats_host, void* workspace,
                           size_t workspace_bytes, const alp_params* params, void* stream) {
  if (!code) return fail(ALP_ERR_INVALID_ARG, "code is NULL");
  if (n_frames < 0) return fail(ALP_ERR_INVALID_ARG, "n_frames < 0");
  if (n_frames == 0) return ALP_OK;
  if (!llr_host || !hard_host || !objective_host || !certificate_host)
    return fail(ALP_ERR_INVALID_ARG, "llr, hard, objective and certificate are required");
  size_t base = alp_decode_workspace_bytes(code, n_frames, params);
  if (!base) return g_last_status != ALP_OK ? g_last_status : ALP_ERR_INVALID_ARG;
  size_t need = alp_decode_host_workspace_bytes(code, n_frames, params);
  if (!workspace || ((uintptr_t)workspace & 255) || workspace_bytes < need)
    return fail(ALP_ERR_WORKSPACE, "workspace NULL, misaligned or too small: need " + std::to_string(need));
  size_t n = code->n, F = (size_t)n_frames;
  char* p = (char*)workspace + base;
  double* d_llr = (double*)p;
  p += al(8 * F * n, 256);
  uint8_t* d_hard = (uint8_t*)p;
  p += al(F * n, 256);
  double* d_obj = (double*)p;
  p += al(8 * F, 256);
  uint8_t* d_cert = (uint8_t*)p;
  p += al(F, 256);
  int32_t* d_st = (int32_t*)p;
  p += al(4 * F, 256);
  alp_frame_stats* d_stats = (alp_frame_stats*)p;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(d_llr, llr_host, 8 * F * n, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D llr");
  alp_status st = alp_decode(code, n_frames, d_llr, d_hard, d_obj, d_cert, d_st, d_stats, nullptr,
                             nullptr, nullptr, workspace, base, params, stream);
  if (st != ALP_OK) return st;
  if ((e = cudaMemcpyAsync(hard_host, d_hard, F * n, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(objective_host, d_obj, 8 * F, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(certificate_host, d_cert, F, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "D2H outputs");
  if (frame_status_host &&
      (e = cudaMemcpyAsync(frame_status_host, d_st, 4 * F, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "D2H status");
  if (stats_host && (e = cudaMemcpyAsync(stats_host, d_stats, sizeof(alp_frame_stats) * F,
                                         cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "D2H stats");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "alp_decode_host synchronize");
  return ALP_OK;
}

alp_status ipm_step_pcg(const alp_code* code, int64_t n_sys, const uint16_t* masks, const uint8_t* flip,
                        const double* d, const double* r, double* dy, int32_t* pcg_iters, double* rel_res,
                        int32_t* sys_status, int32_t* pivot_rows, int32_t* pivot_cols, void* workspace,
                        size_t workspace_bytes, const alp_params* params, void* stream) {
  g_last_launches = 0;
  if (!code) return fail(ALP_ERR_INVALID_ARG, "code is NULL");
  if (n_sys < 0) return fail(ALP_ERR_INVALID_ARG, "n_sys < 0");
  alp_status ps = check_params(params);
  if (ps != ALP_OK) return ps;
  if (n_sys == 0) return ALP_OK;
  if (!masks || !d || !r || !dy) return fail(ALP_ERR_INVALID_ARG, "masks, d, r and dy are required");
  if (!workspace || ((uintptr_t)workspace & 255))
    return fail(ALP_ERR_WORKSPACE, "workspace NULL or not 256-byte aligned");
  DCode C = make_dcode(code);
  Layout L = make_layout(C, smem_budget_for(params));
  LaunchCfg cfg;
  const GraphSmem G = make_graph_smem(C);
  alp_status st = plan_launch(pcg_step_kernel, L, G.bytes, n_sys, params, cfg);
  if (st != ALP_OK) return st;
  size_t need = kCounterBytes + (size_t)cfg.slots * (size_t)L.slot_bytes;
  if (workspace_bytes < need)
    return fail(ALP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* counter = (unsigned long long*)workspace;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  StepIO io{masks, flip, d, r, dy, pcg_iters, rel_res, sys_status, pivot_rows, pivot_cols};
  pcg_step_kernel<<<cfg.grid, 32 * cfg.wpb, cfg.smem_block, s>>>(
      C, make_params(params), L, G, (char*)workspace + kCounterBytes, (long long)n_sys, io, counter);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pcg_step_kernel launch");
  g_last_launches = 1;
  return ALP_OK;
}

}  // extern "C"
