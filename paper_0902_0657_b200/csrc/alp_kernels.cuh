// alp_kernels.cuh — IPM, frame decode and the two persistent kernels (included once per window
// mode by alp.cu, inside namespace alp::ALP_NS; see alp_device.cuh).
namespace alp {
namespace ALP_NS {

#ifndef ALP_UB
#define ALP_UB 4
#endif
constexpr int UB = ALP_UB;   // IPM-body elements per lane per step (load batching)

struct IpmOut {
  int iters, status, pcg_iters, solves, p4_fail, true_fail;
  double pcg_bytes, max_rec, max_true;
};

// IPM-body row loops, specialised on the maximum check degree (DCT): UBR rows per lane per
// step, every load of a step issued before any use (see ipm_solve).
template <int DCT>
__device__ __forceinline__ void ipm_rows_residual(const DCode& C, int lane, const uint16_t* __restrict__ SC,
                                                  const double* __restrict__ B, const double* __restrict__ X,
                                                  const double* __restrict__ Y, const double* __restrict__ Z,
                                                  double* __restrict__ V, double* W, double* __restrict__ RBv,
                                                  double* __restrict__ RCv, double& rbn, double& rcn, double& gap) {
  constexpr int UBR = (DCT <= 6) ? UB : 1;
  const int n = C.n, m = C.m;
  for (int j0 = lane; j0 < m; j0 += 32 * UBR) {
    double xs[UBR][DCT], bj[UBR], xsl[UBR], yj[UBR], zsl[UBR];
    uint16_t sc[UBR];
    int deg[UBR];
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      const int j = min(j0 + 32 * u, m - 1);
      sc[u] = (j0 + 32 * u < m) ? SC[j] : (uint16_t)0;
      deg[u] = ALP_G_CHK_DEG(C)[j];
      bj[u] = B[j];
      xsl[u] = X[n + j];
      yj[u] = Y[j];
      zsl[u] = Z[n + j];
#pragma unroll
      for (int t = 0; t < DCT; ++t) xs[u][t] = (t < deg[u]) ? X[ALP_G_CHK_VAR(C)[j * C.dc + t]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      if (!(sc[u] & PRESENT)) continue;
      const int j = j0 + 32 * u;
      double acc = bj[u] - xsl[u];
#pragma unroll
      for (int t = 0; t < DCT; ++t)
        if (t < deg[u]) acc = ((sc[u] >> t) & 1) ? acc + xs[u][t] : acc - xs[u][t];
      W[j] = acc;
      RBv[j] = acc;
      rbn = fmax(rbn, fabs(acc));
      const double rc = -yj[u] - zsl[u];
      V[n + j] = rc;
      RCv[n + j] = rc;
      rcn = fmax(rcn, fabs(rc));
      gap += xsl[u] * zsl[u];
    }
  }
}

template <int DCT>
__device__ __forceinline__ void ipm_rows_w(const DCode& C, int lane, const uint16_t* __restrict__ SC, double* W,
                                           const double* __restrict__ V) {
  constexpr int UBR = (DCT <= 6) ? UB : 1;
  const int n = C.n, m = C.m;
  for (int j0 = lane; j0 < m; j0 += 32 * UBR) {
    double vs[UBR][DCT], wj[UBR], vsl[UBR];
    uint16_t sc[UBR];
    int deg[UBR];
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      const int j = min(j0 + 32 * u, m - 1);
      sc[u] = (j0 + 32 * u < m) ? SC[j] : (uint16_t)0;
      deg[u] = ALP_G_CHK_DEG(C)[j];
      wj[u] = W[j];
      vsl[u] = V[n + j];
#pragma unroll
      for (int t = 0; t < DCT; ++t) vs[u][t] = (t < deg[u]) ? V[ALP_G_CHK_VAR(C)[j * C.dc + t]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      if (!(sc[u] & PRESENT)) continue;
      double acc = wj[u] + vsl[u];
#pragma unroll
      for (int t = 0; t < DCT; ++t)
        if (t < deg[u]) acc = ((sc[u] >> t) & 1) ? acc - vs[u][t] : acc + vs[u][t];
      W[j0 + 32 * u] = acc;
    }
  }
}

// rho = r_b - A dx on the present rows (the step residual moved onto the basis, C-32), UBR rows
// per lane per step with every gather issued before the sums (the slot arrays are L2-resident).
template <int DCT>
__device__ __forceinline__ void ipm_rows_rho(const DCode& C, int lane, const uint16_t* __restrict__ SC,
                                             const double* __restrict__ RBv, const double* __restrict__ V,
                                             double* __restrict__ rS) {
  constexpr int UBR = (DCT <= 6) ? UB : 1;
  const int n = C.n, m = C.m;
  for (int j0 = lane; j0 < m; j0 += 32 * UBR) {
    double vs[UBR][DCT], rb[UBR], vsl[UBR];
    uint16_t sc[UBR];
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      const int j = min(j0 + 32 * u, m - 1);
      sc[u] = (j0 + 32 * u < m) ? SC[j] : (uint16_t)0;
      const int deg = (sc[u] & PRESENT) ? (int)ALP_G_CHK_DEG(C)[j] : 0;
      rb[u] = RBv[j];
      vsl[u] = V[n + j];
#pragma unroll
      for (int t = 0; t < DCT; ++t) vs[u][t] = (t < deg) ? V[ALP_G_CHK_VAR(C)[j * C.dc + t]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UBR; ++u) {
      if (j0 + 32 * u >= m) continue;
      double acc = 0.0;
      if (sc[u] & PRESENT) {
        acc = rb[u] - vsl[u];
#pragma unroll
        for (int t = 0; t < DCT; ++t) acc = ((sc[u] >> t) & 1) ? acc + vs[u][t] : acc - vs[u][t];
      }
      rS[j0 + 32 * u] = acc;
    }
  }
}

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
__device__ ALP_CALL_IPM IpmOut ipm_solve(const Frame& F, const Params& P, const double* g, int p, int nact,
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
  const double* DY = F.dy_();
  const uint16_t* __restrict__ SC = F.sgnC_();
  const uint8_t* __restrict__ SV = F.sgnV_();
  double* __restrict__ RBv = F.rb;   // r_b and r_c of the current iterate (kept for the recovery)
  double* __restrict__ RCv = F.rc;
  ALP_GL(X);
  ALP_GL(Z);
  ALP_GL(Y);
  ALP_GL(V);
  ALP_GL(B);
  ALP_GL(RBv);
  ALP_GL(RCv);
  ALP_GL_SM(D2);
  ALP_GL_SM(W);
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
    // Every body loop below takes UB elements per lane per step and issues all of their loads
    // (unconditionally: slot arrays cover every index, absent rows hold 0) before any use, so
    // the L1/L2 round trips of a step overlap; presence only predicates the stores.
    if (C.dcr <= 6) ipm_rows_residual<6>(C, lane, SC, B, X, Y, Z, V, W, RBv, RCv, rbn, rcn, gap);
    else ipm_rows_residual<DCMAX>(C, lane, SC, B, X, Y, Z, V, W, RBv, RCv, rbn, rcn, gap);
    for (int i0 = lane; i0 < n; i0 += 32 * UB) {
      double gi[UB], zi[UB], xi[UB], ys[UB][DVMAX];
      uint8_t sv[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int i = min(i0 + 32 * u, n - 1);
        sv[u] = (i0 + 32 * u < n) ? SV[i] : (uint8_t)0;
        gi[u] = g[i];
        zi[u] = Z[i];
        xi[u] = X[i];
#pragma unroll
        for (int k = 0; k < DVMAX; ++k) ys[u][k] = Y[min((int)ALP_G_VAR_CHK(C)[i * C.dv + k], m - 1)];
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (i0 + 32 * u >= n) continue;
        const int i = i0 + 32 * u;
        const double ci = fabs(gi[u]);
        double acc = ci - zi[u];
#pragma unroll
        for (int k = 0; k < DVMAX; ++k)
          if ((sv[u] >> k) & 1) acc = ((sv[u] >> (4 + k)) & 1) ? acc + ys[u][k] : acc - ys[u][k];
        V[i] = acc;
        RCv[i] = acc;
        rcn = fmax(rcn, fabs(acc));
        gap += xi[u] * zi[u];
        cx += ci * xi[u];
      }
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
    for (int c0 = lane; c0 < Q; c0 += 32 * UB) {
      double xc[UB], zc[UB], vc[UB];
      bool ok[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int c = min(c0 + 32 * u, Q - 1);
        ok[u] = (c0 + 32 * u < Q) && ((c < n) || (SC[c - n] & PRESENT));
        xc[u] = X[c];
        zc[u] = Z[c];
        vc[u] = V[c];
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (!ok[u]) continue;
        const int c = c0 + 32 * u;
        const double iz = 1.0 / zc[u];   // one division for D^2 = X Z^-1 and Z^-1 r_e
        const double d2 = xc[u] * iz;
        const double re = mu - xc[u] * zc[u];
        D2[c] = d2;
        V[c] = d2 * vc[u] - re * iz;
      }
    }
    __syncwarp();
    if (C.dcr <= 6) ipm_rows_w<6>(C, lane, SC, W, V);
    else ipm_rows_w<DCMAX>(C, lane, SC, W, V);
    __syncwarp();
    int nLb = 0, nLf = 0;
    const bool mtm = (P.precond != 1);   // MTS-preconditioned PCG (Alg. 7, 8 or 6)
    ALP_TICK(F, CY_IPM, tk);
    // the Alg. 7 triangular set is both the PCG preconditioner (precond = 0) and the basis of
    // the step's feasibility correction (C-32), so plain CG builds it too when that is on
    if (mtm || P.basis_correction) build_precond(F, p, nLb, nLf, P.precond == 1 ? 0 : P.precond);
    ALP_TICK(F, CY_BUILD, tk);
    // inexact-Newton forcing term (R-1): the dual step needs A^T dy accurate to well
    // below z ~ mu on the basic columns, so late in the IPM the recursion aims at
    // min(pcg_rel_tol, 1e-2 mu) (floored at 1e-14); P4 acceptance is pcg_rel_tol.  An inexact
    // dy is admissible because the recovery below keeps every KKT row but the complementarity
    // of the basis columns exact (C-32).
    const double inner = fmin(P.pcg_rel_tol, fmax(1e-14, P.pcg_forcing * mu));
    PcgResult pr = pcg_solve(F, P, mtm ? PC_MTS : PC_NONE, nLb, nLf, inner, 0);
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
    for (int i0 = lane; i0 < n; i0 += 32 * UB) {
      double d2i[UB], vi[UB], rci[UB], dys[UB][DVMAX];
      uint8_t sv[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int i = min(i0 + 32 * u, n - 1);
        sv[u] = (i0 + 32 * u < n) ? SV[i] : (uint8_t)0;
        d2i[u] = D2[i];
        vi[u] = V[i];
        rci[u] = RCv[i];
#pragma unroll
        for (int k = 0; k < DVMAX; ++k) dys[u][k] = ((sv[u] >> k) & 1) ? DY[ALP_G_VAR_CHK(C)[i * C.dv + k]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (i0 + 32 * u >= n) continue;
        const int i = i0 + 32 * u;
        double atdy = 0.0;
#pragma unroll
        for (int k = 0; k < DVMAX; ++k)
          if ((sv[u] >> k) & 1) atdy = ((sv[u] >> (4 + k)) & 1) ? atdy - dys[u][k] : atdy + dys[u][k];
        V[i] = d2i[u] * atdy - vi[u];   // dx
        D2[i] = rci[u] - atdy;          // dz
      }
    }
    for (int j0 = lane; j0 < m; j0 += 32 * UB) {
      double d2s[UB], dyj[UB], vs[UB], rcs[UB];
      bool ok[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int j = min(j0 + 32 * u, m - 1);
        ok[u] = (j0 + 32 * u < m) && (SC[j] & PRESENT);
        d2s[u] = D2[n + j];
        dyj[u] = DY[j];
        vs[u] = V[n + j];
        rcs[u] = RCv[n + j];
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (!ok[u]) continue;
        const int c = n + j0 + 32 * u;
        V[c] = d2s[u] * dyj[u] - vs[u];
        D2[c] = rcs[u] - dyj[u];
      }
    }
    __syncwarp();
    if (P.basis_correction && nLb > 0) {
      double* rS = F.r_();
      double* fS = F.fz_();
      if (C.dcr <= 6) ipm_rows_rho<6>(C, lane, SC, RBv, V, rS);
      else ipm_rows_rho<DCMAX>(C, lane, SC, RBv, V, rS);
      __syncwarp();
      back_sweep(F, nLb, rS, fS);   // f = A_M^-1 rho, f_R = component of row R's pivot column
      __syncwarp();
      const uint16_t* pcolR = F.pcolR_();
      for (int j0 = lane; j0 < m; j0 += 32 * UB) {   // dx_M += f (distinct pivot columns)
        uint16_t cs[UB];
        double vc[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) cs[u] = (j0 + 32 * u < m) ? pcolR[j0 + 32 * u] : NONE16;
#pragma unroll
        for (int u = 0; u < UB; ++u) vc[u] = (cs[u] != NONE16) ? V[cs[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < UB; ++u)
          if (cs[u] != NONE16) V[cs[u]] = vc[u] + fS[j0 + 32 * u];
      }
      __syncwarp();
    }
    // ratio test (C-6)
    double ax = 1e308, az = 1e308;
    for (int c0 = lane; c0 < Q; c0 += 32 * UB) {
      double dxs[UB], dzs[UB], xc[UB], zc[UB];
      bool ok[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int c = min(c0 + 32 * u, Q - 1);
        ok[u] = (c0 + 32 * u < Q) && ((c < n) || (SC[c - n] & PRESENT));
        dxs[u] = V[c];
        dzs[u] = D2[c];
        xc[u] = X[c];
        zc[u] = Z[c];
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (!ok[u]) continue;
        if (dxs[u] < 0.0) ax = fmin(ax, -xc[u] / dxs[u]);
        if (dzs[u] < 0.0) az = fmin(az, -zc[u] / dzs[u]);
      }
    }
    ax = wmin(ax);
    az = wmin(az);
    const double bP = fmin(1.0, P.eta * ax);
    const double bD = fmin(1.0, P.eta * az);
    if (g_trace) {
      if (lane == 0) {
        int slot = atomicAdd(&g_trace_n, 1);
        if (slot < g_trace_cap)
          g_trace[slot] = TraceRec{(int)frame_id, lp_id, it, p, pr.status, pr.iters, nLb, nLf, pr.relres, pr.rec_relres, dmn, dmx, mu, rbn, rcn, gap, bP, bD};
      }
    }
    bool bad = false;
    for (int c0 = lane; c0 < Q; c0 += 32 * UB) {
      double dxs[UB], dzs[UB], xc[UB], zc[UB];
      bool ok[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int c = min(c0 + 32 * u, Q - 1);
        ok[u] = (c0 + 32 * u < Q) && ((c < n) || (SC[c - n] & PRESENT));
        dxs[u] = V[c];
        dzs[u] = D2[c];
        xc[u] = X[c];
        zc[u] = Z[c];
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (!ok[u]) continue;
        const int c = c0 + 32 * u;
        const double xn = xc[u] + bP * dxs[u];
        const double zn = zc[u] + bD * dzs[u];
        X[c] = xn;
        Z[c] = zn;
        bad |= !isfinite(xn) || !isfinite(zn);
      }
    }
    for (int j0 = lane; j0 < m; j0 += 32 * UB) {
      double yv[UB];
      bool ok[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int j = j0 + 32 * u;
        ok[u] = (j < m) && (SC[min(j, m - 1)] & PRESENT);
        yv[u] = ok[u] ? Y[j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (!ok[u]) continue;
        const double yn = yv[u] + bD * DY[j0 + 32 * u];
        Y[j0 + 32 * u] = yn;
        bad |= !isfinite(yn);
      }
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


#ifdef ALP_POISON
// Diagnostics build (-DALP_POISON): before each frame / system, fill the warp's shared window
// and its whole global slot with NaN bit patterns, so any read of state that the frame did not
// write first changes the outputs (tools/poison_check.py compares against the normal build;
// stands in for compute-sanitizer initcheck, which this pool does not allow).
__device__ __forceinline__ void poison_frame(const Frame& F, char* slot) {
  const Layout& L = *F.L;
  unsigned long long* s8 = reinterpret_cast<unsigned long long*>(slot);
  for (long long k = F.lane; k < L.slot_bytes / 8; k += 32) s8[k] = 0xfff8dead0000beefull;
  if (!L.win_global) {
    unsigned long long* w8 = reinterpret_cast<unsigned long long*>(F.sm);
    for (int k = F.lane; k < L.smem_bytes / 8; k += 32) w8[k] = 0xfff8dead0000beefull;
  }
  __syncwarp();
}
#endif

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
  if (lane < 8) ALP_CYC(F)[lane] = 0;
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
#pragma unroll 4
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
    int deg = ALP_G_CHK_DEG(C)[j];
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
      st.cyc_cut = ALP_CYC(F)[CY_CUT];
      st.cyc_ipm = ALP_CYC(F)[CY_IPM];
      st.cyc_build = ALP_CYC(F)[CY_BUILD];
      st.cyc_spmv = ALP_CYC(F)[CY_SPMV];
      st.cyc_sweep = ALP_CYC(F)[CY_SWEEP];
      st.cyc_pcg_other = ALP_CYC(F)[CY_PCG];
      st.cyc_sort = ALP_CYC(F)[CY_SORT];
      st.cyc_peel = ALP_CYC(F)[CY_PEEL];
      O.stats[f] = st;
    }
  }
  __syncwarp();
}

#ifndef ALP_MINB
#define ALP_MINB 1
#endif
__global__ void __launch_bounds__(256, ALP_MINB) alp_decode_kernel(DCode C, Params P, Layout L, GraphSmem G,
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
#ifndef ALP_CYC_STATIC
  __shared__ long long s_cyc[8][8];   // phase clocks in shared memory (a global RMW per tick
  F.cyc = s_cyc[warp];                // would stall the warp on an L2 round trip)
#endif
  while (true) {
    long long f = 0;
    if (lane == 0) f = (long long)atomicAdd(counter, 1ull);   // 64-bit: no wrap at any n_frames
    f = __shfl_sync(FULL, f, 0);
    if (f >= n_frames) break;
#ifdef ALP_POISON
    poison_frame(F, slot);
#endif
    decode_frame(F, P, llr + f * C.n, f, O);
  }
}


// Isolated step solve (eq.`Delta y` P:479) per system: signs, D^2, Alg. 7, PCG.
__global__ void __launch_bounds__(256, 1) pcg_step_kernel(DCode C, Params P, Layout L, GraphSmem G,
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
#ifdef ALP_POISON
    poison_frame(F, slot);
#endif
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
    for (int j = lane; j < m; j += 32) F.w[j] = (F.sgnC_()[j] & PRESENT) ? io.r[s * m + j] : 0.0;
    __syncwarp();
    int nLb = 0, nLf = 0;
    const bool mtm = (P.precond != 1) && p > 0;
    if (mtm) build_precond(F, p, nLb, nLf, P.precond);
    if ((io.prow || io.pcol)) {
      if (mtm) write_pivots(F, p, io.prow ? io.prow + s * m : nullptr, io.pcol ? io.pcol + s * m : nullptr);
      else
        for (int k = lane; k < m; k += 32) {
          if (io.prow) io.prow[s * m + k] = -1;
          if (io.pcol) io.pcol[s * m + k] = -1;
        }
    }
    PcgResult pr = pcg_solve(F, P, mtm ? PC_MTS : PC_NONE, nLb, nLf, P.pcg_rel_tol, P.pcg_refine);
    for (int j = lane; j < m; j += 32) io.dy[s * m + j] = (F.sgnC_()[j] & PRESENT) ? F.dy_()[j] : 0.0;
    if (lane == 0) {
      if (io.iters) io.iters[s] = pr.iters;
      if (io.relres) io.relres[s] = pr.relres;
      if (io.status) io.status[s] = pr.status;
    }
    __syncwarp();
  }
}

}  // namespace ALP_NS
}  // namespace alp
#undef ALP_SH
#undef ALP_GL_SM
#undef ALP_GL
#undef ALP_SHA
