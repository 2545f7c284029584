// alp_device.cuh — warp-per-frame device building blocks of libalp (sm_100a).
//
// One warp owns one frame (or one isolated step system) at a time; every step of the
// method runs inside that warp with lane-strided loops, warp-shuffle reductions and
// __syncwarp barriers.  Per-frame vectors live in a per-warp "slot" of global memory
// (frame-major, contiguous, reused frame after frame so the live set stays L2-resident);
// the latency-critical sequential parts (column sort, Alg. 7 peel, level build) and the
// gathered PCG vectors live in the warp's shared-memory window, whose phases alias, followed
// by whichever PCG-hot slot arrays fit the window budget (Layout::smask).  Each CTA stages the
// Tanner graph and the code / layout descriptors in shared memory (stage_graph).
// Citations: PAPER.md line numbers (P:n) with section / algorithm / equation label.
#include <cstdint>
#include <cuda_runtime.h>

// Large phase functions (ALP_HEAVY).  Compiling them as real calls (-DALP_HEAVY=__noinline__)
// cuts the decode kernel from 255 to 128 registers, but the calls' stack traffic made every
// phase slower (measured 2032 vs 3868 frames/s, C2 3.0 dB), so by default they are inlined.
#ifndef ALP_HEAVY
#define ALP_HEAVY
#endif
// Per-phase call boundaries (tuning experiments): a real call gives the phase its own register
// allocation at the price of passing the Frame through memory.
#ifndef ALP_CALL_PCG
#define ALP_CALL_PCG ALP_HEAVY
#endif
#ifndef ALP_CALL_BUILD
#define ALP_CALL_BUILD ALP_HEAVY
#endif
#ifndef ALP_CALL_IPM
#define ALP_CALL_IPM ALP_HEAVY
#endif
// the PCG loop's parts (SpMV passes, sweeps): inlined by default; as calls (tuning) the hot
// loop's instruction footprint shrinks to one copy of each
#ifndef ALP_PCGPART
#define ALP_PCGPART __forceinline__
#endif

#ifndef ALP_DEVICE_TYPES
#define ALP_DEVICE_TYPES
namespace alp {

extern __shared__ __align__(16) char alp_dsmem[];   // the kernels' dynamic shared memory
#ifdef ALP_CYC_STATIC
// phase clocks as a file-scope static shared array: ticks compile to LDS/STS at a fixed address
// (through a generic pointer kept in the Frame each tick is a generic load + store to shared memory)
__shared__ long long alp_cyc_sh[8][8];
#define ALP_CYC(F) (alp_cyc_sh[threadIdx.x >> 5])
#else
#define ALP_CYC(F) ((F).cyc)
#endif

constexpr unsigned FULL = 0xffffffffu;
constexpr uint16_t PRESENT = 0x8000u;
constexpr uint16_t NONE16 = 0xffffu;
constexpr int DCMAX = 15;  // d_c <= 15 (mask bits 0..14)
constexpr int DVMAX = 4;   // d_v <= 4  (sgnV packing: 4 present bits + 4 sign bits)
constexpr int RF = 4;      // forward-record u16: head + up to d_v - 1 deps (8 bytes)
constexpr uint16_t NODEP = 0xffffu;   // unused dependency slot of a sweep record

// frame status bits (include/alp.h alp_frame_status)
constexpr int ST_ALP_MAXITER = 1, ST_IPM_MAXITER = 2, ST_PCG_MAXITER = 4, ST_PCG_BREAKDOWN = 8,
              ST_NUMERIC = 16, ST_PCG_FLOOR = 32;

struct Params {
  int variant, precond;
  double sigma, eta, gap_tol, feas_tol, pcg_rel_tol, pcg_forcing, tau_viol, tau_act, tau_cert;
  int alp_max_iter, ipm_max_iter, pcg_max_iter;
  int stop_on_lp_failure, basis_correction, pcg_refine;
};

// Device view of the Tanner graph (immutable, shared by all warps; L1/L2 resident).
struct DCode {
  int n, m, dc, dv, Q, W, RB;             // Q = n + m columns, W = bitmap words, RB = back-record u16 (8/16)
  int dcr, dvr;                           // maximum check / variable degree (dc, dv: padded strides 8|16, 4)
  const uint16_t* __restrict__ chk_var;   // [m][dc] sorted variables of each check, 0xffff padded
  const uint8_t* __restrict__ chk_deg;    // [m]
  const uint16_t* __restrict__ var_chk;   // [n][dv] checks of each variable, 0xffff padded
  const uint8_t* __restrict__ var_slot;   // [n][dv] position t of the variable in N(check)
  const uint8_t* __restrict__ var_deg;    // [n]
  // byte offsets of the staged copies in the CTA's dynamic shared memory (stage_graph; sm mode
  // forms the graph addresses from the shared-memory symbol itself, so graph reads are LDS)
  int so_chk_var, so_chk_deg, so_var_chk, so_var_deg;
};

// Per-CTA shared copy of the Tanner graph (host-computed byte offsets; 0 bytes = stay global).
struct GraphSmem {
  int bytes, o_chk_var, o_chk_deg, o_var_chk, o_var_slot, o_var_deg;
};

// Every thread of the CTA copies the graph arrays into the CTA's shared area `g` and gets a
// DCode whose pointers address that copy (graph reads become shared-memory loads).
__device__ __forceinline__ void stage_graph(const DCode& C, const GraphSmem& G, char* g, DCode& out) {
  out = C;
  out.so_chk_var = out.so_chk_deg = out.so_var_chk = out.so_var_deg = 0;
  if (G.bytes == 0) return;
  auto cp = [&](const void* src, int off, int bytes) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(g + off);
    for (int k = threadIdx.x; k < (bytes + 3) / 4; k += blockDim.x) d4[k] = s4[k];
  };
  cp(C.chk_var, G.o_chk_var, C.m * C.dc * 2);
  cp(C.chk_deg, G.o_chk_deg, C.m);
  cp(C.var_chk, G.o_var_chk, C.n * C.dv * 2);
  cp(C.var_deg, G.o_var_deg, C.n);
  out.chk_var = reinterpret_cast<const uint16_t*>(g + G.o_chk_var);
  out.chk_deg = reinterpret_cast<const uint8_t*>(g + G.o_chk_deg);
  out.var_chk = reinterpret_cast<const uint16_t*>(g + G.o_var_chk);
  // var_slot stays global: only build_signs reads it, once per LP
  out.var_deg = reinterpret_cast<const uint8_t*>(g + G.o_var_deg);
  out.so_chk_var = G.o_chk_var;
  out.so_chk_deg = G.o_chk_deg;
  out.so_var_chk = G.o_var_chk;
  out.so_var_deg = G.o_var_deg;
}

// Byte offsets inside one warp's global slot and shared-memory window (host-computed).
struct Layout {
  long long slot_bytes;
  long long g_cyc, g_x, g_z, g_d2, g_v, g_y, g_dy, g_r, g_w, g_u, g_b, g_dinvF, g_recB, g_recF, g_offB,
      g_offF, g_sgnC, g_mask, g_hist, g_sgnV, g_flip, g_rb, g_rc, g_pcol;
  int smem_bytes;
  // win_global: the phase window does not fit the shared-memory budget (large codes, e.g.
  // config 4): it lives in the slot at g_win and is addressed through the same generic pointers
  int win_global;
  long long g_win;
  // Per-frame arrays that live in the warp's shared window instead of the slot
  // (bit k of smask set <=> array k at shared offset soff[k]); order = placement priority.
  unsigned smask;
  int soff[12];
  int s_sortk, s_sorth;                                                        // sort phase
  int s_order, s_rank, s_cnt, s_xr, s_bm, s_pos, s_pcol, s_prow, s_lvB, s_lvF;  // peel phase
  int s_rrank, RS;                      // peel: ranks of each row's columns, RS per row
  int s_poc, s_hist, s_cur;                                                    // post-peel
  int s_h, s_r, s_fz;   // PCG phase: h, r [m]; f and z share s_fz (z overwrites f in place), t [n]
                        // (SpMV, variable pass) overlays s_fz, sized 8 max(m, n)
};

// ------------------------------------------------------------------ warp reductions
// xor-butterflies: every lane ends with the bit-identical result (commutative adds), so
// decisions taken on reduced values are warp-uniform.
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double wmin(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ int wsumi(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ int wmaxi(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// Phase clock: lane 0 adds the cycles since `t` to counter `ph` and restarts `t`.
enum { CY_CUT = 0, CY_IPM = 1, CY_BUILD = 2, CY_SPMV = 3, CY_SWEEP = 4, CY_PCG = 5, CY_SORT = 6, CY_PEEL = 7 };
#define ALP_TICK(F, ph, t)                          \
  do {                                              \
    long long now_ = clock64();                     \
    if ((F).lane == 0) ALP_CYC(F)[ph] += now_ - (t);   \
    (t) = now_;                                     \
  } while (0)

// Relocatable per-frame arrays (window or slot); the sweep programs are u16 records in level
// order (recB / recF) with their level offsets and dinvF = 1 / d^2 of each forward slot's pivot.
enum { RL_SGNC = 0, RL_SGNV, RL_DY, RL_DINVF, RL_OFFB, RL_OFFF, RL_RECF, RL_RECB, RL_D2, RL_W, RL_N };

__device__ __forceinline__ char* rel_ptr(const Layout* L, char* slot, char* sm, int k, long long g) {
  return ((L->smask >> k) & 1u) ? sm + L->soff[k] : slot + g;
}

}  // namespace alp
#endif  // ALP_DEVICE_TYPES

// ---------------------------------------------------------------------------------------------
// Mode-dependent device code, included once per window mode (alp.cu):
//   ALP_NS = sm, ALP_SM = 1: the whole per-frame window and the PCG-hot arrays live in shared
//     memory (fixed layout, make_layout_sm); ALP_SH(p) tells the compiler so, and the loads are
//     LDS instead of generic loads (measured: generic loads dominated the stalls, ncu r2a).
//   ALP_NS = gm, ALP_SM = 0: budget-relocated arrays, possibly a global-memory window (large
//     codes, e.g. config 4); every access is a generic load.
// ---------------------------------------------------------------------------------------------
#define ALP_SH(p) ((void)0)
#define ALP_GL_SM(p) ((void)0)
#define ALP_GL(p) ((void)0)
#ifdef ALP_ASSUME_S_ONLY
#define ALP_SHA(p) ((void)0)
#else
#define ALP_SHA(p) ALP_SH(p)
#endif   // (an __isGlobal assume broke the NVVM module; generic loads stay)
// Graph arrays: in the sm and gs instances the graph is always staged (make_plan), and its addresses
// are formed from the dynamic shared-memory symbol (LDS; a pointer kept in DCode compiles to
// generic loads).
#undef ALP_G_CHK_VAR
#undef ALP_G_CHK_DEG
#undef ALP_G_VAR_CHK
#undef ALP_G_VAR_DEG
#if (ALP_SM || defined(ALP_GRAPH_SH)) && !defined(ALP_GRAPH_GENERIC)
#define ALP_G_CHK_VAR(C) (reinterpret_cast<const uint16_t*>(alp_dsmem + (C).so_chk_var))
#define ALP_G_CHK_DEG(C) (reinterpret_cast<const uint8_t*>(alp_dsmem + (C).so_chk_deg))
#define ALP_G_VAR_CHK(C) (reinterpret_cast<const uint16_t*>(alp_dsmem + (C).so_var_chk))
#define ALP_G_VAR_DEG(C) (reinterpret_cast<const uint8_t*>(alp_dsmem + (C).so_var_deg))
#else
#define ALP_G_CHK_VAR(C) ((C).chk_var)
#define ALP_G_CHK_DEG(C) ((C).chk_deg)
#define ALP_G_VAR_CHK(C) ((C).var_chk)
#define ALP_G_VAR_DEG(C) ((C).var_deg)
#endif
namespace alp {
namespace ALP_NS {

__device__ __forceinline__ int chk_nb(const DCode& C, int j, int t) {
  const unsigned v = ALP_G_CHK_VAR(C)[j * C.dc + t];
  return v == 0xffffu ? -1 : (int)v;
}
__device__ __forceinline__ int var_ck(const DCode& C, int i, int k) {
  const unsigned v = ALP_G_VAR_CHK(C)[i * C.dv + k];
  return v == 0xffffu ? -1 : (int)v;
}

// Per-frame working set: pointers into the warp's global slot and shared window.
struct Frame {
  const DCode* C;
  const Layout* L;
  int lane;
  char* sm;
  double *x, *z, *d2, *v, *y, *dy, *r, *w, *u, *b, *dinvF, *rb, *rc;
  uint16_t* pcolR;  // [m]: pivot column of pivot row R (0..n+m-1), NONE16 if R is not a pivot (slot)
  uint16_t *recB, *recF;  // sweep programs (u16 records, see build_precond)
  uint16_t *offB, *offF;   // level offsets (u16: <= p + 1 <= 32768)
  uint16_t* sgnC;  // [m]: bit t <-> coefficient of x_{N(j)[t]} is -1; bit 15 <-> row present
  uint16_t* mask;  // [m]: cut pool (include/alp.h mask word)
  unsigned long long* hist;  // [alp_max_iter + 1] pool hashes of the LPs solved (C-12)
  uint8_t* sgnV;   // [n]: bit k <-> k-th check of the variable present; bit 4+k <-> coef -1
  uint8_t* flip;   // [n]: 1 <-> gamma_i < 0 (x_i = 1 - u_i, §IV-B)
  long long* cyc;  // [8] per-phase clock64 accumulators (lane 0 writes; alp_frame_stats)
#if ALP_SM
  // sm mode: every window address is formed from the dynamic shared-memory symbol itself, so
  // the compiler emits LDS/STS (a generic pointer kept in the Frame would compile to generic
  // loads).  smo = the frame window's byte offset in dynamic shared memory.
  unsigned smo;
  unsigned o_sgnC, o_sgnV, o_dy, o_dinvF, o_recB, o_recF, o_offB, o_offF;
#ifdef ALP_CACHE_OFFS
  unsigned o_h, o_r, o_fz;   // PCG vectors: offsets kept in registers (L lives in shared memory
                             // behind a generic pointer, a slow load per accessor call)
#endif
  template <class T>
  __device__ __forceinline__ T* S(int off) const { return reinterpret_cast<T*>(alp_dsmem + smo + off); }
  template <class T>
  __device__ __forceinline__ T* W_(unsigned off) const { return reinterpret_cast<T*>(alp_dsmem + smo + off); }
  __device__ __forceinline__ uint16_t* sgnC_() const { return W_<uint16_t>(o_sgnC); }
  __device__ __forceinline__ uint8_t* sgnV_() const { return W_<uint8_t>(o_sgnV); }
  __device__ __forceinline__ double* dinvF_() const { return W_<double>(o_dinvF); }
  __device__ __forceinline__ uint16_t* recB_() const { return W_<uint16_t>(o_recB); }
  __device__ __forceinline__ uint16_t* recF_() const { return W_<uint16_t>(o_recF); }
  __device__ __forceinline__ uint16_t* offB_() const { return W_<uint16_t>(o_offB); }
  __device__ __forceinline__ uint16_t* offF_() const { return W_<uint16_t>(o_offF); }
  __device__ __forceinline__ double* dy_() const { return W_<double>(o_dy); }
#ifdef ALP_SM_R_SLOT
  __device__ __forceinline__ double* r_() const { return r; }     // slot (tuning variant)
#elif defined(ALP_CACHE_OFFS)
  __device__ __forceinline__ double* r_() const { return W_<double>(o_r); }
#else
  __device__ __forceinline__ double* r_() const { return S<double>(L->s_r); }
#endif
#else
  template <class T>
  __device__ __forceinline__ T* S(int off) const { return reinterpret_cast<T*>(sm + off); }
  __device__ __forceinline__ uint16_t* sgnC_() const { return sgnC; }
  __device__ __forceinline__ uint8_t* sgnV_() const { return sgnV; }
  __device__ __forceinline__ double* dinvF_() const { return dinvF; }
  __device__ __forceinline__ uint16_t* recB_() const { return recB; }
  __device__ __forceinline__ uint16_t* recF_() const { return recF; }
  __device__ __forceinline__ uint16_t* offB_() const { return offB; }
  __device__ __forceinline__ uint16_t* offF_() const { return offF; }
  __device__ __forceinline__ double* dy_() const { return dy; }
  __device__ __forceinline__ double* r_() const { return S<double>(L->s_r); }
#endif
  __device__ __forceinline__ uint16_t* pcolR_() const { return pcolR; }
#if ALP_SM && defined(ALP_CACHE_OFFS)
  __device__ __forceinline__ double* h_() const { return W_<double>(o_h); }
  __device__ __forceinline__ double* fz_() const { return W_<double>(o_fz); }
#else
  __device__ __forceinline__ double* h_() const { return S<double>(L->s_h); }
  __device__ __forceinline__ double* fz_() const { return S<double>(L->s_fz); }
#endif
};

__device__ __forceinline__ void frame_bind(Frame& F, const DCode* C, const Layout* L, char* slot,
                                           char* sm, int lane) {
  F.C = C;
  F.L = L;
  F.lane = lane;
  F.sm = sm;
  F.cyc = (long long*)(slot + L->g_cyc);
  F.x = (double*)(slot + L->g_x);
  F.z = (double*)(slot + L->g_z);
  F.d2 = (double*)(slot + L->g_d2);
  F.v = (double*)(slot + L->g_v);
  F.y = (double*)(slot + L->g_y);
  F.dy = (double*)(slot + L->g_dy);
  F.r = (double*)(slot + L->g_r);
  F.w = (double*)(slot + L->g_w);
  F.u = (double*)(slot + L->g_u);
  F.b = (double*)(slot + L->g_b);
  F.dinvF = (double*)(slot + L->g_dinvF);
  F.recB = (uint16_t*)(slot + L->g_recB);
  F.recF = (uint16_t*)(slot + L->g_recF);
  F.offB = (uint16_t*)(slot + L->g_offB);
  F.offF = (uint16_t*)(slot + L->g_offF);
  F.sgnC = (uint16_t*)(slot + L->g_sgnC);
  F.mask = (uint16_t*)(slot + L->g_mask);
  F.hist = (unsigned long long*)(slot + L->g_hist);
  F.rb = (double*)(slot + L->g_rb);
  F.rc = (double*)(slot + L->g_rc);
  F.pcolR = (uint16_t*)(slot + L->g_pcol);
  F.flip = (uint8_t*)(slot + L->g_flip);
#if ALP_SM
  // sm mode: the sweep programs, sign tables and dy are always in the window (make_layout_sm);
  // d^2 and w never
  F.smo = (unsigned)(sm - alp_dsmem);
  F.o_sgnC = L->soff[RL_SGNC];
  F.o_sgnV = L->soff[RL_SGNV];
  F.o_dy = L->soff[RL_DY];
  F.o_dinvF = L->soff[RL_DINVF];
  F.o_recB = L->soff[RL_RECB];
  F.o_recF = L->soff[RL_RECF];
  F.o_offB = L->soff[RL_OFFB];
  F.o_offF = L->soff[RL_OFFF];
#ifdef ALP_CACHE_OFFS
  F.o_h = L->s_h;
  F.o_r = L->s_r;
  F.o_fz = L->s_fz;
#endif
  F.sgnC = F.sgnC_();
  F.sgnV = F.sgnV_();
  F.dy = F.dy_();
  F.dinvF = F.dinvF_();
  F.recB = F.recB_();
  F.recF = F.recF_();
  F.offB = F.offB_();
  F.offF = F.offF_();
  if ((L->smask >> RL_D2) & 1u) F.d2 = (double*)(sm + L->soff[RL_D2]);
  return;
#endif
  F.recB = (uint16_t*)rel_ptr(L, slot, sm, RL_RECB, L->g_recB);
  F.recF = (uint16_t*)rel_ptr(L, slot, sm, RL_RECF, L->g_recF);
  F.offB = (uint16_t*)rel_ptr(L, slot, sm, RL_OFFB, L->g_offB);
  F.offF = (uint16_t*)rel_ptr(L, slot, sm, RL_OFFF, L->g_offF);
  F.dinvF = (double*)rel_ptr(L, slot, sm, RL_DINVF, L->g_dinvF);
  F.sgnC = (uint16_t*)rel_ptr(L, slot, sm, RL_SGNC, L->g_sgnC);
  F.sgnV = (uint8_t*)rel_ptr(L, slot, sm, RL_SGNV, L->g_sgnV);
  F.d2 = (double*)rel_ptr(L, slot, sm, RL_D2, L->g_d2);
  F.dy = (double*)rel_ptr(L, slot, sm, RL_DY, L->g_dy);
  F.w = (double*)rel_ptr(L, slot, sm, RL_W, L->g_w);
}

// =====================================================================================
// Sign tables of the augmented constraint matrix (§IV-B, eq.`MALP matrix form`).
// Check j with cut V, variable i = N(j)[t]: A_ji = a s, a = +1 on V else -1 (eq.`constraints`
// P:107-110), s = -1 if gamma_i < 0.  A_ji < 0 <=> (i in V) == flipped.
// b_j = |V| - 1 - sum_{i in N(j), flipped} a_ji.  Returns p (rows), n_act (standard columns
// with >= 1 row), ||b||_inf.
// =====================================================================================
__device__ ALP_HEAVY void build_signs(const Frame& F, bool want_b, int& p_out, int& nact_out,
                            double& bmax_out) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  int p = 0;
  double bmax = 0.0;
  for (int j = F.lane; j < C.m; j += 32) {
    uint16_t mk = F.mask[j];
    uint16_t s = 0;
    if (mk & PRESENT) {
      int deg = ALP_G_CHK_DEG(C)[j];
      int nflipV = 0, nflipNotV = 0;
      for (int t = 0; t < deg; ++t) {
        int i = chk_nb(C, j, t);
        int inV = (mk >> t) & 1, fl = F.flip[i];
        if (inV == fl) s |= (uint16_t)(1u << t);
        if (fl) {
          if (inV) ++nflipV;
          else ++nflipNotV;
        }
      }
      s |= PRESENT;
      ++p;
      if (want_b) {
        double bj = (double)(__popc(mk & 0x7fff) - 1) - (double)(nflipV - nflipNotV);
        F.b[j] = bj;
        bmax = fmax(bmax, fabs(bj));
      }
    }
    F.sgnC_()[j] = s;
  }
  __syncwarp();
  int nact = 0;
  for (int i = F.lane; i < C.n; i += 32) {
    int dv = ALP_G_VAR_DEG(C)[i];
    uint8_t s = 0;
    for (int k = 0; k < dv; ++k) {
      int j = var_ck(C, i, k);
      int t = C.var_slot[i * C.dv + k];
      uint16_t sc = F.sgnC_()[j];
      if (sc & PRESENT) {
        s |= (uint8_t)(1u << k);
        if ((sc >> t) & 1) s |= (uint8_t)(1u << (4 + k));
      }
    }
    F.sgnV_()[i] = s;
    nact += (s & 0xf) ? 1 : 0;
  }
  p_out = wsumi(p);
  nact_out = wsumi(nact);
  bmax_out = wmax(bmax);
  __syncwarp();
}

// =====================================================================================
// Alg. 2 + MALP-A / MALP-B pool update (Alg. 3 lines 5-11 P:224-235).
// Every check reads the same u^{k-1}.  A present cut that is active (slack <= tau_act,
// C-4) excludes its check (line 6, Cor. 2 P:208-213); MALP-B drops inactive cuts first.
// S = {u_i > 1/2}; |S| even -> toggle i* = argmin |u_i - 1/2| (lowest position on ties,
// C-2); violated iff lhs < 1 - tau_viol (C-3) -> the check's cut is replaced (line 8-9).
// Returns warp-uniform "changed".
// =====================================================================================
__device__ ALP_HEAVY bool cut_search(const Frame& F, const Params& P) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  bool changed = false;
  for (int j = F.lane; j < C.m; j += 32) {
    int deg = ALP_G_CHK_DEG(C)[j];
    double uu[DCMAX];
#pragma unroll
    for (int t = 0; t < DCMAX; ++t) uu[t] = (t < deg) ? F.u[chk_nb(C, j, t)] : 0.0;
    uint16_t mk = F.mask[j];
    if (mk & PRESENT) {
      double lhs = 0.0;
#pragma unroll
      for (int t = 0; t < DCMAX; ++t)
        if (t < deg) lhs += ((mk >> t) & 1) ? (1.0 - uu[t]) : uu[t];
      if (lhs - 1.0 <= P.tau_act) continue;   // active cut: check skipped
      if (P.variant == 1) F.mask[j] = 0;       // MALP-B: remove the inactive cut
    }
    int S = 0, cnt = 0, istar = 0;
    double best = 4.0;
#pragma unroll
    for (int t = 0; t < DCMAX; ++t) {
      if (t < deg) {
        if (uu[t] > 0.5) {
          S |= 1 << t;
          ++cnt;
        }
        double dd = fabs(uu[t] - 0.5);
        if (dd < best) {
          best = dd;
          istar = t;
        }
      }
    }
    int V = (cnt & 1) ? S : (S ^ (1 << istar));
    double lhs = 0.0;
#pragma unroll
    for (int t = 0; t < DCMAX; ++t)
      if (t < deg) lhs += ((V >> t) & 1) ? (1.0 - uu[t]) : uu[t];
    if (lhs < 1.0 - P.tau_viol) {
      F.mask[j] = (uint16_t)(V | PRESENT);
      changed = true;
    }
  }
  __syncwarp();
  return __any_sync(FULL, changed);
}

// =====================================================================================
// Preconditioner build, part 1: rank the columns by weight (Alg. 7 needs "the maximum
// weight d_i" among DEG1; weight d^2 = x/z gives the same order, C-10).
// Valid columns (>= 1 present row; degree 0 in the extended Tanner graph otherwise) are
// compacted in ascending column order with the 32-bit key ~bits(float(d^2)) (ascending key =
// descending weight), then a stable LSD radix sort (8 passes of 4 bits, per-lane contiguous
// chunks, passes whose digit is the same for every key skipped) orders them: descending float
// weight, ascending column on equal floats.  Runs of equal float keys are then re-ordered by the exact fp64 weight (ties
// -> lower column).  Result: order[r] = column of rank r (r < nv), returns nv.
// Buffers (shared window, sort phase): kA/kB u32[Q], cA/cB u16[Q]; order
// u16[Q] must not overlap them (layout: s_order, then s_sortk).
// =====================================================================================
__device__ ALP_HEAVY int sort_columns(const Frame& F) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const Layout& L = *F.L;
  const uint16_t* __restrict__ sgnC = F.sgnC_();
  const uint8_t* __restrict__ sgnV = F.sgnV_();
  const double* __restrict__ d2 = F.d2;
  ALP_GL_SM(d2);
  uint32_t* kA = F.S<uint32_t>(L.s_sortk);
  uint32_t* kB = kA + C.Q;
  uint16_t* cA = reinterpret_cast<uint16_t*>(kB + C.Q);
  uint16_t* cB = cA + C.Q;
  uint16_t* order = F.S<uint16_t>(L.s_order);
  uint32_t* offs = F.S<uint32_t>(L.s_sorth);   // [16 digits][32 lanes]
  const unsigned lt = (1u << F.lane) - 1u;
  int nv = 0;
  // compaction of the valid columns with their keys, four 32-column chunks per step so that
  // the d^2 loads (slot array, L1/L2) of a step are in flight together
  for (int cb = 0; cb < C.Q; cb += 128) {
    bool valid[4];
    uint32_t kk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = cb + 32 * u + F.lane;
      const int cc = min(c, C.Q - 1);
      valid[u] = (c < C.Q) && ((cc < C.n) ? ((sgnV[cc] & 0xf) != 0) : ((sgnC[cc - C.n] & PRESENT) != 0));
      kk[u] = ~(__float_as_uint(__double2float_rn(d2[cc])) & 0x7fffffffu);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned bal = __ballot_sync(FULL, valid[u]);
      if (valid[u]) {
        const int at = nv + __popc(bal & lt);
        kA[at] = kk[u];
        cA[at] = (uint16_t)(cb + 32 * u + F.lane);
      }
      nv += __popc(bal);
    }
  }
  __syncwarp();
  // LSD radix sort, 8 passes of 4-bit digits.  Lane l owns the contiguous chunk
  // [l*ch, (l+1)*ch) of the current sequence, so lane order = sequence order and the scatter
  // (digit base + earlier lanes' counts + this lane's running count) is stable.  Per-lane digit
  // counts live in registers (four packed u64, 16 bits per digit: ch <= 65535).
  const int ch = ((nv + 31) >> 5) | 1;   // odd chunk stride: the lanes' u32 loads hit distinct banks
  const int lo = min(nv, F.lane * ch), hi = min(nv, lo + ch);
  uint32_t* ks = kA;
  uint32_t* kd = kB;
  uint16_t* cs = cA;
  uint16_t* cd = cB;
  for (int sh = 0; sh < 32; sh += 4) {
    unsigned long long q0 = 0ull, q1 = 0ull, q2 = 0ull, q3 = 0ull;
#pragma unroll 4
    for (int i = lo; i < hi; ++i) {
      const int dg = (ks[i] >> sh) & 0xf;
      const unsigned long long inc = 1ull << (16 * (dg & 3));
      const int w = dg >> 2;
      q0 += (w == 0) ? inc : 0ull;
      q1 += (w == 1) ? inc : 0ull;
      q2 += (w == 2) ? inc : 0ull;
      q3 += (w == 3) ? inc : 0ull;
    }
    // exclusive offsets per (digit, lane) in a [16 digits][32 lanes] table (conflict-free);
    // a pass whose digit is the same for every key is skipped
    int base = 0;
    bool skip = false;
#pragma unroll
    for (int dg = 0; dg < 16; ++dg) {
      const unsigned long long qw = (dg < 4) ? q0 : (dg < 8) ? q1 : (dg < 12) ? q2 : q3;
      const int cnt = (int)((qw >> (16 * (dg & 3))) & 0xffffull);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (F.lane >= o) incl += y;
      }
      const int tot = __shfl_sync(FULL, incl, 31);
      skip |= (tot == nv);
      offs[dg * 32 + F.lane] = (uint32_t)(base + incl - cnt);
      base += tot;
    }
    if (skip) {   // warp-uniform (tot is)
      __syncwarp();
      continue;
    }
    __syncwarp();
    // this lane's 16 running digit offsets packed two per register (u16: Q <= 65535), so the
    // scatter has no read-after-write chain through shared memory
    // (eight named registers with select chains: an indexed array would go to local memory)
#define ALP_OFF2(w) (offs[(2 * (w)) * 32 + F.lane] | (offs[(2 * (w) + 1) * 32 + F.lane] << 16))
    uint32_t o0 = ALP_OFF2(0), o1 = ALP_OFF2(1), o2 = ALP_OFF2(2), o3 = ALP_OFF2(3), o4 = ALP_OFF2(4),
             o5 = ALP_OFF2(5), o6 = ALP_OFF2(6), o7 = ALP_OFF2(7);
#undef ALP_OFF2
#pragma unroll 2
    for (int i = lo; i < hi; ++i) {
      const uint32_t k = ks[i];
      const uint16_t cv = cs[i];
      const int dg = (k >> sh) & 0xf;
      const int w = dg >> 1, hs = 16 * (dg & 1);
      const uint32_t lo4 = (w & 2) ? ((w & 1) ? o3 : o2) : ((w & 1) ? o1 : o0);
      const uint32_t hi4 = (w & 2) ? ((w & 1) ? o7 : o6) : ((w & 1) ? o5 : o4);
      const uint32_t at = (((w & 4) ? hi4 : lo4) >> hs) & 0xffffu;
      const uint32_t inc = 1u << hs;
      o0 += (w == 0) ? inc : 0u;
      o1 += (w == 1) ? inc : 0u;
      o2 += (w == 2) ? inc : 0u;
      o3 += (w == 3) ? inc : 0u;
      o4 += (w == 4) ? inc : 0u;
      o5 += (w == 5) ? inc : 0u;
      o6 += (w == 6) ? inc : 0u;
      o7 += (w == 7) ? inc : 0u;
      kd[at] = k;
      cd[at] = cv;
    }
    __syncwarp();
    uint32_t* tk = ks; ks = kd; kd = tk;
    uint16_t* tc = cs; cs = cd; cd = tc;
  }
  for (int r = F.lane; r < C.Q; r += 32) order[r] = (r < nv) ? cs[r] : NONE16;
  __syncwarp();
  // Equal float keys are ordered by column; that is the exact (fp64 weight desc, column asc)
  // order unless some adjacent pair inside a float tie has a strictly smaller exact weight
  // first.  Checked in parallel; only then does the serial fix-up below run (e.g. never at
  // IPM iteration 0, where every weight is exactly 1).
  bool tie = false;
  for (int r = F.lane; r + 1 < nv; r += 32) {
    if (ks[r] != ks[r + 1]) continue;   // only equal float keys need the exact weights
    if (d2[order[r]] < d2[order[r + 1]]) tie = true;
  }
  if (__any_sync(FULL, tie)) {
    if (F.lane == 0) {
      int r = 0;
      while (r + 1 < nv) {
        const uint32_t key = ks[r];
        int e = r + 1;
        while (e < nv && ks[e] == key) ++e;
        for (int a = r + 1; a < e; ++a) {   // insertion sort by (d2 desc, column asc)
          const uint16_t ca = order[a];
          const double wa = d2[ca];
          int b = a - 1;
          while (b >= r) {
            const uint16_t cb = order[b];
            const double wb = d2[cb];
            if (!((wa > wb) || (wa == wb && ca < cb))) break;
            order[b + 1] = cb;
            --b;
          }
          order[b + 1] = ca;
        }
        r = e;
      }
    }
    __syncwarp();
  }
  return nv;
}

// Alg. 7 lines 5-9, the p picks.  DEG1 as a rank bitmap: bit r set <=> the column of rank r
// currently has exactly one live row; "the maximum-weight column in DEG1" (line 6) is the
// first set bit.  Pick k: r -> its live row R = xrR[r] (XOR of the column's live rows, kept per
// rank) and column c = order[r]; record it (line 7); kill row R (line 8): the <= d_c + 1 columns
// of R (their ranks precomputed in rrank[R][.]) lose a live row, entering DEG1 at degree 1 and
// leaving it at degree 0 (line 9).  The critical path of a pick is three dependent shared-memory
// loads (xrR, rrank, cntR / xrR) plus the bitmap search and update.
// Register variant: lane l owns bitmap words l, 32 + l, ... (K per lane), so the search is a
// ballot and the updates are shuffles — no shared-memory atomics on the pick's critical path.
template <int K, int RS>
__device__ __forceinline__ void peel_picks_reg(const Frame& F, int p, const uint16_t* __restrict__ order,
                                               const uint16_t* __restrict__ rrank,
                                               uint8_t* __restrict__ cntR, uint16_t* __restrict__ xrR,
                                               const unsigned long long* bm, uint16_t* pos,
                                               uint16_t* pcol, uint16_t* prow) {
  const int W = F.C->W;
  unsigned long long wd[K];
#pragma unroll
  for (int kk = 0; kk < K; ++kk) {
    const int w = 32 * kk + F.lane;
    wd[kk] = (w < W) ? bm[w] : 0ull;
  }
  for (int k = 0; k < p; ++k) {
    int r = 0;
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      const unsigned bal = __ballot_sync(FULL, wd[kk] != 0ull);
      if (bal) {
        const int src = __ffs(bal) - 1;
        const unsigned long long w0 = __shfl_sync(FULL, wd[kk], src);
        r = (32 * kk + src) * 64 + (__ffsll((long long)w0) - 1);
        break;
      }
    }
    const int R = xrR[r];
    if (F.lane == 0) {
      pos[R] = (uint16_t)k;
      pcol[R] = order[r];
      prow[k] = (uint16_t)R;
    }
    int upd = -1;   // rank << 1 | (degree now 1) ; -1: no DEG1 change
    const int rr = (F.lane < RS) ? (int)rrank[R * RS + F.lane] : (int)NONE16;
    if (rr != (int)NONE16) {
      const int nc = (int)cntR[rr] - 1;
      cntR[rr] = (uint8_t)nc;
      xrR[rr] = (uint16_t)(xrR[rr] ^ R);
      if (nc <= 1) upd = (rr << 1) | (nc == 1 ? 1 : 0);
    }
    // apply the (<= d_c + 1) bit updates in the owning lanes: shuffles issued back to back,
    // branch-free set / clear masks per owned word (a column changes at most once per pick;
    // measured faster than enumerating the active lanes by ballot)
    int us[RS];
#pragma unroll
    for (int t = 0; t < RS; ++t) us[t] = __shfl_sync(FULL, upd, t);
    unsigned long long setm[K], clrm[K];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) setm[kk] = clrm[kk] = 0ull;
#pragma unroll
    for (int t = 0; t < RS; ++t) {
      const int u = us[t];
      const int rk = u >> 1;
      const bool mine = (u >= 0) && (((rk >> 6) & 31) == F.lane);
      const unsigned long long bit = mine ? (1ull << (rk & 63)) : 0ull;
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const unsigned long long b = ((rk >> 11) == kk) ? bit : 0ull;
        setm[kk] |= (u & 1) ? b : 0ull;
        clrm[kk] |= (u & 1) ? 0ull : b;
      }
    }
#pragma unroll
    for (int kk = 0; kk < K; ++kk) wd[kk] = (wd[kk] | setm[kk]) & ~clrm[kk];
    __syncwarp();
  }
}

// Batched variant of the same picks (-DALP_PEEL_BATCH; measured no faster).  A batch
// takes the first NB = 32 / RS set bits of DEG1, ranks r_0 < r_1 < ... with live rows R_g, and
// makes all picks of its longest prefix that the sequential loop above would make in the same
// order: candidate i is pick k + i when
//   (a) R_i differs from R_0..R_{i-1} (else the earlier kill empties r_i's column), and
//   (b) every column that the kills of R_0..R_{i-1} can bring to degree 1 ranks after r_i.
// For (b) the "threat" of row R_g is the lowest rank among its columns other than r_g with >= 2
// live rows (the only columns a kill can move into DEG1; a degree-1 column of R_g other than
// r_g ranked before r_i would itself be a candidate with row R_g and fail (a)).  By induction
// the sequential loop then finds r_i at the head of DEG1 after the first i picks.  The kills
// of a batch commute (live-row count decrement, XOR of the row id), so lane (g, t) applies row
// R_g's column t with shared-memory atomics on the containing 32-bit words, and the DEG1 bits
// (Refinement of (b): a column with c >= 3 live rows is a threat only if >= c - 1 of the NB
// candidate rows hold it — the prefix's kills are a subset of the candidates'.)
// follow the final counts.  Lane layout: g = lane / RS (candidate), t = lane % RS (column).
template <int K, int RS>
__device__ __forceinline__ void peel_picks_batch(const Frame& F, int p, const uint16_t* __restrict__ order,
                                                 const uint16_t* __restrict__ rrank,
                                                 uint8_t* cntR, uint16_t* xrR,
                                                 unsigned long long* bm, uint16_t* pos,
                                                 uint16_t* pcol, uint16_t* prow) {
  constexpr int NB = 32 / RS;
  constexpr int BIG = 0x7fffffff;
  const int W = F.C->W;
  const int g = F.lane / RS, t = F.lane % RS;
  unsigned long long wd[K > 0 ? K : 1];
#pragma unroll
  for (int kk = 0; kk < K; ++kk) {
    const int w = 32 * kk + F.lane;
    wd[kk] = (w < W) ? bm[w] : 0ull;
  }
  for (int k = 0; k < p;) {
    // the first NB set bits of DEG1 in rank order (warp-uniform)
    int cand[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) cand[i] = BIG;
    int nc = 0;
    // K > 0: lane l holds words l, 32 + l, ... in registers; K == 0 (large codes): scan the
    // shared bitmap 32 words at a time
    for (int kk = 0; ((K > 0) ? (kk < K) : (32 * kk < W)) && nc < NB; ++kk) {
      unsigned long long wk = 0ull;
      if constexpr (K > 0) {
#pragma unroll
        for (int q = 0; q < (K > 0 ? K : 1); ++q) wk = (q == kk) ? wd[q] : wk;
      } else {
        const int w = 32 * kk + F.lane;
        wk = (w < W) ? bm[w] : 0ull;
      }
      unsigned bal = __ballot_sync(FULL, wk != 0ull);
      while (bal != 0u && nc < NB) {
        const int src = __ffs(bal) - 1;
        unsigned long long w0 = __shfl_sync(FULL, wk, src);
        while (w0 != 0ull && nc < NB) {
          const int r = (32 * kk + src) * 64 + (__ffsll((long long)w0) - 1);
#pragma unroll
          for (int i = 0; i < NB; ++i) cand[i] = (i == nc) ? r : cand[i];
          ++nc;
          w0 &= w0 - 1ull;
        }
        bal &= bal - 1u;
      }
    }
    int rg = cand[0];
#pragma unroll
    for (int i = 1; i < NB; ++i) rg = (g == i) ? cand[i] : rg;
    const bool vg = g < nc;
    const int Rg = vg ? (int)xrR[rg] : -1;
    const int x = vg ? (int)rrank[Rg * RS + t] : (int)NONE16;
    const bool xv = x != (int)NONE16;
    const int c = xv ? (int)cntR[x] : 0;
    // a column with c live rows reaches degree 1 only if >= c - 1 of the candidate rows hold it
    const unsigned same = __match_any_sync(FULL, xv ? (unsigned)x : 0x10000u + (unsigned)F.lane);
    int thr = (xv && x != rg && c >= 2 && c - __popc(same) <= 1) ? x : BIG;
#pragma unroll
    for (int o = 1; o < RS; o <<= 1) thr = min(thr, __shfl_xor_sync(FULL, thr, o));
    int Rs[NB], Th[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      Rs[i] = __shfl_sync(FULL, Rg, i * RS);
      Th[i] = __shfl_sync(FULL, thr, i * RS);
    }
    // longest valid prefix (warp-uniform)
    int nb = 1, tmin = Th[0];
#pragma unroll
    for (int i = 1; i < NB; ++i) {
      bool ok = (nb == i) && (i < nc) && (k + i < p) && (tmin > cand[i]);
#pragma unroll
      for (int j = 0; j < i; ++j) ok = ok && (Rs[j] != Rs[i]);
      if (ok) {
        nb = i + 1;
        tmin = min(tmin, Th[i]);
      }
    }
    // kill R_0..R_{nb-1}: count and XOR updates commute -> atomics on the containing words
    const bool act = (g < nb) && xv;
    const unsigned accm = __ballot_sync(FULL, act);
    if (act) {
      const uintptr_t ac = (uintptr_t)(cntR + x), ax = (uintptr_t)(xrR + x);
      atomicSub(reinterpret_cast<unsigned*>(ac & ~(uintptr_t)3), 1u << (8 * (ac & 3)));
      atomicXor(reinterpret_cast<unsigned*>(ax & ~(uintptr_t)3), (unsigned)Rg << (8 * (ax & 2)));
      // DEG1 bit from the final count c - (accepted rows holding x): the same idempotent
      // update from every lane that shares x
      const int fc = c - __popc(same & accm);
      if (fc == 1) atomicOr(&bm[x >> 6], 1ull << (x & 63));
      else if (fc == 0) atomicAnd(&bm[x >> 6], ~(1ull << (x & 63)));
    }
    if (t == 0 && g < nb) {
      pos[Rg] = (uint16_t)(k + g);
      pcol[Rg] = order[rg];
      prow[k + g] = (uint16_t)Rg;
    }
    __syncwarp();
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      const int w = 32 * kk + F.lane;
      wd[kk] = (w < W) ? bm[w] : 0ull;
    }
    k += nb;
#ifdef ALP_PEEL_COUNT
    if (F.lane == 0) {   // diagnostics: batches in the sort clock, picks in the peel clock
      ALP_CYC(F)[CY_SORT] += 1;
      ALP_CYC(F)[CY_PEEL] += nb;
    }
#endif
  }
}

// Shared-memory bitmap variant for large codes (W > 128 words).
__device__ __noinline__ void peel_picks_smem(const Frame& F, int p, const uint16_t* order,
                                             const uint16_t* rrank, int RS, uint8_t* cntR,
                                             uint16_t* xrR, unsigned long long* bm, uint16_t* pos,
                                             uint16_t* pcol, uint16_t* prow) {
  const int W = F.C->W;
  for (int k = 0; k < p; ++k) {
    int r = 0;
    for (int base = 0; base < W; base += 32) {
      unsigned long long wd = (base + F.lane < W) ? bm[base + F.lane] : 0ull;
      unsigned bal = __ballot_sync(FULL, wd != 0ull);
      if (bal) {
        int src = __ffs(bal) - 1;
        unsigned long long w0 = __shfl_sync(FULL, wd, src);
        r = (base + src) * 64 + (__ffsll((long long)w0) - 1);
        break;
      }
    }
    const int R = xrR[r];
    if (F.lane == 0) {
      pos[R] = (uint16_t)k;
      pcol[R] = order[r];
      prow[k] = (uint16_t)R;
    }
    __syncwarp();
    const int rr = (F.lane < RS) ? (int)rrank[R * RS + F.lane] : (int)NONE16;
    if (rr != (int)NONE16) {
      const int nc = (int)cntR[rr] - 1;
      cntR[rr] = (uint8_t)nc;
      xrR[rr] = (uint16_t)(xrR[rr] ^ R);
      if (nc == 1) atomicOr(&bm[rr >> 6], 1ull << (rr & 63));
      else if (nc == 0) atomicAnd(&bm[rr >> 6], ~(1ull << (rr & 63)));
    }
    __syncwarp();
  }
}

// Part 2: Alg. 7 initialisation: rank of every valid column, live-row count and
// XOR of live rows per rank, the ranks of each present row's columns, the DEG1 bitmap.
__device__ ALP_HEAVY void peel_columnwise(const Frame& F, int p) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const Layout& L = *F.L;
#ifdef ALP_PEEL_SPLIT
  const long long tp0 = clock64();
#endif
  const uint16_t* order = F.S<uint16_t>(L.s_order);
  uint16_t* rank = F.S<uint16_t>(L.s_rank);
  uint8_t* cntR = F.S<uint8_t>(L.s_cnt);
  uint16_t* xrR = F.S<uint16_t>(L.s_xr);
  unsigned long long* bm = F.S<unsigned long long>(L.s_bm);
  uint16_t* rrank = F.S<uint16_t>(L.s_rrank);
  uint16_t* pos = F.S<uint16_t>(L.s_pos);
  uint16_t* pcol = F.S<uint16_t>(L.s_pcol);
  uint16_t* prow = F.S<uint16_t>(L.s_prow);
  const int RS = L.RS;
  for (int c = F.lane; c < C.Q; c += 32) rank[c] = NONE16;
  for (int w = F.lane; w < C.W; w += 32) bm[w] = 0ull;
  __syncwarp();
  for (int r = F.lane; r < C.Q; r += 32) {
    uint16_t c = order[r];
    if (c != NONE16) rank[c] = (uint16_t)r;
  }
  __syncwarp();
  for (int c = F.lane; c < C.Q; c += 32) {
    const int rk = rank[c];
    if (rk == (int)NONE16) continue;   // no present row (C-10): never in DEG1
    int cn = 0, x = 0;
    if (c < C.n) {
      uint8_t s = F.sgnV_()[c];
      int dv = ALP_G_VAR_DEG(C)[c];
      for (int k = 0; k < dv; ++k)
        if ((s >> k) & 1) {
          ++cn;
          x ^= var_ck(C, c, k);
        }
    } else {
      cn = 1;
      x = c - C.n;
    }
    cntR[rk] = (uint8_t)cn;
    xrR[rk] = (uint16_t)x;
    if (cn == 1) atomicOr(&bm[rk >> 6], 1ull << (rk & 63));
  }
  for (int R = F.lane; R < C.m; R += 32) {
    if (!(F.sgnC_()[R] & PRESENT)) continue;
    const int deg = ALP_G_CHK_DEG(C)[R];
    for (int t = 0; t < RS; ++t)
      rrank[R * RS + t] = (t < deg) ? rank[chk_nb(C, R, t)] : (t == deg ? rank[C.n + R] : NONE16);
  }
  __syncwarp();
#ifdef ALP_PEEL_SPLIT
  if (F.lane == 0) ALP_CYC(F)[CY_CUT] += clock64() - tp0;   // diagnostics: peel initialisation
#endif
#ifdef ALP_PEEL_BATCH
  if (C.W <= 32 && RS == 8) peel_picks_batch<1, 8>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 32 && RS == 16) peel_picks_batch<1, 16>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 128 && RS == 8) peel_picks_batch<4, 8>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 128 && RS == 16) peel_picks_batch<4, 16>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (RS == 8) peel_picks_batch<0, 8>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else peel_picks_batch<0, 16>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
#else
  if (C.W <= 32 && RS == 8) peel_picks_reg<1, 8>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 32 && RS == 16) peel_picks_reg<1, 16>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 128 && RS == 8) peel_picks_reg<4, 8>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else if (C.W <= 128 && RS == 16) peel_picks_reg<4, 16>(F, p, order, rrank, cntR, xrR, bm, pos, pcol, prow);
  else peel_picks_smem(F, p, order, rrank, RS, cntR, xrR, bm, pos, pcol, prow);
#endif
}

// =====================================================================================
// Alg. 8, row-wise greedy search for the MTS, with diagonal expansion (line 14;
// G11), SURVEY f-1.  Residual matrix state per row: live-column count and XOR of the live
// column ids (the unique live column of a degree-1 row); a row bitmap of the degree-1 rows
// not yet represented ("any degree-1 row" = the lowest index, as the oracle); the columns in
// ascending weight order (ties -> lower index, C-10) for the erasures of line 11.  Every step
// removes one column (picked on line 8 or erased on line 11), so the loop ends within q steps;
// it stops as soon as no unrepresented row has a live column.  The pick sequence is lower
// triangular; it is stored reversed, so that A_M is upper triangular in pivot order
// like Alg. 7's and the level / sweep machinery is shared.  Returns the number of pivots (= p).
// Arrays (peel window): asc = reversed `order` with runs of equal weight re-reversed;
// rdeg (u8, bit 7 = represented) over `cnt`, rxor over `xr`, column-alive flags over `rank`,
// row bitmap over `bm`; picks go to pcol / prow in reverse.
template <int K>
__device__ __noinline__ void peel_rowwise_t(const Frame& F, int p, int nv) {
  const DCode C = *F.C;
  const Layout& L = *F.L;
  uint16_t* order = F.S<uint16_t>(L.s_order);
  uint8_t* rdeg = F.S<uint8_t>(L.s_cnt);
  uint16_t* rxor = F.S<uint16_t>(L.s_xr);
  uint8_t* alive = reinterpret_cast<uint8_t*>(F.S<uint16_t>(L.s_rank));
  unsigned long long* bm = F.S<unsigned long long>(L.s_bm);
  uint16_t* pos = F.S<uint16_t>(L.s_pos);
  uint16_t* pcol = F.S<uint16_t>(L.s_pcol);
  uint16_t* prow = F.S<uint16_t>(L.s_prow);
  const uint16_t* sgnC = F.sgnC_();
  const uint8_t* sgnV = F.sgnV_();
  const double* d2 = F.d2;
  const int m = C.m, n = C.n;
  // ascending weight order: reverse `order`, then restore ascending column order inside runs of
  // exactly equal weight (lane 0; only long at the first IPM step, where all weights are 1)
  for (int r = F.lane; r < nv / 2; r += 32) {
    const uint16_t a = order[r], b = order[nv - 1 - r];
    order[r] = b;
    order[nv - 1 - r] = a;
  }
  __syncwarp();
  if (F.lane == 0) {
    int r = 0;
    while (r < nv) {
      const double w = d2[order[r]];
      int e = r + 1;
      while (e < nv && d2[order[e]] == w) ++e;
      for (int a = r, b = e - 1; a < b; ++a, --b) {
        const uint16_t t = order[a];
        order[a] = order[b];
        order[b] = t;
      }
      r = e;
    }
  }
  const int WR = (m + 63) >> 6;
  for (int c = F.lane; c < C.Q; c += 32) alive[c] = 0;
  for (int w = F.lane; w < WR; w += 32) bm[w] = 0ull;
  __syncwarp();
  for (int r = F.lane; r < nv; r += 32) alive[order[r]] = 1;
  int live = 0;
  for (int j = F.lane; j < m; j += 32) {
    int dg = 0, x = 0;
    if (sgnC[j] & PRESENT) {
      const int deg = ALP_G_CHK_DEG(C)[j];
      for (int t = 0; t < deg; ++t) {
        const int c = ALP_G_CHK_VAR(C)[j * C.dc + t];
        ++dg;
        x ^= c;
      }
      ++dg;          // the slack column n + j
      x ^= n + j;
      ++live;
    }
    rdeg[j] = (uint8_t)dg;
    rxor[j] = (uint16_t)x;
  }
  live = wsumi(live);
  __syncwarp();
  unsigned long long wd[K];
#pragma unroll
  for (int kk = 0; kk < K; ++kk) wd[kk] = 0ull;   // no degree-1 row yet (every row has >= 2 columns)
  int k = 0, e = 0;
  while (live > 0) {
    int j = -1;
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      const unsigned bal = __ballot_sync(FULL, wd[kk] != 0ull);
      if (bal && j < 0) {
        const int src = __ffs(bal) - 1;
        const unsigned long long w0 = __shfl_sync(FULL, wd[kk], src);
        j = (32 * kk + src) * 64 + (__ffsll((long long)w0) - 1);
      }
    }
    int c;
    if (j >= 0) {                       // line 7-9: degree-1 row j, its unique live column
      c = rxor[j];
      if (F.lane == 0) {
        prow[k] = (uint16_t)j;
        pcol[k] = (uint16_t)c;
        rdeg[j] = (uint8_t)(rdeg[j] | 0x80);   // represented
      }
      ++k;
      --live;
    } else {                            // line 11: erase the lowest-weight live column
      while (true) {
        const int r = e + F.lane;
        const bool al = (r < nv) && alive[order[r]];
        const unsigned bal = __ballot_sync(FULL, al);
        if (bal) {
          e += __ffs(bal) - 1;
          break;
        }
        e += 32;
      }
      c = order[e];
    }
    if (F.lane == 0) alive[c] = 0;
    __syncwarp();
    // remove column c from A~: its rows lose one live column
    int r = -1;
    if (c < n) {
      if (F.lane < DVMAX && ((sgnV[c] >> F.lane) & 1)) r = ALP_G_VAR_CHK(C)[c * C.dv + F.lane];
    } else if (F.lane == 0) {
      r = c - n;
    }
    int upd = -1, dead = 0;
    if (r >= 0) {
      const int dg = rdeg[r];
      const int nd = (dg & 0x7f) - 1;
      rdeg[r] = (uint8_t)((dg & 0x80) | nd);
      rxor[r] = (uint16_t)(rxor[r] ^ c);
      if (!(dg & 0x80) || r == j) {     // DEG1 holds only unrepresented rows (j just left it)
        if (nd == 1 && !(dg & 0x80)) upd = (r << 1) | 1;
        else if (nd == 0) {
          upd = r << 1;
          dead = (r != j) ? 1 : 0;      // an unrepresented row left without columns
        }
      }
    }
    live -= __popc(__ballot_sync(FULL, dead != 0));
    int us[DVMAX];
#pragma unroll
    for (int t = 0; t < DVMAX; ++t) us[t] = __shfl_sync(FULL, upd, t);
#pragma unroll
    for (int t = 0; t < DVMAX; ++t) {
      const int u = us[t];
      if (u < 0) continue;
      const int rr = u >> 1;
      const int wi = rr >> 6;
      if ((wi & 31) == F.lane) {
        const unsigned long long bit = 1ull << (rr & 63);
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
          if ((wi >> 5) == kk) wd[kk] = (u & 1) ? (wd[kk] | bit) : (wd[kk] & ~bit);
      }
    }
    __syncwarp();
  }
  // diagonal expansion (line 14): every present row not represented gets its slack column
  const unsigned lt = (1u << F.lane) - 1u;
  for (int j0 = 0; j0 < m; j0 += 32) {
    const int j = j0 + F.lane;
    const bool need = (j < m) && (sgnC[j] & PRESENT) && !(rdeg[j] & 0x80);
    const unsigned bal = __ballot_sync(FULL, need);
    if (need) {
      const int at = k + __popc(bal & lt);
      prow[at] = (uint16_t)j;
      pcol[at] = (uint16_t)(n + j);
    }
    k += __popc(bal);
  }
  __syncwarp();
  // reverse into upper-triangular pivot order; pcol / pos become indexed by row (as Alg. 7's)
  for (int t = F.lane; t < k / 2; t += 32) {
    const uint16_t ra = prow[t], rb = prow[k - 1 - t];
    const uint16_t ca = pcol[t], cb = pcol[k - 1 - t];
    prow[t] = rb;
    prow[k - 1 - t] = ra;
    pcol[t] = cb;
    pcol[k - 1 - t] = ca;
  }
  __syncwarp();
  // pcol[] was filled in pick order; Alg. 7 keeps it indexed by row: convert through pos
  for (int t = F.lane; t < k; t += 32) pos[prow[t]] = (uint16_t)t;
  __syncwarp();
  for (int t = F.lane; t < k; t += 32) rxor[prow[t]] = pcol[t];   // row -> column (rxor is dead)
  __syncwarp();
  for (int j = F.lane; j < m; j += 32) pcol[j] = rxor[j];
  __syncwarp();
  (void)p;
}

__device__ ALP_HEAVY void peel_rowwise(const Frame& F, int p, int nv) {
  const int WR = (F.C->m + 63) >> 6;
  if (WR <= 32) peel_rowwise_t<1>(F, p, nv);
  else if (WR <= 128) peel_rowwise_t<4>(F, p, nv);
  else peel_rowwise_t<16>(F, p, nv);
}

// =====================================================================================
// Alg. 6, incremental greedy search for the MTS with the Triangulation Step of
// Alg. 5, SURVEY f-1 (precond = 3; O(q) triangulations of O(E) each — a reference
// variant for the E5 comparison, not a throughput path).  Columns are tried in the ranked order
// of sort_columns (decreasing weight, ties -> lower index; columns without a present row are
// excluded, they can never be triangulated); column pi_i is kept iff M u {pi_i} passes the
// Triangulation Step, until |M| = p (the paper's argument P:656: the slack columns guarantee
// it).  Triangulation Step (reading G10): repeatedly take the lowest-index row with exactly one
// live column of S, record (column, row), kill that column (its rows lose it; the row itself
// drops to degree 0); fails iff no row has degree 1 before |S| picks.  The final pick sequence
// of M is lower triangular; it is stored reversed (upper triangular in pivot order, like
// Alg. 7's), pcol indexed by row.
// Arrays (peel window): inM (u8) over `rank`, row degree (u8) over `cnt`, row XOR of live
// columns over `xr`; picks to prow / pcol.
__device__ __noinline__ int tri_step(const Frame& F, const uint8_t* inM, uint8_t* rdeg, uint16_t* rx,
                                     bool record, uint16_t* prow, uint16_t* pcol) {
  const DCode C = *F.C;
  const uint16_t* sgnC = F.sgnC_();
  const uint8_t* sgnV = F.sgnV_();
  const int m = C.m, n = C.n;
  int total = 0;
  for (int j = F.lane; j < m; j += 32) {
    int dg = 0, x = 0;
    if (sgnC[j] & PRESENT) {
      const int deg = ALP_G_CHK_DEG(C)[j];
      for (int t = 0; t < deg; ++t) {
        const int c = ALP_G_CHK_VAR(C)[j * C.dc + t];
        if (inM[c]) {
          ++dg;
          x ^= c;
        }
      }
      if (inM[n + j]) {
        ++dg;
        x ^= n + j;
        ++total;   // slack columns of S (each in exactly one row)
      }
    }
    rdeg[j] = (uint8_t)dg;
    rx[j] = (uint16_t)x;
  }
  for (int c = F.lane; c < n; c += 32) total += inM[c] ? 1 : 0;
  total = wsumi(total);
  __syncwarp();
  int picks = 0;
  while (picks < total) {
    int j = -1;
    for (int j0 = 0; j0 < m && j < 0; j0 += 32) {
      const int jj = j0 + F.lane;
      const unsigned bal = __ballot_sync(FULL, jj < m && rdeg[jj] == 1);
      if (bal) j = j0 + __ffs(bal) - 1;
    }
    if (j < 0) break;   // Alg. 5 line 5: no degree-1 row -> failure
    const int c = rx[j];
    if (record && F.lane == 0) {
      prow[picks] = (uint16_t)j;
      pcol[picks] = (uint16_t)c;
    }
    ++picks;
    __syncwarp();
    // line 8: zero column c (its rows, the picked row j among them, lose it)
    int r = -1;
    if (c < n) {
      if (F.lane < DVMAX && ((sgnV[c] >> F.lane) & 1)) r = ALP_G_VAR_CHK(C)[c * C.dv + F.lane];
    } else if (F.lane == 0) {
      r = c - n;
    }
    if (r >= 0) {
      rdeg[r] = (uint8_t)(rdeg[r] - 1);
      rx[r] = (uint16_t)(rx[r] ^ c);
    }
    __syncwarp();
  }
  return (picks == total) ? picks : -1;
}

__device__ __noinline__ void peel_incremental(const Frame& F, int p, int nv) {
  const DCode C = *F.C;
  const Layout& L = *F.L;
  const uint16_t* order = F.S<uint16_t>(L.s_order);
  uint8_t* inM = reinterpret_cast<uint8_t*>(F.S<uint16_t>(L.s_rank));
  uint8_t* rdeg = F.S<uint8_t>(L.s_cnt);
  uint16_t* rx = F.S<uint16_t>(L.s_xr);
  uint16_t* pos = F.S<uint16_t>(L.s_pos);
  uint16_t* pcol = F.S<uint16_t>(L.s_pcol);
  uint16_t* prow = F.S<uint16_t>(L.s_prow);
  for (int c = F.lane; c < C.Q; c += 32) inM[c] = 0;
  __syncwarp();
  int cnt = 0;
  for (int r = 0; r < nv && cnt < p; ++r) {   // Alg. 6 lines 5-10
    const int c = order[r];
    if (F.lane == 0) inM[c] = 1;
    __syncwarp();
    if (tri_step(F, inM, rdeg, rx, false, prow, pcol) >= 0) {
      ++cnt;
    } else {
      if (F.lane == 0) inM[c] = 0;
      __syncwarp();
    }
  }
  const int k = max(tri_step(F, inM, rdeg, rx, true, prow, pcol), 0);   // A_M in lower-triangular order
  // reverse into upper-triangular pivot order; pcol / pos become indexed by row (as Alg. 7's)
  for (int t = F.lane; t < k / 2; t += 32) {
    const uint16_t ra = prow[t], rb = prow[k - 1 - t];
    const uint16_t ca = pcol[t], cb = pcol[k - 1 - t];
    prow[t] = rb;
    prow[k - 1 - t] = ra;
    pcol[t] = cb;
    pcol[k - 1 - t] = ca;
  }
  __syncwarp();
  for (int t = F.lane; t < k; t += 32) pos[prow[t]] = (uint16_t)t;
  __syncwarp();
  for (int t = F.lane; t < k; t += 32) rx[prow[t]] = pcol[t];   // row -> column (rx is dead)
  __syncwarp();
  for (int j = F.lane; j < C.m; j += 32) pcol[j] = rx[j];
  __syncwarp();
}

// Sweep dependencies of the pivot on row R (A_M is upper triangular in pick order):
//  back  (A_M f = r):   the other pivot columns of row R -> their pivot rows (picked later)
//  fwd   (A_M^T z = g): the other present rows of column C_k (killed earlier)
// Encoded row | (coefficient < 0) << 31, in FIXED slots (back: position t in N(R), forward:
// position k in the column's check list) with DEP_NONE where there is none, so the arrays stay
// in registers (no dynamically indexed local arrays).
constexpr int DEP_NONE = 0x40000000;
template <int DCT>
__device__ __forceinline__ void back_deps(const Frame& F, int R, int (&deps)[DCT]) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const uint16_t* poc = F.S<uint16_t>(F.L->s_poc);
  const int deg = ALP_G_CHK_DEG(C)[R];
  const uint16_t s = F.sgnC_()[R];
  const int pc = F.S<uint16_t>(F.L->s_pcol)[R];
#pragma unroll
  for (int t = 0; t < DCT; ++t) {
    int v = DEP_NONE;
    if (t < deg) {
      const int c = ALP_G_CHK_VAR(C)[R * C.dc + t];
      const uint16_t rr = (c == pc) ? NONE16 : poc[c];
      if (rr != NONE16) v = (int)rr | (int)(((unsigned)(s >> t) & 1u) << 31);
    }
    deps[t] = v;
  }
}
__device__ __forceinline__ void fwd_deps(const Frame& F, int R, int (&deps)[DVMAX]) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const int c = F.S<uint16_t>(F.L->s_pcol)[R];
  const uint8_t s = (c < C.n) ? F.sgnV_()[c] : (uint8_t)0;
#pragma unroll
  for (int k = 0; k < DVMAX; ++k) {
    int v = DEP_NONE;
    if ((s >> k) & 1) {
      const int j = ALP_G_VAR_CHK(C)[c * C.dv + k];
      if (j != R) v = j | (int)(((unsigned)(s >> (4 + k)) & 1u) << 31);
    }
    deps[k] = v;
  }
}
// sign of the diagonal entry A[R, C_k]
__device__ __forceinline__ int diag_neg(const Frame& F, int R) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  int c = F.S<uint16_t>(F.L->s_pcol)[R];
  if (c >= C.n) return 0;
  uint8_t s = F.sgnV_()[c];
  int dv = ALP_G_VAR_DEG(C)[c];
  for (int k = 0; k < dv; ++k)
    if (var_ck(C, c, k) == R) return (s >> (4 + k)) & 1;
  return 0;
}

// Dependency level of every pivot for one sweep (level = 1 + max level of its deps).
// Pivots are processed in chunks of 32 in dependency order (fwd: ascending k, back:
// descending k); dependencies inside the chunk are resolved by shuffle fixed-point rounds.
// lv is indexed by pivot k.  Returns the number of levels.
template <bool FWD, int ND>
__device__ int compute_levels_t(const Frame& F, int p, uint16_t* lv) {
  const uint16_t* prow = F.S<uint16_t>(F.L->s_prow);
  const uint16_t* pos = F.S<uint16_t>(F.L->s_pos);
  int maxlv = 0;
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int k = FWD ? (c0 + F.lane) : (p - 1 - c0 - F.lane);
    const bool valid = FWD ? (k < p) : (k >= 0);
    int deps[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) deps[d] = DEP_NONE;
    if (valid) {
      const int R = prow[k];
      if constexpr (FWD) fwd_deps(F, R, deps);
      else back_deps<ND>(F, R, deps);
    }
    int ext = 0, anyin = 0;
    int inl[ND];   // in-chunk source lane of slot d, -1 if none
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      inl[d] = -1;
      if (deps[d] != DEP_NONE) {
        const int kd = pos[deps[d] & 0x7fff];
        const int off = FWD ? (kd - c0) : (p - 1 - c0 - kd);
        if (off >= 0 && off < 32) {
          inl[d] = off;
          anyin = 1;
        } else {
          ext = max(ext, (int)lv[kd] + 1);
        }
      }
    }
    int cur = ext;
    if (__any_sync(FULL, anyin)) {
      for (int it = 0; it <= 32; ++it) {
        int nw = ext;
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          const int vv = __shfl_sync(FULL, cur, inl[d] < 0 ? F.lane : inl[d]);
          if (inl[d] >= 0) nw = max(nw, vv + 1);
        }
        const bool ch = (nw != cur);
        cur = nw;
        if (!__any_sync(FULL, ch)) break;
      }
    }
    if (valid) {
      lv[k] = (uint16_t)cur;
      maxlv = max(maxlv, cur);
    }
    __syncwarp();
  }
  return wmaxi(maxlv) + 1;
}

template <bool FWD>
__device__ int compute_levels(const Frame& F, int p, uint16_t* lv) {
  if constexpr (FWD) return compute_levels_t<true, DVMAX>(F, p, lv);
  else return (F.C->dcr <= 8) ? compute_levels_t<false, 8>(F, p, lv) : compute_levels_t<false, 16>(F, p, lv);
}

// Deterministic counting sort of pivots by level: lv[k] (level) is replaced by the slot of
// pivot k in level order; off[0..nL] (global) receives the level boundaries.
__device__ void level_slots(const Frame& F, int p, int nL, uint16_t* lv, uint16_t* off) {
  int* hist = F.S<int>(F.L->s_hist);
  int* cur = F.S<int>(F.L->s_cur);
  for (int l = F.lane; l <= nL; l += 32) hist[l] = 0;
  __syncwarp();
  for (int k = F.lane; k < p; k += 32) atomicAdd(&hist[lv[k]], 1);
  __syncwarp();
  int carry = 0;
  for (int b0 = 0; b0 < nL; b0 += 32) {  // exclusive prefix sum
    int l = b0 + F.lane;
    int hv = (l < nL) ? hist[l] : 0;
    int incl = hv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL, incl, o);
      if (F.lane >= o) incl += t;
    }
    if (l < nL) {
      off[l] = (uint16_t)(carry + incl - hv);
      cur[l] = carry + incl - hv;
    }
    carry += __shfl_sync(FULL, incl, 31);
  }
  if (F.lane == 0) off[nL] = (uint16_t)carry;
  __syncwarp();
  const unsigned lt = (1u << F.lane) - 1u;
  for (int b0 = 0; b0 < p; b0 += 32) {
    int k = b0 + F.lane;
    bool valid = k < p;
    int lvl = valid ? (int)lv[k] : -1 - F.lane;
    unsigned peers = __match_any_sync(FULL, lvl);
    int slot = 0;
    if (valid) slot = cur[lvl] + __popc(peers & lt);
    __syncwarp();
    if (valid && (__ffs(peers) - 1) == F.lane) cur[lvl] += __popc(peers);
    if (valid) lv[k] = (uint16_t)slot;
    __syncwarp();
  }
}

// Builds both sweep programs.  Record layout (ints):
//  back  recB[slot*RB]: head = R | nd << 24 | diag_neg << 31, then nd deps (row | neg << 31)
//  fwd   recF[slot*RF]: same head/deps; dinvF[slot] = 1 / d^2 of the pivot column
// Preconditioner build: the column ranking, then Alg. 7 (mts = 0, the default) or
// Alg. 8 with diagonal expansion (mts = 2) or Alg. 6 (mts = 3) (SURVEY f-1), then the level
// schedules and the sweep programs shared by all three.
__device__ ALP_CALL_BUILD void build_precond(const Frame& F, int p, int& nLb, int& nLf, int mts = 0) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const Layout& L = *F.L;
  long long t0 = clock64();
  const int nv = sort_columns(F);
  long long t1 = clock64();
  if (mts == 2) peel_rowwise(F, p, nv);
  else if (mts == 3) peel_incremental(F, p, nv);
  else peel_columnwise(F, p);
  long long t2 = clock64();
#ifndef ALP_PEEL_COUNT
  if (F.lane == 0) {
    ALP_CYC(F)[CY_SORT] += t1 - t0;
    ALP_CYC(F)[CY_PEEL] += t2 - t1;
  }
#endif
  uint16_t* poc = F.S<uint16_t>(L.s_poc);
  const uint16_t* prow = F.S<uint16_t>(L.s_prow);
  const uint16_t* pcol = F.S<uint16_t>(L.s_pcol);
  for (int c = F.lane; c < C.Q; c += 32) poc[c] = NONE16;
  for (int j = F.lane; j < C.m; j += 32) F.pcolR[j] = NONE16;
  __syncwarp();
  for (int k = F.lane; k < p; k += 32) {
    int R = prow[k];
    poc[pcol[R]] = (uint16_t)R;
    F.pcolR[R] = pcol[R];   // kept past the PCG (the peel arrays are aliased by its vectors)
  }
  __syncwarp();
  uint16_t* lvB = F.S<uint16_t>(L.s_lvB);
  uint16_t* lvF = F.S<uint16_t>(L.s_lvF);
  nLb = compute_levels<false>(F, p, lvB);
  nLf = compute_levels<true>(F, p, lvF);
  level_slots(F, p, nLb, lvB, F.offB_());
  level_slots(F, p, nLf, lvF, F.offF_());
  // Records (u16, rows < 32768): word 0 = R | diag_neg << 15, then the dependencies
  // (row | coefficient_neg << 15), unused slots NODEP.  Back: RB words (8 or 16) per pivot,
  // forward: RF = 4 words per pivot (d_v <= 4) + dinvF = 1 / d^2 of the pivot column.
  for (int k = F.lane; k < p; k += 32) {
    const int R = prow[k];
    const int dn = diag_neg(F, R);
    uint16_t* rb = F.recB_() + (size_t)lvB[k] * C.RB;
    rb[0] = (uint16_t)(R | (dn << 15));
    if (C.RB == 8) {
      int deps[8];
      back_deps<8>(F, R, deps);
#pragma unroll
      for (int t = 0; t < 7; ++t)
        rb[1 + t] = (deps[t] == DEP_NONE) ? NODEP : (uint16_t)((deps[t] & 0x7fff) | ((deps[t] < 0) << 15));
    } else {
      int deps[16];
      back_deps<16>(F, R, deps);
#pragma unroll
      for (int t = 0; t < 15; ++t)
        rb[1 + t] = (deps[t] == DEP_NONE) ? NODEP : (uint16_t)((deps[t] & 0x7fff) | ((deps[t] < 0) << 15));
    }
    int fd[DVMAX];
    fwd_deps(F, R, fd);
    const int sf = lvF[k];
    uint16_t* rf = F.recF_() + (size_t)sf * RF;
    rf[0] = (uint16_t)(R | (dn << 15));
    int at = 1;   // compact the <= d_v - 1 forward deps into RF - 1 slots (record in memory)
#pragma unroll
    for (int q = 0; q < DVMAX; ++q)
      if (fd[q] != DEP_NONE && at < RF) rf[at++] = (uint16_t)((fd[q] & 0x7fff) | ((fd[q] < 0) << 15));
    for (int q = at; q < RF; ++q) rf[q] = NODEP;
    F.dinvF_()[sf] = 1.0 / F.d2[pcol[R]];
  }
  __syncwarp();
}

// Pivot sequence output (ipm_step_pcg debug/parity): rows[k], cols[k], -1 past p.
__device__ void write_pivots(const Frame& F, int p, int* rows, int* cols) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  const uint16_t* prow = F.S<uint16_t>(F.L->s_prow);
  const uint16_t* pcolR = F.pcolR;
  for (int k = F.lane; k < C.m; k += 32) {
    int R = (k < p) ? (int)prow[k] : -1;
    if (rows) rows[k] = R;
    if (cols) cols[k] = (k < p) ? (int)pcolR[R] : -1;
  }
}

// =====================================================================================
// PCG (Alg. 4) on (A D^2 A^T) dy = w with x^0 = 0 (C-9), matrix-free:
//   l = A (D^2 (A^T h)):  t_i = d2_i sum_j A_ji h_j (variable pass), l_j = sum_i A_ji t_i
//                         + d2_{n+j} h_j (check pass)                  [eq.`Delta y` LHS]
//   M^-1 r: back sweep A_M f = r, scale by D_M^-2, forward sweep A_M^T z = f
// Stops after line 9 once ||r||_2 <= tol ||w||_2 (G15).  h^T l <= 0 -> breakdown.
// w is read from F.w; the solution accumulates in F.dy_().
// =====================================================================================
// Sweeps run over the level schedule: level l holds the pivots in slots off[l] .. off[l+1];
// lanes take one pivot each (a loop covers levels wider than 32).
// Level offsets off[0..nL] held in registers: lane l keeps off[l] and off[32 + l]; levels
// beyond 63 fall back to memory.
struct OffReg {
  int a, b;
  const uint16_t* mem;
  __device__ __forceinline__ void load(const uint16_t* off, int nL, int lane) {
    mem = off;
    a = (lane <= nL) ? off[lane] : 0;
    b = (32 + lane <= nL) ? off[32 + lane] : 0;
  }
  __device__ __forceinline__ int operator()(int l) const {   // l warp-uniform
    if (l < 32) return __shfl_sync(FULL, a, l);
    if (l < 64) return __shfl_sync(FULL, b, l - 32);
    return mem[l];
  }
};

// Back substitution A_M f = r over the level schedule (P:585 stage 1), f_R = component of row R's
// pivot column, stored at index R.  A record is RBW uint4 (8 u16 each): [R | neg, dep...]; the
// records of a level are contiguous, and each level's first 32-slot chunk is prefetched during
// the previous level (records do not depend on the values being computed).
// The <= ND dependency gathers of a step are predicated loads issued back to back (no load
// inside the sum chain), and the signed terms are summed as a balanced tree: the step's latency
// is one gather round plus log2(ND + 1) fp64 adds (measured: with a load per dependency inside the sum chain, a level cost ~700
// cycles on the late-IPM systems of fractional frames, tools/straggler_trace.py).
template <int RBW, int ND>
__device__ __forceinline__ void back_step(const uint4 (&q)[RBW], const double* rS, double* fS) {
  const uint16_t* v = reinterpret_cast<const uint16_t*>(&q[0]);
  const int head = v[0];
  const int R = head & 0x7fff;
  if constexpr (ND > 7) {   // d_c > 8 (config 3): the serial chain (the tree's registers would
    double acc = rS[R];     // spill across the whole inlined kernel)
#pragma unroll
    for (int d = 1; d <= ND; ++d) {
      const int dep = v[d];
      if (dep != (int)NODEP) {
        const double fv = fS[dep & 0x7fff];
        acc = (dep & 0x8000) ? acc + fv : acc - fv;
      }
    }
    fS[R] = (head & 0x8000) ? -acc : acc;
  } else {
  double t[ND + 1];
  t[0] = rS[R];
#pragma unroll
  for (int d = 1; d <= ND; ++d) {
    const int dep = v[d];
    const double fv = (dep != (int)NODEP) ? fS[dep & 0x7fff] : 0.0;   // predicated gather
    t[d] = (dep & 0x8000) ? fv : -fv;
  }
#pragma unroll
  for (int w = 1; w <= ND; w *= 2)
#pragma unroll
    for (int d = 0; d + w <= ND; d += 2 * w) t[d] += t[d + w];
  fS[R] = (head & 0x8000) ? -t[0] : t[0];
  }
}

template <int RBW, int ND>
__device__ __forceinline__ void back_sweep_t(const Frame& F, int nLb, const double* rS, double* fS) {
  const uint4* rec = reinterpret_cast<const uint4*>(F.recB_());
  OffReg off;
  off.load(F.offB_(), nLb, F.lane);
  int a = off(0), b = off(1);
  if constexpr (RBW > 1) {
    // d_c > 7 (config 3): no prefetch (two live 32-byte records would raise the register
    // allocation of the whole inlined decode kernel; measured ~200 B of spills)
    for (int lvl = 0; lvl < nLb; ++lvl) {
      for (int s = a + F.lane; s < b; s += 32) {
        uint4 t[RBW];
#pragma unroll
        for (int k = 0; k < RBW; ++k) t[k] = rec[(size_t)s * RBW + k];
        back_step<RBW, ND>(t, rS, fS);
      }
      __syncwarp();
      a = b;
      b = (lvl + 2 <= nLb) ? off(lvl + 2) : b;
    }
    return;
  }
  uint4 cur[RBW];
  bool hc = a + F.lane < b;
  if (hc) {
#pragma unroll
    for (int k = 0; k < RBW; ++k) cur[k] = rec[(size_t)(a + F.lane) * RBW + k];
  }
  for (int lvl = 0; lvl < nLb; ++lvl) {
    const int c = (lvl + 2 <= nLb) ? off(lvl + 2) : b;
    uint4 nxt[RBW];
    const bool hn = (lvl + 1 < nLb) && (b + F.lane < c);
    if (hn) {
#pragma unroll
      for (int k = 0; k < RBW; ++k) nxt[k] = rec[(size_t)(b + F.lane) * RBW + k];
    }
    if (hc) back_step<RBW, ND>(cur, rS, fS);
    for (int s = a + F.lane + 32; s < b; s += 32) {
      uint4 t[RBW];
#pragma unroll
      for (int k = 0; k < RBW; ++k) t[k] = rec[(size_t)s * RBW + k];
      back_step<RBW, ND>(t, rS, fS);
    }
    __syncwarp();
    a = b;
    b = c;
#pragma unroll
    for (int k = 0; k < RBW; ++k) cur[k] = nxt[k];
    hc = hn;
  }
}

__device__ ALP_PCGPART void back_sweep(const Frame& F, int nLb, const double* rS, double* fS) {
  if (nLb <= 0) return;
  // dependency slots per record: position t in N(R) (t < d_c; the pivot's own column is NODEP)
  if (F.C->dcr <= 6) back_sweep_t<1, 6>(F, nLb, rS, fS);
  else if (F.C->RB == 8) back_sweep_t<1, 7>(F, nLb, rS, fS);
  else back_sweep_t<2, 15>(F, nLb, rS, fS);
}

// Forward substitution A_M^T z = D_M^-2 f (P:585 stages 2-3), z overwriting f in place (row R's
// f is read only by row R's own step, just before it writes z_R); returns this lane's part of
// z^T r = f^T D_M^-2 f (a sum of squares).  Record: uint2 = 4 u16 [R | neg, dep1..3].
__device__ __forceinline__ double fwd_step(uint2 rec, double dinv, double* zS) {
  const int head = rec.x & 0xffff;
  const int R = head & 0x7fff;
  const int d1 = rec.x >> 16, d2 = rec.y & 0xffff, d3 = rec.y >> 16;
  const bool u1 = d1 != (int)NODEP, u2 = d2 != (int)NODEP, u3 = d3 != (int)NODEP;
  // predicated gathers issued together, then a two-level add tree
  const double fr = zS[R];
  const double z1 = u1 ? zS[d1 & 0x7fff] : 0.0;   // predicated gathers
  const double z2 = u2 ? zS[d2 & 0x7fff] : 0.0;
  const double z3 = u3 ? zS[d3 & 0x7fff] : 0.0;
  const double t1 = (d1 & 0x8000) ? z1 : -z1;
  const double t2 = (d2 & 0x8000) ? z2 : -z2;
  const double t3 = (d3 & 0x8000) ? z3 : -z3;
  const double acc = (fr * dinv + t1) + (t2 + t3);
  zS[R] = (head & 0x8000) ? -acc : acc;
  return fr * fr * dinv;
}

__device__ ALP_PCGPART double fwd_sweep(const Frame& F, int nLf, double* fzS) {
  const uint2* __restrict__ recF = reinterpret_cast<const uint2*>(F.recF_());   // RF == 4 u16
  const double* __restrict__ dinvF = F.dinvF_();
  double rz = 0.0;
  if (nLf <= 0) return rz;
  OffReg off;
  off.load(F.offF_(), nLf, F.lane);
  int a = off(0), b = off(1);
  uint2 cur = make_uint2(0u, 0u);
  double dcur = 0.0;
  bool hc = a + F.lane < b;
  if (hc) {
    cur = recF[a + F.lane];
    dcur = dinvF[a + F.lane];
  }
  for (int lvl = 0; lvl < nLf; ++lvl) {
    const int c = (lvl + 2 <= nLf) ? off(lvl + 2) : b;
    uint2 nxt = make_uint2(0u, 0u);
    double dnxt = 0.0;
    const bool hn = (lvl + 1 < nLf) && (b + F.lane < c);
    if (hn) {
      nxt = recF[b + F.lane];
      dnxt = dinvF[b + F.lane];
    }
    if (hc) rz += fwd_step(cur, dcur, fzS);
    for (int s = a + F.lane + 32; s < b; s += 32) rz += fwd_step(recF[s], dinvF[s], fzS);
    __syncwarp();
    a = b;
    b = c;
    cur = nxt;
    dcur = dnxt;
    hc = hn;
  }
  return rz;
}

// Preconditioner modes of one PCG run.
constexpr int PC_MTS = 0, PC_NONE = 1;

// z = M^-1 r into fz; rz = z^T r.
__device__ __forceinline__ void precond_apply(const Frame& F, int mode, int nLb, int nLf, double& rz) {
  const DCode C = *F.C;
  const double* rS = F.r_();
  double* fzS = F.fz_();
  if (mode != PC_MTS) {   // identity (plain CG)
    double acc_rz = 0.0;
    for (int j = F.lane; j < C.m; j += 32) {
      double r = rS[j];
      fzS[j] = r;
      acc_rz += r * r;
    }
    __syncwarp();
    rz = wsum(acc_rz);
    return;
  }
  back_sweep(F, nLb, rS, fzS);
  rz = wsum(fwd_sweep(F, nLf, fzS));
}

struct PcgResult {
  int iters, status;
  double relres;       // TRUE ||w - Q dy|| / ||w|| at exit
  double rec_relres;   // recursive ||r|| / ||w|| at exit of the last recursion
  double relres_prev;  // refine mode: the true relres before the current restart
};

// SpMV l = Q h = A (D^2 (A^T h)) in two passes over the edges (eq.`Delta y` LHS), h in
// shared memory (absent rows hold 0), t over fz.
// Variable pass: t_i = d2_i (A^T h)_i; returns this lane's part of h^T Q h, accumulated as the
// sum of squares sum_i d2_i (A^T h)_i^2 + sum_j d2_{n+j} h_j^2 (never <= 0 by cancellation), so
// alpha (Alg. 4 line 7) is known before the check pass.  ABS: |A| D^2 |A|^T |h| (the rounding-
// floor estimate), returns 0.
template <bool ABS>
__device__ ALP_PCGPART double spmv_vars(const Frame& F, const DCode& C) {
  const double* __restrict__ hS = F.h_();
  double* __restrict__ tS = F.fz_();
  const uint8_t* __restrict__ sgnV = F.sgnV_();
  const uint16_t* __restrict__ sgnC = F.sgnC_();
  const uint16_t* __restrict__ var_chk = ALP_G_VAR_CHK(C);
  const double* __restrict__ d2 = F.d2;
  const int n = C.n;
  double hl = 0.0;
  // U variables per lane per step: all their index / sign / weight loads are issued before any
  // gather, and all gathers before any store (the shared-memory store of t would otherwise
  // block hoisting the next variable's loads)
#ifndef ALP_SPMV_UV
#define ALP_SPMV_UV 2
#endif
  constexpr int U = ALP_SPMV_UV;
  const double* __restrict__ d2s = d2 + n;
  const int m = C.m;
  // step k covers variables 32 U k + lane + 32 u and, for the slack columns, check 32 k + lane
  // (d2_{n+j} h_j^2), so both sums take one loop (m <= U n for every code in use; a remainder
  // loop covers the rest)
  // d^2 lives in the slot (L2): each step's weights are loaded one step ahead
  double dnx[U], dsnx = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) dnx[u] = (F.lane + 32 * u < n) ? d2[F.lane + 32 * u] : 0.0;
  if (!ABS && F.lane < m) dsnx = d2s[F.lane];
  int k = 0;
  for (int i0 = F.lane; i0 < n; i0 += 32 * U, ++k) {
    uint8_t sv[U];
    double dv[U];
    int jn[U][DVMAX];
    const int js = 32 * k + F.lane;
    double hs = 0.0, ds = 0.0;
    if (!ABS && js < m && (sgnC[js] & PRESENT)) {   // (absent rows: d2 is stale slot memory)
      hs = hS[js];
      ds = dsnx;
    }
    if (!ABS && js + 32 < m) dsnx = d2s[js + 32];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + 32 * u;
      const bool ok = i < n;
      sv[u] = ok ? sgnV[i] : (uint8_t)0;
      dv[u] = dnx[u];
      const int inx = i + 32 * U;
      dnx[u] = (inx < n) ? d2[inx] : 0.0;
      // scalar u16 index loads (measured: 16-byte vector loads of the padded rows were 1.8x slower)
#pragma unroll
      for (int kk = 0; kk < DVMAX; ++kk) jn[u][kk] = ((sv[u] >> kk) & 1) ? (int)var_chk[i * DVMAX + kk] : 0;
    }
    // predicated gathers, summed as a tree
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double g[DVMAX];
#pragma unroll
      for (int kk = 0; kk < DVMAX; ++kk) {
        const bool use = (sv[u] >> kk) & 1;
        const double hv = use ? hS[jn[u][kk]] : 0.0;   // predicated gather: absent rows load nothing
        g[kk] = ABS ? fabs(hv) : (((sv[u] >> (4 + kk)) & 1) ? -hv : hv);
      }
      acc[u] = (g[0] + g[1]) + (g[2] + g[3]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + 32 * u;
      if (i < n && (sv[u] & 0xf)) {
        const double tv = dv[u] * acc[u];
        tS[i] = tv;
        hl += acc[u] * tv;
      }
    }
    if (!ABS) hl += ds * hs * hs;
  }
  if (!ABS) {   // slack columns past the variable loop's coverage
    for (int j = 32 * k + F.lane; j < m; j += 32) {
      const double hj = hS[j];
      if (sgnC[j] & PRESENT) hl += d2s[j] * hj * hj;
    }
  }
  __syncwarp();
  return hl;
}

// Check pass: l_j = sum_t A_jt t_t + d2_{n+j} h_j, consumed at once (l is never stored):
//   CP_UPDATE: Alg. 4 lines 8-9, dy_j += alpha h_j, r_j -= alpha l_j; returns the lane's part
//              of ||r||^2;
//   CP_RESID:  r_j = w_j - l_j (h holds dy); returns the lane's part of ||r||^2;
//   CP_ABS:    returns the lane's part of || |A| D^2 |A|^T |h| ||^2.
// DCT >= the code's maximum check degree (compile-time, so the gathers unroll exactly).
constexpr int CP_UPDATE = 0, CP_RESID = 1, CP_ABS = 2;
template <int MODE, int DCT>
__device__ ALP_PCGPART double spmv_checks(const Frame& F, const DCode& C, double alpha) {
  const double* __restrict__ hS = F.h_();
  const double* __restrict__ tS = F.fz_();
  const uint16_t* __restrict__ sgnC = F.sgnC_();
  const uint16_t* __restrict__ chk_var = ALP_G_CHK_VAR(C);
  const uint8_t* __restrict__ chk_deg = ALP_G_CHK_DEG(C);
  const double* __restrict__ d2s_ = F.d2 + C.n;
  const double* __restrict__ W = F.w;
  double* __restrict__ rS = F.r_();
  double* __restrict__ dyS = F.dy_();
  const int m = C.m, dc = C.dc;
#ifndef ALP_SPMV_UC
#define ALP_SPMV_UC 2
#endif
  constexpr int UC = ALP_SPMV_UC;   // checks per lane per step
  double acc2 = 0.0;
  // the slack weights d2_{n+j} (slot, L2) are loaded one step ahead
  double dnx[UC];
#pragma unroll
  for (int u = 0; u < UC; ++u) dnx[u] = d2s_[min(F.lane + 32 * u, m - 1)];
  for (int j0 = F.lane; j0 < m; j0 += 32 * UC) {
    uint16_t sc[UC];
    double hj[UC], d2s[UC], rj[UC], yj[UC];
    int in[UC][DCT];
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int j = j0 + 32 * u;
      const bool ok = j < m;
      const int jj = ok ? j : 0;
      sc[u] = ok ? sgnC[j] : (uint16_t)0;
      const int deg = ok ? (int)chk_deg[j] : 0;
      hj[u] = hS[jj];
      d2s[u] = dnx[u];
      dnx[u] = d2s_[min(j + 32 * UC, m - 1)];
      if (MODE == CP_UPDATE) {
        rj[u] = rS[jj];
        yj[u] = dyS[jj];
      } else if (MODE == CP_RESID) {
        rj[u] = W[jj];
      }
#pragma unroll
      for (int t = 0; t < DCT; ++t) in[u][t] = (t < deg && (sc[u] & PRESENT)) ? (int)chk_var[j * dc + t] : -1;
    }
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      // predicated gathers (absent rows and slots past the degree load nothing), summed as a tree
      double g[DCT + 1];
      g[0] = d2s[u] * ((MODE == CP_ABS) ? fabs(hj[u]) : hj[u]);
#pragma unroll
      for (int t = 0; t < DCT; ++t) {
        const bool use = in[u][t] >= 0;
        const double tv = use ? tS[in[u][t]] : 0.0;
        g[t + 1] = (MODE == CP_ABS) ? tv : (((sc[u] >> t) & 1) ? -tv : tv);
      }
#pragma unroll
      for (int w = 1; w <= DCT; w *= 2)
#pragma unroll
        for (int d = 0; d + w <= DCT; d += 2 * w) g[d] += g[d + w];
      const double l = g[0];
      const int j = j0 + 32 * u;
      if (!(sc[u] & PRESENT)) continue;   // also j >= m (sc = 0)
      if (MODE == CP_UPDATE) {
        dyS[j] = yj[u] + alpha * hj[u];   // line 8
        const double r = rj[u] - alpha * l;   // line 9
        rS[j] = r;
        acc2 += r * r;
      } else if (MODE == CP_RESID) {
        const double r = rj[u] - l;
        rS[j] = r;
        acc2 += r * r;
      } else {
        acc2 += l * l;
      }
    }
  }
  __syncwarp();
  return acc2;
}

template <int MODE>
__device__ __forceinline__ double spmv_checks_any(const Frame& F, const DCode& C, double alpha) {
  const int dcs = C.dcr;
  if (dcs <= 6) return spmv_checks<MODE, 6>(F, C, alpha);
  if (dcs <= 12) return spmv_checks<MODE, 12>(F, C, alpha);
  return spmv_checks<MODE, DCMAX>(F, C, alpha);
}

// h = dy on the present rows (0 elsewhere), then r = w - Q dy (returns ||r||^2) or, with ABS,
// || |A| D^2 |A|^T |dy| ||^2.
template <bool ABS>
__device__ ALP_HEAVY double true_residual(const Frame& F) {
  const DCode C = *F.C;
  double* hS = F.h_();
  const double* dy = F.dy_();
  const uint16_t* sgnC = F.sgnC_();
  for (int j = F.lane; j < C.m; j += 32) hS[j] = (sgnC[j] & PRESENT) ? dy[j] : 0.0;
  __syncwarp();
  spmv_vars<ABS>(F, C);
  return wsum(ABS ? spmv_checks_any<CP_ABS>(F, C, 0.0) : spmv_checks_any<CP_RESID>(F, C, 0.0));
}

constexpr int PCG_REFINE_MAX = 6;

// double-double helpers (Knuth two-sum, fma two-product)
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, double b) {
  const double s = a.hi + b;
  const double bb = s - a.hi;
  const double e = (a.hi - (s - bb)) + (b - bb) + a.lo;
  const double h = s + e;
  return DD{h, e - (h - s)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD t = dd_add(a, b.hi);
  return dd_add(t, b.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, double b) {
  const double p = a.hi * b;
  const double e = fma(a.hi, b, -p) + a.lo * b;
  const double h = p + e;
  return DD{h, e - (h - p)};
}

// r = w - Q dy in double-double (Q = A D^2 A^T applied matrix-free, one pass over the checks,
// (A^T dy)_i recomputed per edge); rounded r to rS, returns ||r||^2.  The residual itself is then
// accurate far below the fp64 evaluation floor, which is what lets refinement converge.
__device__ __noinline__ double residual_dd(const Frame& F, double* rS) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  double acc = 0.0;
  for (int j = F.lane; j < C.m; j += 32) {
    const uint16_t sc = F.sgnC_()[j];
    double r = 0.0;
    if (sc & PRESENT) {
      DD l = dd_mul(DD{F.dy_()[j], 0.0}, F.d2[C.n + j]);
      const int deg = ALP_G_CHK_DEG(C)[j];
      for (int t = 0; t < deg; ++t) {
        const int i = chk_nb(C, j, t);
        const uint8_t sv = F.sgnV_()[i];
        DD ti{0.0, 0.0};
        for (int k = 0; k < ALP_G_VAR_DEG(C)[i]; ++k) {
          if (!((sv >> k) & 1)) continue;
          const double h = F.dy_()[var_ck(C, i, k)];
          ti = dd_add(ti, ((sv >> (4 + k)) & 1) ? -h : h);
        }
        DD ui = dd_mul(ti, F.d2[i]);
        if ((sc >> t) & 1) ui = DD{-ui.hi, -ui.lo};
        l = dd_add(l, ui);
      }
      const DD rr = dd_add(DD{-l.hi, -l.lo}, F.w[j]);
      r = rr.hi + rr.lo;
    }
    rS[j] = r;
    acc += r * r;
  }
  __syncwarp();
  return wsum(acc);
}

// PCG (Alg. 4) from dy = 0, r = w, in preconditioner mode `mode`.  The recursion
// stops after line 9 once ||r||_2 <= itol ||w||_2 (G15, C-9; itol <= pcg_rel_tol is the
// inexact-Newton target of the caller); once ||r|| <= pcg_rel_tol ||w|| (the acceptance test of
// C-9) the recursion gets at most 50 more iterations towards itol.  It also ends at the cap, on a
// breakdown (h^T Q h or z^T r not > 0 / non-finite; both are sums of squares, so only 0 / inf /
// nan), or on divergence (||r|| 1e8-fold above its minimum).  There is no early stall exit:
// late-IPM systems of fractional LPs often make no progress for a few hundred
// iterations and then converge, and cutting them short stalls the IPM (measured, R-1).  The TRUE residual w - Q dy is then evaluated once.
// `refine` (ipm_step_pcg only): while the true residual fails pcg_rel_tol, restart from it
// (iterative refinement with the same preconditioner, at most 4 restarts); a restart that no
// longer halves it within 1e3x of the fp64 evaluation floor 16 eps || |A| D^2 |A|^T |dy| ||
// stops with ST_PCG_FLOOR (attainable accuracy, informational).
// Status: 0 = the last recursion met pcg_rel_tol (P4), ST_PCG_MAXITER (cap or stall),
// ST_PCG_BREAKDOWN, ST_PCG_FLOOR (refine mode).  w is read from F.w; dy accumulates in F.dy_().
__device__ ALP_CALL_PCG PcgResult pcg_solve(const Frame& F, const Params& P, int mode, int nLb, int nLf,
                                         double itol_rel, int refine) {
  const DCode C = *F.C;   // register copy: graph pointers / dims not re-read from shared memory
  double* hS = F.h_();
  double* rS = F.r_();
  double* fzS = F.fz_();
  double* dyS = F.dy_();
  const uint16_t* __restrict__ sgnC = F.sgnC_();
  double ww = 0.0;
#pragma unroll 4
  for (int j = F.lane; j < C.m; j += 32) {   // (unrolled: the w loads from the slot overlap)
    const bool pr = (sgnC[j] & PRESENT) != 0;
    const double wj = pr ? F.w[j] : 0.0;
    ww += wj * wj;
    rS[j] = wj;        // lines 1-2: x^0 = 0, r^0 = w
    dyS[j] = 0.0;
    fzS[j] = 0.0;      // absent rows stay exactly 0 in z, f and h (C-19)
    hS[j] = 0.0;
  }
  __syncwarp();
  const double wn = sqrt(wsum(ww));
  PcgResult res{0, 0, 0.0, 0.0, 0.0};
  if (wn == 0.0) return res;
  const double tol = P.pcg_rel_tol * wn;                       // acceptance (C-9)
  double itol = fmin(itol_rel, P.pcg_rel_tol) * wn;            // recursion target
  const int cap = P.pcg_max_iter;
  int it = 0;
  double prev_trn = 1e308;
  for (int restart = 0; restart <= (refine ? PCG_REFINE_MAX : 0); ++restart) {
    double rz;
    precond_apply(F, mode, nLb, nLf, rz);   // line 3
    if (!(rz > 0.0) || !isfinite(rz)) {
      res.status = ST_PCG_BREAKDOWN;
      break;
    }
    for (int j = F.lane; j < C.m; j += 32) hS[j] = (sgnC[j] & PRESENT) ? fzS[j] : 0.0;   // line 4
    __syncwarp();
    int st = ST_PCG_MAXITER, past = -1, since_min = 0;
    double rrmin = 1e308, rr = 0.0;
    long long tk = clock64();
    const int cap_run = (restart > 0) ? min(cap, it + 200) : cap;   // a refinement restart gets <= 200
    while (it < cap_run) {
      ALP_TICK(F, CY_PCG, tk);
      // line 6 (l = Q h) fused with lines 7-9: h^T Q h from the variable pass gives alpha, the
      // check pass then forms l_j and updates dy_j, r_j at once
      const double hl = wsum(spmv_vars<false>(F, C));
      if (!(hl > 0.0) || !isfinite(hl)) {
        ALP_TICK(F, CY_SPMV, tk);
        st = ST_PCG_BREAKDOWN;
        break;
      }
      const double alpha = rz / hl;   // line 7
      rr = wsum(spmv_checks_any<CP_UPDATE>(F, C, alpha));
      ALP_TICK(F, CY_SPMV, tk);
      ++it;
      const double rn = sqrt(rr);
      if (rn <= itol) {
        st = 0;
        break;
      }
      if (rn <= tol) {   // accepted; at most 50 more iterations towards the forcing target
        if (past < 0) past = it;
        else if (it - past >= 50) {
          st = 0;
          break;
        }
      }
      if (rr < rrmin) {
        rrmin = rr;
        since_min = 0;
      } else if (rr > 1e16 * rrmin || ++since_min > 1000) {
        st = (rrmin <= tol * tol) ? 0 : ST_PCG_MAXITER;   // stall
        break;
      }
      double rz_new;
      ALP_TICK(F, CY_PCG, tk);
      precond_apply(F, mode, nLb, nLf, rz_new);   // line 10
      ALP_TICK(F, CY_SWEEP, tk);
      if (!(rz_new > 0.0) || !isfinite(rz_new)) {
        st = ST_PCG_BREAKDOWN;
        break;
      }
      const double nu = rz_new / rz;   // line 11
      rz = rz_new;
#pragma unroll 4
      for (int j = F.lane; j < C.m; j += 32) {
        if (!(sgnC[j] & PRESENT)) continue;
        hS[j] = fzS[j] + nu * hS[j];   // line 12
      }
      __syncwarp();
    }
    ALP_TICK(F, CY_PCG, tk);
    res.rec_relres = sqrt(rr) / wn;
    if (st == 0 && !(res.rec_relres <= P.pcg_rel_tol)) st = ST_PCG_MAXITER;
    // TRUE residual r = w - Q dy: fp64 in the decode (reported), double-double in refine mode
    // (ipm_step_pcg), where it drives the refinement restarts
    const double trn = (refine == 2) ? sqrt(residual_dd(F, rS)) : sqrt(true_residual<false>(F));
    res.relres = trn / wn;
    res.status = st;
    ALP_TICK(F, CY_PCG, tk);
    if (!refine || st == ST_PCG_BREAKDOWN || !isfinite(trn)) break;
    if (refine == 1) {
      // fp64 iterative refinement: restart from the true residual (each restart aiming 1e-6
      // below it) until it is 1e-4 below the acceptance pcg_rel_tol (so that the forward error
      // meets SURVEY C-27's 1e-8 on systems with kappa(Q) up to ~1e12, not only the residual),
      // or reaches the fp64 evaluation floor 16 eps || |A| D^2 |A|^T |dy| ||, or a restart no
      // longer halves it within 1e3x of that floor.  PCG_FLOOR: the TRUE residual stayed above
      // pcg_rel_tol (informational).
      const bool met = trn <= tol;
      // a refinement restart (capped at 200 iterations) is judged by the true residual alone
      if (restart > 0 && st == ST_PCG_MAXITER) st = 0;
      res.status = st;
      if (trn <= 1e-4 * tol) break;
      const double aa = true_residual<true>(F);   // (leaves r = w - Q dy in place)
      const double floor_est = 16.0 * 2.220446049250313e-16 * sqrt(aa);
      if (trn <= floor_est || (trn > 0.5 * prev_trn && trn <= 1e3 * floor_est) || restart == 4 || st != 0) {
        if (!met) res.status = (st == 0) ? ST_PCG_FLOOR : st;
        break;
      }
      prev_trn = trn;
      itol = 1e-6 * trn;
      continue;
    }
    // Iterative refinement with double-double residuals: restart PCG on Q delta = r (the same
    // preconditioner), dy += delta, while the correction keeps shrinking: stop once
    // ||delta|| <= 1e-13 ||dy||, or ||delta|| no longer halves, or after PCG_REFINE_MAX restarts.
    // (The residual of a rounded fp64 dy cannot fall below ~eps || |A| D^2 |A|^T |dy| ||, so its
    // norm is no stopping signal near the floor; the correction size is.)  Each restart aims
    // 1e-6 below its starting residual.  PCG_FLOOR: the TRUE residual stayed above pcg_rel_tol.
    double dn = 0.0, yn = 0.0;
    if (restart > 0) {
      for (int j = F.lane; j < C.m; j += 32) {
        const double d = dyS[j] - F.v[j];
        dn += d * d;
        yn += dyS[j] * dyS[j];
      }
      dn = sqrt(wsum(dn));
      yn = sqrt(wsum(yn));
    }
    if (restart > 0 && st != 0) {
      // a refinement restart that did not converge: keep dy from before it (the last good one)
      for (int j = F.lane; j < C.m; j += 32) dyS[j] = F.v[j];
      __syncwarp();
      res.status = (res.relres_prev > P.pcg_rel_tol) ? ST_PCG_FLOOR : 0;
      res.relres = res.relres_prev;
      break;
    }
    if (st != 0 || restart == PCG_REFINE_MAX || (restart > 0 && (dn <= 1e-13 * yn || dn > 0.5 * prev_trn))) {
      if (st == 0 && trn > tol) res.status = ST_PCG_FLOOR;
      break;
    }
    res.relres_prev = res.relres;
    if (restart > 0) prev_trn = dn;
    for (int j = F.lane; j < C.m; j += 32) F.v[j] = dyS[j];   // dy before the next correction
    __syncwarp();
    itol = 1e-6 * trn;
  }
  res.iters = it;
  return res;
}

}  // namespace ALP_NS
}  // namespace alp
