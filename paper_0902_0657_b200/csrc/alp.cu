// alp.cu — kernels and C ABI of libalp.so (see include/alp.h).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
// One persistent kernel per call: each warp repeatedly claims a frame (atomic counter),
// runs the whole adaptive-LP decode of that frame (Alg. 3 with the IPM of §IV-B and the
// PCG of Alg. 4 preconditioned by Alg. 7) and writes its outputs; no host round trips.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "alp.h"
#include "alp_device.cuh"   // mode-independent types (first inclusion also defines them)

namespace alp {

// Optional per-Newton-step trace (alp_debug_trace): one record per step solve.
struct TraceRec {
  int frame, lp, ipm_it, p, status, iters, nLb, nLf;
  double relres, rec_relres, d2min, d2max, mu, rb, rc, gap, beta_p, beta_d;
};
__device__ TraceRec* g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ int g_trace_n = 0;

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

}  // namespace alp

// The device code three times: shared-memory window (sm), generic window with the graph in
// global memory (gm; large codes), generic window with the graph staged in shared memory and
// read by LDS (gs; config 5).
#define ALP_NS sm
#define ALP_SM 1
#include "alp_device.cuh"
#include "alp_kernels.cuh"
#undef ALP_NS
#undef ALP_SM
#define ALP_NS gm
#define ALP_SM 0
#include "alp_device.cuh"
#include "alp_kernels.cuh"
#undef ALP_NS
#undef ALP_SM
#define ALP_NS gs
#define ALP_SM 0
#define ALP_GRAPH_SH 1
#include "alp_device.cuh"
#include "alp_kernels.cuh"
#undef ALP_NS
#undef ALP_SM
#undef ALP_GRAPH_SH

// =====================================================================================
// Host side
// =====================================================================================
using namespace alp;

struct alp_code {
  int n, m, dc, dv, dcr, dvr, E;   // dc, dv: padded strides of chk_var / var_chk; dcr, dvr: degrees
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
  C.dcr = c->dcr;
  C.dvr = c->dvr;
  C.Q = c->n + c->m;
  C.W = (C.Q + 63) / 64;
  C.RB = (c->dcr + 1 <= 8) ? 8 : 16;   // back-record u16 words: head + <= d_c - 1 deps
  C.chk_var = c->d_chk_var;
  C.chk_deg = c->d_chk_deg;
  C.var_chk = c->d_var_chk;
  C.var_slot = c->d_var_slot;
  C.var_deg = c->d_var_deg;
  C.so_chk_var = C.so_chk_deg = C.so_var_chk = C.so_var_deg = 0;   // set by stage_graph
  return C;
}

// Per-frame global slot (both window modes); returns the byte count used so far.
size_t make_slot(const DCode& C, Layout& L) {
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
  L.g_w = g(8 * m);
  L.g_u = g(8 * n);
  L.g_b = g(8 * m);
  L.g_dinvF = g(8 * m);
  L.g_recB = g(2 * m * C.RB);
  L.g_recF = g(2 * m * RF);
  L.g_offB = g(2 * (m + 2));
  L.g_offF = g(2 * (m + 2));
  L.g_sgnC = g(2 * m);
  L.g_mask = g(2 * m);
  L.g_hist = g(8 * 256);
  L.g_sgnV = g(n);
  L.g_flip = g(n);
  L.g_rb = g(8 * m);
  L.g_rc = g(8 * Q);
  L.g_pcol = g(2 * m);
  L.g_r = g(8 * m);
  L.slot_bytes = (long long)al(o, 256);
  return o;
}

// Window layout of the shared-memory mode (kernel alp::sm::*): one fixed per-frame window,
//   S: sgnC [m], sgnV [n] (live throughout);
//   P: PCG vectors h, r, dy [m] and fz [max(m, n)] (f, z in place; t of the SpMV over it);
//   D: the sweep programs: back / forward records, dinvF, level offsets.
// The preconditioner build overlays P and D (both dead while it runs): the column sort's radix
// buffers from the start of P with `order` after them; the peel's pos / pcol / prow at the start
// of P and its rank / count / XOR / bitmap / row-rank arrays after them; the post-peel arrays
// (levels, pivot-of-column map, level histograms) after pos / pcol / prow, inside P (the
// records in D are written from them).  d^2, w and the IPM arrays stay in the slot (L1/L2).
// Returns false when the post-peel arrays do not fit P (then the generic mode is used).
bool make_layout_sm(const DCode& C, Layout& L, bool sm_d2) {
  const size_t n = C.n, m = C.m, Q = C.Q;
  make_slot(C, L);
  L.win_global = 0;
  L.g_win = 0;
  size_t a = 0;
  auto s = [&](size_t bytes) {
    size_t r = a;
    a += al(bytes, 16);
    return (int)r;
  };
  L.smask = 0;
  auto rel = [&](int k, size_t bytes) {
    L.smask |= 1u << k;
    L.soff[k] = s(bytes);
  };
  rel(RL_SGNC, 2 * m);
  rel(RL_SGNV, n);
  const size_t S0 = a;
  // P
  L.s_h = s(8 * m);
#ifdef ALP_SM_R_SLOT
  L.s_r = -1;   // r lives in the slot (tuning variant)
#else
  L.s_r = s(8 * m);
#endif
  rel(RL_DY, 8 * m);
  L.s_fz = s(8 * std::max(m, n));
  const size_t endP = a;
  // D
  rel(RL_RECB, 2 * m * (size_t)C.RB);
  rel(RL_RECF, 2 * m * (size_t)RF);
  rel(RL_DINVF, 8 * m);
  rel(RL_OFFB, 2 * (m + 2));
  rel(RL_OFFF, 2 * (m + 2));
  if (sm_d2) rel(RL_D2, 8 * Q);   // d^2 too (fewer frames per SM; tuning)
  const size_t endD = a;
  // build, post-peel: pos / pcol / prow, then the level arrays, inside P
  a = S0;
  L.s_pos = s(2 * m);
  L.s_pcol = s(2 * m);
  L.s_prow = s(2 * m);
  const size_t L0 = a;
  L.s_lvB = s(2 * m);
  L.s_lvF = s(2 * m);
  L.s_poc = s(2 * Q);
  L.s_hist = s(4 * (m + 2));
  L.s_cur = s(4 * (m + 2));
  if (a > endP) return false;
  // build, peel: after pos / pcol / prow
  a = L0;
  L.s_rank = s(2 * Q);
  L.s_cnt = s(Q);
  L.s_xr = s(2 * Q);
  L.s_bm = s(8 * (size_t)C.W);
  L.RS = (C.dcr + 1 <= 8) ? 8 : 16;
  L.s_rrank = s(2 * m * (size_t)L.RS);
  const size_t endPeel = a;
  // build, sort: radix buffers kA/kB u32[Q], cA/cB u16[Q] and the digit table from S0; the
  // ranked column order after both the sort buffers and the peel arrays
  L.s_sortk = (int)S0;
  L.s_sorth = (int)(S0 + al(12 * Q, 16));
  a = std::max(S0 + al(12 * Q, 16) + 2048, endPeel);
  L.s_order = s(2 * Q);
  L.smem_bytes = (int)al(std::max(endD, a), 128);
  return true;
}

Layout make_layout(const DCode& C, int smem_budget) {
  Layout L;
  const size_t n = C.n, m = C.m, Q = C.Q;
  size_t o = make_slot(C, L);
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
  L.RS = (C.dcr + 1 <= 8) ? 8 : 16;
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
  // PCG phase: h, r [m], fz [max(m, n)] (f and z in place; t over it)
  a = 0;
  L.s_h = s(8 * m);
  L.s_r = s(8 * m);
  L.s_fz = s(8 * std::max(m, n));
  size_t end_pcg = a;
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
  // priority (sign tables, dy, sweep programs, D^2, w), while the window fits the budget.
  L.smask = 0;
  size_t rel_bytes[RL_N];
  rel_bytes[RL_SGNC] = 2 * m;
  rel_bytes[RL_SGNV] = n;
  rel_bytes[RL_DY] = 8 * m;
  rel_bytes[RL_DINVF] = 8 * m;
  rel_bytes[RL_OFFB] = 2 * (m + 2);
  rel_bytes[RL_OFFF] = 2 * (m + 2);
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
  G.o_var_slot = 0;   // not staged (build_signs reads it from global memory once per LP)
  G.o_var_deg = a(C.n);
  G.bytes = (int)al(o, 128);
  // large codes: graph stays global (ALP_GRAPH_MAX_KB overrides the 72 KB limit for tuning runs;
  // make_plan drops a staged graph above 48 KB when it would cost a resident frame)
  int max_kb = 72;
  if (const char* ev = getenv("ALP_GRAPH_MAX_KB")) max_kb = atoi(ev);
  if (G.bytes > max_kb * 1024) G = GraphSmem{0, 0, 0, 0, 0, 0};
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
  P.pcg_refine = p->pcg_refine;
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
  if (p->precond < 0 || p->precond > 3)
    return fail(ALP_ERR_INVALID_ARG, "params.precond must be 0 (Alg. 7), 1 (plain CG), 2 (Alg. 8) or 3 (Alg. 6)");
  if (!(p->sigma > 0 && p->sigma < 1) || !(p->eta > 0 && p->eta < 1))
    return fail(ALP_ERR_INVALID_ARG, "params.sigma and params.eta must lie in (0,1)");
  if (p->alp_max_iter < 0 || p->alp_max_iter > 255 || p->ipm_max_iter < 0 || p->pcg_max_iter < 1)
    return fail(ALP_ERR_INVALID_ARG, "iteration caps: 0 <= alp_max_iter <= 255, ipm >= 0, pcg >= 1");
  if (p->pcg_refine < 0 || p->pcg_refine > 2)
    return fail(ALP_ERR_INVALID_ARG, "params.pcg_refine must be 0, 1 or 2");
  if (p->warps_per_block < 0 || p->warps_per_block > 8 || p->smem_frames_per_sm < 0 || p->smem_frames_per_sm > 32)
    return fail(ALP_ERR_INVALID_ARG, "params.warps_per_block must be 0..8, smem_frames_per_sm 0..32");
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

// relocation mask of the shared-memory mode's fixed layout (make_layout_sm)
constexpr unsigned SM_FIXED_MASK = (1u << RL_SGNC) | (1u << RL_SGNV) | (1u << RL_DY) | (1u << RL_DINVF) |
                                   (1u << RL_OFFB) | (1u << RL_OFFF) | (1u << RL_RECF) | (1u << RL_RECB);

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
  // frames (warps) per CTA: the caller's choice, else 4 for the generic mode and, for the
  // shared-memory mode (one CTA per SM), as many windows as fit (<= 8)
  int wpb = (p && p->warps_per_block > 0) ? p->warps_per_block : (L.win_global || L.smask != SM_FIXED_MASK ? 4 : 8);
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

// Launch plan: the shared-memory window mode (alp::sm kernels, fixed layout, LDS everywhere)
// when its per-frame window fits at least 2 frames per CTA and the caller did not ask for a
// specific shared-memory split; otherwise the generic mode (alp::gm kernels, budget relocation,
// global window for large codes).
struct Plan {
  bool sm;
  bool gs = false;
  Layout L;
  GraphSmem G;
  LaunchCfg cfg;
};

alp_status make_plan(const alp_code* code, int64_t units, const alp_params* p, bool step, Plan& pl) {
  const DCode C = make_dcode(code);
  pl.G = make_graph_smem(C);
  units = std::max<int64_t>(units, 1);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || optin <= 0)
    optin = 227 * 1024;
  const bool want_gm = p && p->smem_frames_per_sm > 0;
  const char* ev = getenv("ALP_SM_D2");
  const bool sm_d2 = ev && ev[0] == '1';
  if (!want_gm && make_layout_sm(C, pl.L, sm_d2)) {
    // worth it when at least 4 windows fit a CTA (C1, C2; measured: config 5's 92 KB windows run
    // faster in the generic mode, 151 k vs 103 k systems/s)
    // (sm mode reads the graph from its staged shared copy: G.bytes > 0 is required)
    if (pl.G.bytes > 0 && 4LL * pl.L.smem_bytes + pl.G.bytes <= optin - 1024) {
      pl.sm = true;
      return step ? plan_launch(sm::pcg_step_kernel, pl.L, pl.G.bytes, units, p, pl.cfg)
                  : plan_launch(sm::alp_decode_kernel, pl.L, pl.G.bytes, units, p, pl.cfg);
    }
  }
  pl.sm = false;
  pl.L = make_layout(C, smem_budget_for(p));
  // gs kernels: graph staged in shared memory and read by LDS (the window keeps generic pointers:
  // an LDS-addressed window measured 8 % slower on config 5, profiles/r2_ab_g31.log).  A graph
  // above 48 KB is staged only if it costs no resident frame (config 3: 2 x 78 KB windows + 69 KB).
  if (pl.G.bytes > 48 * 1024) {
    const int want = (p && p->warps_per_block > 0) ? p->warps_per_block : 4;
    int w0 = want;
    while (w0 > 1 && (long long)w0 * pl.L.smem_bytes > optin - 1024) --w0;
    if (pl.L.win_global || (long long)w0 * pl.L.smem_bytes + pl.G.bytes > optin - 1024) pl.G = GraphSmem{0, 0, 0, 0, 0, 0};
  }
  pl.gs = pl.G.bytes > 0;
  if (pl.gs)
    return step ? plan_launch(gs::pcg_step_kernel, pl.L, pl.G.bytes, units, p, pl.cfg)
                : plan_launch(gs::alp_decode_kernel, pl.L, pl.G.bytes, units, p, pl.cfg);
  return step ? plan_launch(gm::pcg_step_kernel, pl.L, pl.G.bytes, units, p, pl.cfg)
              : plan_launch(gm::alp_decode_kernel, pl.L, pl.G.bytes, units, p, pl.cfg);
}

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
  p->pcg_refine = 1;
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

alp_status alp_launch_info(const alp_code* code, int64_t units, const alp_params* params, int32_t step,
                           int32_t* info) {
  if (!code || !info || units < 0) return fail(ALP_ERR_INVALID_ARG, "code / info NULL or units < 0");
  alp_status ps = check_params(params);
  if (ps != ALP_OK) return ps;
  Plan pl;
  alp_status st = make_plan(code, units, params, step != 0, pl);
  if (st != ALP_OK) return st;
  info[0] = pl.sm ? 1 : 0;
  info[1] = pl.cfg.wpb;
  info[2] = pl.cfg.grid;
  info[3] = pl.L.smem_bytes;
  info[4] = pl.cfg.smem_block;
  info[5] = (int32_t)pl.L.slot_bytes;
  return ALP_OK;
}

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
  // padded strides (vector loads of a whole row / column list): checks 8 or 16 u16 per row,
  // variables DVMAX = 4 u16; the real maximum degrees are kept beside them
  const int dcr = dc, dvr = dv;
  dc = (dcr <= 8) ? 8 : 16;
  dv = DVMAX;
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
  c->dcr = dcr;
  c->dvr = dvr;
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
  Plan pl;
  if (make_plan(code, n_frames, params, false, pl) != ALP_OK) return 0;
  return kCounterBytes + (size_t)pl.cfg.slots * (size_t)pl.L.slot_bytes;
}

size_t alp_pcg_workspace_bytes(const alp_code* code, int64_t n_sys, const alp_params* params) {
  g_last_status = ALP_OK;
  if (!code || n_sys < 0 || check_params(params) != ALP_OK) {
    if (!code || n_sys < 0) fail(ALP_ERR_INVALID_ARG, "bad code or n_sys");
    return 0;
  }
  Plan pl;
  if (make_plan(code, n_sys, params, true, pl) != ALP_OK) return 0;
  return kCounterBytes + (size_t)pl.cfg.slots * (size_t)pl.L.slot_bytes;
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
  const DCode C = make_dcode(code);
  Plan pl;
  alp_status st = make_plan(code, n_frames, params, false, pl);
  if (st != ALP_OK) return st;
  size_t need = kCounterBytes + (size_t)pl.cfg.slots * (size_t)pl.L.slot_bytes;
  if (workspace_bytes < need)
    return fail(ALP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* counter = (unsigned long long*)workspace;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  DecodeOut O{hard, objective, certificate, frame_status, stats, u_out, y_out, mask_out};
  char* slots = (char*)workspace + kCounterBytes;
  if (pl.sm)
    sm::alp_decode_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, llr, (long long)n_frames, O, counter);
  else if (pl.gs)
    gs::alp_decode_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, llr, (long long)n_frames, O, counter);
  else
    gm::alp_decode_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, llr, (long long)n_frames, O, counter);
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
  const DCode C = make_dcode(code);
  Plan pl;
  alp_status st = make_plan(code, n_sys, params, true, pl);
  if (st != ALP_OK) return st;
  size_t need = kCounterBytes + (size_t)pl.cfg.slots * (size_t)pl.L.slot_bytes;
  if (workspace_bytes < need)
    return fail(ALP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* counter = (unsigned long long*)workspace;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(*counter), s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
  StepIO io{masks, flip, d, r, dy, pcg_iters, rel_res, sys_status, pivot_rows, pivot_cols};
  char* slots = (char*)workspace + kCounterBytes;
  if (pl.sm)
    sm::pcg_step_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, (long long)n_sys, io, counter);
  else if (pl.gs)
    gs::pcg_step_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, (long long)n_sys, io, counter);
  else
    gm::pcg_step_kernel<<<pl.cfg.grid, 32 * pl.cfg.wpb, pl.cfg.smem_block, s>>>(
        C, make_params(params), pl.L, pl.G, slots, (long long)n_sys, io, counter);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pcg_step_kernel launch");
  g_last_launches = 1;
  return ALP_OK;
}

}  // extern "C"
