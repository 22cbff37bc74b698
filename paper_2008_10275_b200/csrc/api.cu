// liblrcheb C ABI (include/lrcheb.h): context, validation, workspaces, and the ChebyshevT driver.
//
// One iteration k (X_k -> X_{k+1}, reading S1) is enqueued as
//   fork:  [s0] K1 spmm S2STEP(U_k) -> W3 = [U_k - g W0], [W1], [W2] (three contiguous arrays) (a1)
//          [s1] vside: Vcat, Householder QR -> T1 = R_V^T, Q_V                    (a2)
//   join:  ts GRAM(Ucat, T1 = R_V^T) -> Y (stored, M x p), G1 -> reduce -> chol1 -> R1^{-1}   (a3)
//          ts GRAM(Y, R1^{-1}) -> G2 -> reduce -> chol2 + Jacobi + rank -> W_r, V_{k+1}       (a4, a5)
//          ts STORE(Y, W_r Sigma_r^{-1}) -> U_{k+1}                                          (a6)
// with Ucat = [B_U | W0' | W1 | W2 | U_{k-1}] never copied (five strided blocks), ranks device-resident,
// so the whole N-iteration loop is captured once into a CUDA graph and replayed.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <iterator>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lrcheb.h"
#include "lrc_internal.cuh"

namespace lrc {
size_t vside_smem_bytes(int n, int wmax, int pmax);
cudaError_t spmm_prepare();
cudaError_t ts_prepare();
cudaError_t small_prepare();
}  // namespace lrc

using namespace lrc;

static thread_local std::string g_create_err;   // lrc_last_error(NULL): lrc_create failures
static std::atomic<int64_t> g_gen{0};           // workspace / operator generations, unique across contexts
static int64_t next_gen() { return ++g_gen; }

namespace {

constexpr size_t kSmemLimit = 232448;   // B200 opt-in dynamic shared memory per CTA

struct Workspace {
  int64_t M = 0, n = 0;
  int rb = 0, cap = 0, N = 0, pmax = 0, wmax = 0, capp = 0, grid = 0, ngrp = 3;
  bool record = false;
  int LDB = 0, LDU = 0;
  double* BUb = nullptr;      // B_U (M x r_B, ld LDB)
  double* W3 = nullptr;       // [W0' | W1 | W2]: three contiguous M x LDU blocks (stream stride M*LDU)
  double* Ubuf[3] = {nullptr, nullptr, nullptr};
  double* Vbuf[3] = {nullptr, nullptr, nullptr};
  double* BV = nullptr;
  double* omega = nullptr;
  int* ints = nullptr;        // rk[N+4], p, w, flags, esc
  double* sigma = nullptr;    // (N+2) x 128
  double* scal = nullptr;     // 8
  double* T1 = nullptr; double* QV = nullptr; double* G = nullptr; double* R1 = nullptr;
  double* R1i = nullptr; double* Wz = nullptr; double* Wv = nullptr;
  double* W0 = nullptr; double* Wfull = nullptr; double* Bprev = nullptr;
  double* partials = nullptr;
  double* Y = nullptr;                          // M x pmax: Y = Ucat R_V^T of the current truncation
  double* Uh = nullptr; double* Vh = nullptr;   // iterate history
  bool arena = false;                           // carved from the caller's lrc_set_workspace buffer
};

enum ProfClass { P_SPMM = 0, P_VSIDE, P_TS_GRAM, P_REDUCE, P_CHOL1, P_CHOL2, P_TS_STORE, P_TRACE,
                 P_MISC, P_TINY, P_TS_GRAM2, P_PREC, P_NCLASS };
const char* const kProfNames[P_NCLASS] = {"spmm", "vside_qr", "ts_gram", "gram_reduce", "chol1",
                                          "chol2_svd", "ts_store", "trace", "misc", "tiny_gemm", "ts_gram2",
                                          "precond"};

struct Pending {             // a solve enqueued by lrc_solve (completed by finish_solve)
  bool active = false;
  int N = 0, rb = 0, cap = 0;
  int64_t M = 0, n = 0;
  uint32_t opt_flags = 0;
  bool record = false;
  lrc_mem where = LRC_MEM_HOST;
  double* U_out = nullptr; double* V_out = nullptr;
  int64_t ld_u = 0, ld_v = 0;
  const double* UN = nullptr; const double* VN = nullptr;
};

struct GraphKey {
  int64_t gen = -1, N = 0; int rb = 0, cap = 0; double gamma = 0, tol = 0; uint32_t flags = 0;
  int64_t pc_gen = 0;
  bool operator==(const GraphKey& o) const {
    return gen == o.gen && N == o.N && rb == o.rb && cap == o.cap && gamma == o.gamma &&
           tol == o.tol && flags == o.flags && pc_gen == o.pc_gen;
  }
};

}  // namespace

struct lrc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::string err;
  // operator
  bool op_set = false, borrowed = false;
  int64_t M = 0, nnz = 0;
  int* row_ptr = nullptr; int* col_idx = nullptr; double* vals[kMaxT] = {};
  int* group_ptr = nullptr; int ngroups = 0;
  int* tdesc = nullptr; int ntiles = 0;
  int* tlist_u = nullptr; int ntl_u = 0; int* tlist_g = nullptr; int ntl_g = 0;
  int* tile_ev = nullptr;   // [ntiles][2] (first nnz, nnz count) of each tile (U tiles first)
  int* trec = nullptr;      // [ntl_u][kRecInts] tile records of the persistent TMA SpMM
  int* tmeta = nullptr;     // [ntl_u][kMetaInts] their first nnz, nnz and U row runs
  size_t meta_bytes = 0;
  double rho = 0, lam = 0;
  // params
  bool par_set = false;
  int64_t n = 0;
  double* dmu = nullptr; double* dnu = nullptr;   // legacy views into dtab (rows 1, 2)
  double* dtab = nullptr;   // right-diagonal table, G x n (legacy: [1, d_mu, d_nu])
  // term list (legacy: the six arrays / three groups of P:30-36; general)
  bool general = false;
  int T = 6, G = 3, id_group = 0;
  int gl_n[kMaxG] = {};
  int gl_t[kMaxG][kGroupTerms] = {};
  double gl_c[kMaxG][kGroupTerms] = {};
  Workspace ws;
  void* user_ws = nullptr;  // caller-owned device arena for the workspace (lrc_set_workspace)
  size_t user_ws_bytes = 0;
  // mean-based preconditioner: P_T values, its spectrum bounds, inner Chebyshev steps
  bool pc_set = false, pc_active = false;
  double pc_min = 0, pc_max = 0;
  int pc_q = 0;
  int64_t pc_gen = 0;
  double* pvals = nullptr;
  double* pcbuf = nullptr; size_t pcbuf_sz = 0;     // Z (3 rotating) + Y: 4 x (3 M LDU) + P^-1 B_U
  double* pc_zero = nullptr;                        // zero diagonals for the dense P application
  std::vector<double> hdtab;                        // host copy of the right-diagonal table (G x n)
  double* gmU = nullptr; double* gmV = nullptr; size_t gm_cap = 0;   // GMREST Krylov basis (library-owned)
  double* gmI = nullptr; double* gmP = nullptr; double* gmG = nullptr;   // identity T, Gram partials, Gram
  double* tmpA = nullptr; size_t tmpA_sz = 0;   // hook scratch (library-owned)
  double* tmpB = nullptr; size_t tmpB_sz = 0;
  double* tmpC = nullptr; size_t tmpC_sz = 0;
  int64_t gen = 0;
  // graph
  cudaGraphExec_t gexec = nullptr;
  GraphKey gkey;
  cudaGraphExec_t bgexec = nullptr;       // lrc_solve_batch graph (this ctx first in the batch)
  std::vector<int64_t> bkey;
  int64_t bgraph_kernels = 0;
  cudaEvent_t ev_k1 = nullptr;            // lrc_solve_batch: the batched SpMM of an iteration is done
  // last solve
  int64_t last_N = 0; bool last_record = false; int last_cap = 0;
  Pending pending;                                   // enqueued solve awaiting finish_solve
  int* h_ints = nullptr; double* h_scal = nullptr; double* h_sigma = nullptr; int h_cap = 0;   // pinned
  float last_kernel_ms = 0.f;
  bool warm_start = true;   // LRC_NO_WARM_START clears it per solve
  int reserved_sms = 0;     // SMs the persistent kernels leave free (concurrent subset solves)
  // kernel launch accounting + optional per-kernel CUDA-event profiling (direct launches only)
  int64_t launches = 0;
  bool capturing = false;
  int64_t capture_count = 0, graph_kernels = 0;
  bool profiling = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<int> evcls;
  double prof_ms[P_NCLASS] = {};
  int64_t prof_n[P_NCLASS] = {};
};

namespace {

lrc_status fail(lrc_ctx* c, lrc_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

#define KL(cls, strm, call)                                                              \
  do {                                                                                    \
    cudaEvent_t e0_ = prof_event(ctx, cls);                                               \
    if (e0_) CK(cudaEventRecord(e0_, strm));                                              \
    CK(call);                                                                             \
    if (e0_) CK(cudaEventRecord(prof_event(ctx, -1), strm));                              \
    if (ctx->capturing) ++ctx->capture_count; else ++ctx->launches;                       \
  } while (0)

// next event of the profiling pool (nullptr when profiling is off); cls < 0: the closing event
cudaEvent_t prof_event(lrc_ctx* ctx, int cls) {
  if (!ctx->profiling || ctx->capturing) return nullptr;
  if (ctx->evused == ctx->evpool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    ctx->evpool.push_back(e);
  }
  if (cls >= 0) ctx->evcls.push_back(cls);
  return ctx->evpool[ctx->evused++];
}

void prof_collect(lrc_ctx* ctx) {   // after a stream synchronize
  for (size_t i = 0; i + 1 < ctx->evused && i / 2 < ctx->evcls.size(); i += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->evpool[i], ctx->evpool[i + 1]) == cudaSuccess) {
      ctx->prof_ms[ctx->evcls[i / 2]] += ms;
      ctx->prof_n[ctx->evcls[i / 2]] += 1;
    }
  }
  ctx->evused = 0;
  ctx->evcls.clear();
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? LRC_ERR_NOMEM : LRC_ERR_CUDA,   \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

void dfree(void* p) { if (p) cudaFree(p); }

cudaMemcpyKind kind_in(lrc_mem where) {
  return where == LRC_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
}
cudaMemcpyKind kind_out(lrc_mem where) {
  return where == LRC_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
}

void free_ws(Workspace& w) {
  if (!w.arena) {
    dfree(w.BUb); dfree(w.W3);
    for (int i = 0; i < 3; ++i) { dfree(w.Ubuf[i]); dfree(w.Vbuf[i]); }
    dfree(w.BV); dfree(w.omega); dfree(w.ints); dfree(w.sigma); dfree(w.scal);
    dfree(w.T1); dfree(w.QV); dfree(w.G); dfree(w.R1); dfree(w.Y);
    dfree(w.R1i); dfree(w.Wz); dfree(w.Wv); dfree(w.W0); dfree(w.Wfull); dfree(w.Bprev);
    dfree(w.partials); dfree(w.Uh); dfree(w.Vh);
  }
  w = Workspace();
}

void drop_graph(lrc_ctx* ctx) {
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  ctx->gexec = nullptr;
  ctx->gkey = GraphKey();
}

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, sizeof(T) * (count ? count : 1));
}

// Hands out the workspace buffers: cudaMalloc (library-owned), a caller arena (lrc_set_workspace,
// 256-byte aligned carving) or a dry run that only counts bytes (lrc_workspace_bytes).
struct Carver {
  char* base = nullptr;     // arena, or null
  size_t cap = 0, used = 0;
  bool dry = false;
  template <typename T>
  cudaError_t get(T** p, size_t count) {
    const size_t bytes = (sizeof(T) * (count ? count : 1) + 255) & ~(size_t)255;
    if (dry) { *p = nullptr; used += bytes; return cudaSuccess; }
    if (base) {
      if (used + bytes > cap) return cudaErrorMemoryAllocation;
      *p = reinterpret_cast<T*>(base + used);
      used += bytes;
      return cudaSuccess;
    }
    used += bytes;
    return dalloc(p, count);
  }
};

// The shape of a workspace for (M, n, r_B <= rb, rank cap, N iterations, wmax).
void ws_shape(const lrc_ctx* ctx, Workspace& w, int rb, int cap, int N, int wmax, bool record) {
  const int p_need = (int)std::min<int64_t>(ctx->n, wmax);
  w.M = ctx->M; w.n = ctx->n; w.rb = rb; w.cap = cap; w.N = N;
  w.pmax = ts_pmax_for(p_need < 1 ? 1 : p_need);
  w.wmax = wmax;
  w.capp = ts_pmax_for(cap);
  w.record = record;
  w.LDB = rb + (rb & 1);
  w.LDU = cap + (cap & 1);
  w.grid = ts_grid_for((int)ctx->M, ctx->reserved_sms);
  w.ngrp = ctx->G;
}

// Every device buffer of a workspace whose shape fields are set.
cudaError_t ws_carve(Workspace& w, Carver& c) {
  const size_t M = (size_t)w.M, n = (size_t)w.n, N = (size_t)w.N, pmax = (size_t)w.pmax;
  cudaError_t e = cudaSuccess;
#define CV(ptr, count) do { if ((e = c.get(ptr, count)) != cudaSuccess) return e; } while (0)
  CV(&w.BUb, M * w.LDB);
  CV(&w.W3, (size_t)w.ngrp * M * w.LDU);
  for (int i = 0; i < 3; ++i) {
    CV(&w.Ubuf[i], M * w.LDU);
    CV(&w.Vbuf[i], n * w.cap);
  }
  CV(&w.BV, n * (w.rb > 0 ? w.rb : 1));
  CV(&w.omega, N + 1);
  CV(&w.ints, N + 16);
  CV(&w.sigma, (N + 4) * kSigmaStride);
  CV(&w.scal, 8);
  CV(&w.T1, (size_t)w.wmax * pmax);
  CV(&w.QV, n * pmax);
  CV(&w.G, pmax * pmax);
  CV(&w.R1, pmax * pmax);
  CV(&w.R1i, pmax * pmax);
  CV(&w.Wz, pmax * w.capp);
  CV(&w.Wv, pmax * w.capp);
  CV(&w.W0, pmax * pmax);
  CV(&w.Wfull, pmax * pmax);
  CV(&w.Bprev, n * pmax);
  CV(&w.partials, (size_t)w.grid * pmax * pmax);
  CV(&w.Y, M * pmax);
  if (w.record) {
    CV(&w.Uh, N * M * w.LDU);
    CV(&w.Vh, N * n * w.cap);
  }
#undef CV
  return e;
}

// Ensure a workspace for (M, n, r_B <= rb, rank cap, N iterations, wmax).  All or nothing: on an
// allocation failure everything allocated so far is released and the workspace is left empty.
lrc_status ensure_ws(lrc_ctx* ctx, int rb, int cap, int N, int wmax, bool record) {
  Workspace& w = ctx->ws;
  const int p_need = (int)std::min<int64_t>(ctx->n, wmax);
  const int pmax = ts_pmax_for(p_need < 1 ? 1 : p_need);
  if (pmax < 0) return fail(ctx, LRC_ERR_ARG, "Gram width out of range");
  if (w.W3 && w.M == ctx->M && w.n == ctx->n && w.ngrp == ctx->G && w.rb >= rb && w.cap == cap && w.N >= N &&
      w.wmax >= wmax && w.pmax == pmax && (!record || w.record))
    return LRC_OK;
  cudaStreamSynchronize(ctx->stream);
  drop_graph(ctx);
  free_ws(w);
  ctx->gen = next_gen();
  Workspace nw;
  ws_shape(ctx, nw, rb, cap, N, wmax, record);
  Carver c;
  c.base = static_cast<char*>(ctx->user_ws);
  c.cap = ctx->user_ws_bytes;
  nw.arena = c.base != nullptr;
  const cudaError_t e = ws_carve(nw, c);
  if (e != cudaSuccess) {
    free_ws(nw);                          // releases the partial allocation (no-op for an arena)
    cudaGetLastError();
    return fail(ctx, LRC_ERR_NOMEM, nw.arena ? "workspace arena too small (see lrc_workspace_bytes)"
                                              : std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  w = nw;
  const size_t M = (size_t)ctx->M, n = (size_t)ctx->n;
  CK(cudaMemsetAsync(w.BUb, 0, sizeof(double) * M * w.LDB, ctx->stream));
  CK(cudaMemsetAsync(w.W3, 0, sizeof(double) * w.ngrp * M * w.LDU, ctx->stream));
  for (int i = 0; i < 3; ++i) {
    CK(cudaMemsetAsync(w.Ubuf[i], 0, sizeof(double) * M * w.LDU, ctx->stream));
    CK(cudaMemsetAsync(w.Vbuf[i], 0, sizeof(double) * n * cap, ctx->stream));
  }
  return LRC_OK;
}

// ensure_ws, and make sure the (possibly reused, wider) workspace still fits the single-CTA V-side
// kernel's shared memory at the wmax / pmax its launches will use
lrc_status ensure_ws_fit(lrc_ctx* ctx, int rb, int cap, int N, int wmax, bool record) {
  lrc_status st = ensure_ws(ctx, rb, cap, N, wmax, record);
  if (st != LRC_OK) return st;
  if (lrc::vside_smem_bytes((int)ctx->n, ctx->ws.wmax, ctx->ws.pmax) > kSmemLimit) {
    cudaStreamSynchronize(ctx->stream);
    drop_graph(ctx);
    free_ws(ctx->ws);
    st = ensure_ws(ctx, rb, cap, N, wmax, record);
    if (st != LRC_OK) return st;
    if (lrc::vside_smem_bytes((int)ctx->n, ctx->ws.wmax, ctx->ws.pmax) > kSmemLimit)
      return fail(ctx, LRC_ERR_ARG, "n x w too large for the single-CTA V-side QR");
  }
  return LRC_OK;
}

lrc_status ensure_tmp(lrc_ctx* ctx, double** p, size_t* sz, size_t count) {
  if (*sz >= count && *p) return LRC_OK;
  cudaStreamSynchronize(ctx->stream);
  dfree(*p);
  *p = nullptr; *sz = 0;
  CK(dalloc(p, count));
  *sz = count;
  return LRC_OK;
}

State make_state(Workspace& w) {
  State s;
  s.rk = w.ints;
  s.p = w.ints + w.N + 4;
  s.w = w.ints + w.N + 5;
  s.flags = w.ints + w.N + 6;
  s.esc = w.ints + w.N + 7;
  s.sweeps = w.ints + w.N + 8;
  s.prevp = w.ints + w.N + 9;
  s.sigma = w.sigma;
  s.scal = w.scal;
  return s;
}

SmallBufs make_bufs(Workspace& w) {
  SmallBufs b{};
  b.T1 = w.T1; b.QV = w.QV; b.G = w.G; b.R1 = w.R1;
  b.R1i = w.R1i; b.Wz = w.Wz; b.Wv = w.Wv;
  b.W0 = nullptr; b.Wfull = w.Wfull; b.Bprev = w.Bprev;
  b.ldT = w.pmax; b.ldZ = w.capp;
  return b;
}

SpmmArgs spmm_base(lrc_ctx* ctx) {
  SpmmArgs a{};
  a.M = (int)ctx->M;
  a.ngroups = ctx->ngroups;
  a.group_ptr = ctx->group_ptr;
  a.ntiles = ctx->ntiles;
  a.tdesc = ctx->tdesc;
  a.tlist_u = ctx->tlist_u; a.ntl_u = ctx->ntl_u;
  a.tile_ev = ctx->tile_ev;
  a.trec = ctx->trec;
  a.tmeta = ctx->tmeta;
  a.reserved_sms = ctx->reserved_sms;
  a.tlist_g = ctx->tlist_g; a.ntl_g = ctx->ntl_g;
  a.tlist = nullptr;
  a.row_ptr = ctx->row_ptr;
  a.col_idx = ctx->col_idx;
  for (int t = 0; t < kMaxT; ++t) a.v[t] = ctx->vals[t];
  a.gen = ctx->general ? 1 : 0; a.T = ctx->T; a.G = ctx->G; a.id_group = ctx->id_group;
  for (int g = 0; g < kMaxG; ++g) {
    a.gl_n[g] = ctx->gl_n[g];
    for (int k = 0; k < kGroupTerms; ++k) { a.gl_t[g][k] = ctx->gl_t[g][k]; a.gl_c[g][k] = ctx->gl_c[g][k]; }
  }
  a.rho = ctx->rho;
  a.lam = ctx->lam;
  return a;
}

// Truncation of Ucat V^T given the Vcat descriptor (a2-a6).  rank_slot / sigma_row: where the
// rank and singular values go; Vout / Uout receive V_{new} (n x cap) and U_{new} (M x cap).
lrc_status enqueue_truncation(lrc_ctx* ctx, const UDesc& ud, const VDesc& vd, const double* omega,
                              int k, double tol, int cap, int rank_slot, int sigma_row,
                              double* Uout, int ldu_out, double* Vout, int ldv_out,
                              cudaStream_t s, bool fork_from_spmm, bool warm = false) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  SmallBufs b = make_bufs(w);
  // warm start of the core Jacobi SVD (p == n only, n <= 256 for the tiny GEMM staging)
  const bool use_warm = warm && ctx->n <= kMaxW;
  if (use_warm) b.W0 = w.W0;
  if (fork_from_spmm && !ctx->profiling) {   // profiling: serial, so per-kernel times are isolated
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    KL(P_VSIDE, ctx->side, launch_vside(vd, (int)ctx->n, ctx->dtab, omega, k, st, b, w.wmax, ctx->side));
    if (use_warm)   // W0 = Q_V^T B_prev (p x p, p = n), overlapping the SpMM
      KL(P_TINY, ctx->side, launch_tiny_gemm(w.QV, w.pmax, w.Bprev, w.pmax, w.W0, w.pmax, w.pmax, st.p, 0,
                                             w.pmax, nullptr, (int)ctx->n, ctx->side, 1));
    CK(cudaEventRecord(ctx->ev_join, ctx->side));
    CK(cudaStreamWaitEvent(s, ctx->ev_join, 0));
  } else {
    KL(P_VSIDE, s, launch_vside(vd, (int)ctx->n, ctx->dtab, omega, k, st, b, w.wmax, s));
    if (use_warm)
      KL(P_TINY, s, launch_tiny_gemm(w.QV, w.pmax, w.Bprev, w.pmax, w.W0, w.pmax, w.pmax, st.p, 0,
                                     w.pmax, nullptr, (int)ctx->n, s, 1));
  }
  // pass 1 over Ucat: Y = Ucat R_V^T (kept: M x pmax), G1 = Y^T Y
  TsArgs ta{};
  ta.M = (int)ctx->M;
  ta.u = ud;
  ta.rk = st.rk;
  ta.T = w.T1;
  ta.ldt = w.pmax;
  ta.d_p = st.p;
  ta.partials = w.partials;
  ta.t_lower = 1;
  ta.yout = w.Y;
  ta.ldy = w.pmax;
  KL(P_TS_GRAM, s, launch_ts(0, ta, w.pmax, w.grid, s));
  KL(P_REDUCE, s, launch_gram_reduce(w.partials, w.grid, w.pmax, w.G, s));
  KL(P_CHOL1, s, launch_chol1(st, b, w.pmax, w.wmax, s));
  // pass 2 over Y (textbook CholeskyQR2: Q1 = Y R1^{-1} from the stored Y), G2 = Q1^T Q1.  The Y block
  // is p wide (p read from the device state); its pad column (odd p) is an exact zero column.
  UDesc yd{};
  yd.nb = 1;
  yd.pad_even = ud.pad_even;
  yd.b[0].p = w.Y;
  yd.b[0].ld = w.pmax;
  yd.b[0].w_fixed = 0;
  yd.b[0].w_idx = (int)(st.p - st.rk);
  TsArgs t2{};
  t2.M = (int)ctx->M;
  t2.u = yd;
  t2.rk = st.rk;
  t2.T = w.R1i;
  t2.ldt = w.pmax;
  t2.d_p = st.p;
  t2.partials = w.partials;
  t2.t_upper = 1;
  KL(P_TS_GRAM2, s, launch_ts(0, t2, w.pmax, w.grid, s));
  KL(P_REDUCE, s, launch_gram_reduce(w.partials, w.grid, w.pmax, w.G, s));
  KL(P_CHOL2, s, launch_chol2_svd(st, b, w.pmax, w.wmax, (int)ctx->n, tol, cap, rank_slot, sigma_row, Vout,
                      ldv_out, s));
  KL(P_TINY, s, launch_tiny_gemm(w.QV, w.pmax, w.Wv, w.capp, Vout, ldv_out, cap, nullptr,
                                 (int)ctx->n, (int)ctx->n, st.p, 0, s));
  if (use_warm)   // B = Q_V W (n x p): the right singular basis of X for the next warm start
    KL(P_TINY, s, launch_tiny_gemm(w.QV, w.pmax, w.Wfull, w.pmax, w.Bprev, w.pmax, w.pmax, nullptr,
                                   (int)ctx->n, (int)ctx->n, st.p, 0, s));
  // basis pass: U' = Y W_r Sigma_r^{-1}
  TsArgs tb{};
  tb.M = (int)ctx->M;
  tb.u = yd;
  tb.rk = st.rk;
  tb.T = w.Wz;
  tb.ldt = w.capp;
  tb.d_p = st.rk + rank_slot;
  tb.out = Uout;
  tb.ldo = ldu_out;
  KL(P_TS_STORE, s, launch_ts(1, tb, w.capp, w.grid, s));
  return LRC_OK;
}

// ||Ucat Vcat^T||_F^2 -> scal[slot]  (vside QR + one Gram pass; X = Y Q_V^T, ||X|| = ||Y||)
lrc_status enqueue_norm2(lrc_ctx* ctx, const UDesc& ud, const VDesc& vd, int slot, cudaStream_t s) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  SmallBufs b = make_bufs(w);
  KL(P_VSIDE, s, launch_vside(vd, (int)ctx->n, ctx->dtab, nullptr, 0, st, b, w.wmax, s));
  TsArgs ta{};
  ta.M = (int)ctx->M;
  ta.u = ud;
  ta.rk = st.rk;
  ta.T = w.T1;
  ta.ldt = w.pmax;
  ta.d_p = st.p;
  ta.partials = w.partials;
  ta.t_lower = 1;
  KL(P_TS_GRAM, s, launch_ts(0, ta, w.pmax, w.grid, s));
  KL(P_REDUCE, s, launch_gram_reduce(w.partials, w.grid, w.pmax, w.G, s));
  KL(P_TRACE, s, launch_trace(st, w.G, w.pmax, slot, s));
  return LRC_OK;
}

UBlock ublock(const double* p, int ld, int w_fixed, int w_idx) {
  UBlock b{};
  b.p = p; b.ld = ld; b.w_fixed = w_fixed; b.w_idx = w_idx;
  return b;
}

// Ucat = [B_U | W0' | W1 | W2 | extra]: the three W blocks have width rk[ridx]
UDesc ucat_desc(const Workspace& w, int64_t M, int rb, int ridx, const double* extra, int extra_idx, int G,
                const double* bu = nullptr) {
  UDesc u{};
  u.nb = 0;
  u.pad_even = 1;      // every block at an even column: 16-byte Ucat copies in the ts kernels
  u.b[u.nb++] = ublock(bu ? bu : w.BUb, w.LDB, rb, -1);
  if (ridx >= 0)
    for (int t = 0; t < G; ++t) u.b[u.nb++] = ublock(w.W3 + (size_t)t * M * w.LDU, w.LDU, 0, ridx);
  if (extra) u.b[u.nb++] = ublock(extra, w.LDU, 0, extra_idx);
  return u;
}

VBlock vblock(const double* ptr, int ld, int w_fixed, int w_idx, double scale, int diag, int use_omega) {
  VBlock v{};
  v.ptr = ptr; v.ld = ld; v.w_fixed = w_fixed; v.w_idx = w_idx; v.w_mul = 1;
  v.scale = scale; v.diag = diag; v.use_omega = use_omega;
  return v;
}

// One ChebyshevT iteration k: X_k -> X_{k+1}.
// K1 of iteration k (a1): W3 = [U_k - g W0 | W1 | W2] from U_k (rank rk[k+1]).
SpmmArgs iteration_spmm_args(lrc_ctx* ctx, int k, double gamma) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  SpmmArgs a = spmm_base(ctx);
  a.U = w.Ubuf[(k + 1) % 3];
  a.ldu = w.LDU;
  a.d_r = st.rk + (k + 1);
  a.out = w.W3;
  a.ldo = w.LDU;
  a.out_off = 0;
  a.out_sstride = (long long)ctx->M * w.LDU;
  a.gamma = gamma;
  return a;
}

// The truncation of iteration k (a2-a6) once W3 holds K1's output; the V-side assembly forks from
// ctx->ev_fork (recorded when U_k / V_k became final) onto the side stream.
const double* pc_pbu(lrc_ctx* ctx);

lrc_status enqueue_iteration_trunc(lrc_ctx* ctx, int k, int rb, int cap, double gamma, double tol, bool record) {
  Workspace& w = ctx->ws;
  cudaStream_t s = ctx->stream;
  double* Uprev = w.Ubuf[k % 3];
  double* Unext = w.Ubuf[(k + 2) % 3];
  double* Vcur = w.Vbuf[(k + 1) % 3];
  double* Vprev = w.Vbuf[k % 3];
  double* Vnext = w.Vbuf[(k + 2) % 3];
  // Vcat = [w g B_V | per group g: w V_k (identity group, paired with W' = U_k - g W) or
  //         -w g d_g * V_k | (1-w) V_{k-1}]   (legacy: d_1 = d_mu, d_2 = d_nu)
  VDesc vd{};
  vd.nb = 0;
  vd.pad_even = 1;
  vd.b[vd.nb++] = vblock(w.BV, rb, rb, -1, gamma, -1, 1);
  for (int g = 0; g < ctx->G; ++g)
    vd.b[vd.nb++] = (g == ctx->id_group) ? vblock(Vcur, cap, 0, k + 1, 1.0, -1, 1)
                                          : vblock(Vcur, cap, 0, k + 1, -gamma, g, 1);
  vd.b[vd.nb++] = vblock(Vprev, cap, 0, k, 1.0, -1, 2);
  const UDesc ud = ucat_desc(w, ctx->M, rb, k + 1, Uprev, k, ctx->G, ctx->pc_active ? pc_pbu(ctx) : nullptr);
  lrc_status r = enqueue_truncation(ctx, ud, vd, w.omega, k, tol, cap, k + 2, k, Unext, w.LDU,
                                    Vnext, cap, s, true, ctx->warm_start);
  if (r != LRC_OK) return r;
  if (record) {
    CK(cudaMemcpyAsync(w.Uh + (size_t)k * ctx->M * w.LDU, Unext,
                       sizeof(double) * ctx->M * w.LDU, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(w.Vh + (size_t)k * ctx->n * cap, Vnext, sizeof(double) * ctx->n * cap,
                       cudaMemcpyDeviceToDevice, s));
  }
  return LRC_OK;
}

std::vector<double> omega_schedule(double lmin, double lmax, int N, int restart);

// Z / Y buffer size of the inner solve: three U-sized blocks (the G <= 6 W blocks go through in
// slices of <= 3) or one B_U block
size_t pc_block(lrc_ctx* ctx) {
  return (size_t)ctx->M * std::max(3 * ctx->ws.LDU, ctx->ws.LDB);
}

// ---- Z = P_T^{-1} R by an inner Chebyshev semi-iteration on P_T (q steps, spectrum
//      bounds [pc_min, pc_max]; reading R15): nb blocks of rows x ncols (ld, block stride bs)
//      of R; the result goes to out (may alias R: the last step reads R before writing the element).
lrc_status enqueue_pinv(lrc_ctx* ctx, const double* R, double* out, int nb, int rows, int ncols, int ld,
                        long long bs, int r_fixed, const int* d_r, cudaStream_t s) {
  const size_t blk = pc_block(ctx);                          // one rotating buffer (<= 3 blocks)
  double* Z[3] = {ctx->pcbuf, ctx->pcbuf + blk, ctx->pcbuf + 2 * blk};
  double* Y = ctx->pcbuf + 3 * blk;
  const std::vector<double> om = omega_schedule(ctx->pc_min, ctx->pc_max, ctx->pc_q, 0);
  const double g = 2.0 / (ctx->pc_min + ctx->pc_max);
  int zc = 0, zp = 1, zn = 2;
  for (int j = 0; j < ctx->pc_q; ++j) {
    double* dst = (j == ctx->pc_q - 1) ? out : Z[zn];
    if (j > 0) {                                             // Y = P Z_c, one dense application per block
      for (int b = 0; b < nb; ++b) {
        SpmmArgs a = spmm_base(ctx);
        a.gen = 0;
        for (int t = 0; t < 6; ++t) a.v[t] = ctx->pvals;
        a.rho = 0.0; a.lam = 0.0; a.dmu = ctx->pc_zero; a.dnu = ctx->pc_zero;
        a.U = Z[zc] + (size_t)b * bs; a.ldu = ld; a.d_r = d_r; a.r_fixed = r_fixed;
        a.out = Y + (size_t)b * bs; a.ldo = ld; a.out_off = 0;
        KL(P_PREC, s, launch_spmm(SPMM_DENSE, a, ncols, s));
      }
    }
    KL(P_PREC, s, launch_cheb_inner(nb, rows, ncols, ld, bs, R, Y, Z[zc], j == 1 ? nullptr : Z[zp], dst, om[j], g,
                                    j == 0 ? 1 : 0, d_r, r_fixed, s));
    const int t = zp; zp = zc; zc = zn; zn = t;
  }
  return LRC_OK;
}

const double* pc_pbu(lrc_ctx* ctx) {                         // P^{-1} B_U (M x LDB) after the buffers
  return ctx->pcbuf + 4 * pc_block(ctx);
}

// the preconditioner's buffers for the current workspace shape
lrc_status ensure_pc_buffers(lrc_ctx* ctx) {
  const size_t need = 4 * pc_block(ctx) + (size_t)ctx->M * ctx->ws.LDB;
  if (ctx->pcbuf_sz < need || !ctx->pcbuf) {
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx->pcbuf);
    ctx->pcbuf = nullptr; ctx->pcbuf_sz = 0;
    CK(dalloc(&ctx->pcbuf, need));
    CK(cudaMemset(ctx->pcbuf, 0, sizeof(double) * need));
    ctx->pcbuf_sz = need;
    drop_graph(ctx);
  }
  return LRC_OK;
}

// One ChebyshevT iteration k: X_k -> X_{k+1}.
lrc_status enqueue_iteration(lrc_ctx* ctx, int k, int rb, int cap, double gamma, double tol,
                             bool record) {
  cudaStream_t s = ctx->stream;
  CK(cudaEventRecord(ctx->ev_fork, s));
  if (!ctx->pc_active) {
    const SpmmArgs a = iteration_spmm_args(ctx, k, gamma);
    KL(P_SPMM, s, launch_spmm(SPMM_S2STEP, a, cap, s));
  } else {
    // preconditioned step (f2): W = L-pieces of U_k (plain), W <- P^{-1} W, W0 <- U_k - gamma W0
    Workspace& w = ctx->ws;
    const SpmmArgs a = iteration_spmm_args(ctx, k, gamma);
    KL(P_SPMM, s, launch_spmm(SPMM_PLAIN3, a, cap, s));
    const long long bs = (long long)ctx->M * w.LDU;
    for (int g0 = 0; g0 < ctx->G; g0 += 3) {
      const int nb = std::min(3, ctx->G - g0);
      lrc_status r = enqueue_pinv(ctx, w.W3 + g0 * bs, w.W3 + g0 * bs, nb, (int)ctx->M, w.LDU, w.LDU, bs, cap, a.d_r, s);
      if (r != LRC_OK) return r;
    }
    const size_t g0 = (size_t)ctx->id_group * ctx->M * w.LDU;
    KL(P_PREC, s, launch_s2_update((int)ctx->M, w.LDU, w.LDU, w.Ubuf[(k + 1) % 3], w.LDU, w.W3 + g0, gamma, s));
  }
  return enqueue_iteration_trunc(ctx, k, rb, cap, gamma, tol, record);
}

std::vector<double> omega_schedule(double lmin, double lmax, int N, int restart) {
  const double c = 0.5 * (lmax - lmin), d = 0.5 * (lmax + lmin);
  std::vector<double> om(N > 0 ? N : 1, 1.0);
  int j = 0;
  double prev = 1.0;
  for (int k = 0; k < N; ++k) {
    if (restart > 0 && k > 0 && k % restart == 0) j = 0;
    double wk;
    if (j == 0) wk = 1.0;
    else if (j == 1) wk = 1.0 / (1.0 - c * c / (2.0 * d * d));
    else wk = 1.0 / (1.0 - prev * c * c / (4.0 * d * d));
    om[k] = wk;
    prev = wk;
    ++j;
  }
  return om;
}

bool valid_mem(lrc_mem m) { return m == LRC_MEM_HOST || m == LRC_MEM_DEVICE; }

cudaError_t ensure_pinned(lrc_ctx* ctx, int N) {
  if (ctx->h_cap >= N && ctx->h_ints) return cudaSuccess;
  if (ctx->h_ints) cudaFreeHost(ctx->h_ints);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->h_sigma) cudaFreeHost(ctx->h_sigma);
  ctx->h_ints = nullptr; ctx->h_scal = nullptr; ctx->h_sigma = nullptr; ctx->h_cap = 0;
  cudaError_t e;
  if ((e = cudaMallocHost((void**)&ctx->h_ints, sizeof(int) * ((size_t)N + 16))) != cudaSuccess) return e;
  if ((e = cudaMallocHost((void**)&ctx->h_scal, sizeof(double) * 8)) != cudaSuccess) return e;
  if ((e = cudaMallocHost((void**)&ctx->h_sigma, sizeof(double) * (size_t)N * kSigmaStride)) != cudaSuccess) return e;
  ctx->h_cap = N;
  return cudaSuccess;
}

lrc_status finish_solve(lrc_ctx* ctx, lrc_solve_info* info) {
  Pending pd = ctx->pending;
  ctx->pending.active = false;
  cudaStream_t s = ctx->stream;
  CK(cudaStreamSynchronize(s));
  prof_collect(ctx);
  Workspace& w = ctx->ws;
  const int N = pd.N;
  const int* ints = ctx->h_ints;
  const double* scal = ctx->h_scal;
  ctx->last_N = N;
  ctx->last_record = pd.record;
  ctx->last_cap = pd.cap;
  const int flags = pd.rb > 0 ? ints[w.N + 6] : 0;
  if (info) {
    float ms_it = 0.f, ms_tot = 0.f;
    cudaEventElapsedTime(&ms_it, ctx->ev[1], ctx->ev[2]);
    cudaEventElapsedTime(&ms_tot, ctx->ev[0], ctx->ev[3]);
    info->rank = pd.rb > 0 ? ints[N + 1] : 0;
    const double b2 = pd.rb > 0 ? scal[0] : 0.0;
    info->b_norm = std::sqrt(b2);
    if (pd.opt_flags & LRC_SKIP_FINAL_RESIDUAL) info->rel_residual = NAN;
    else info->rel_residual = (b2 > 0.0) ? std::sqrt(scal[1] / b2) : 0.0;
    info->diverged = (info->rel_residual > 1.0) ? 1 : 0;
    info->shift_escalations = pd.rb > 0 ? ints[w.N + 7] : 0;
    info->ms_iterations = ms_it;
    info->ms_total = ms_tot;
    if (info->rank_history)
      for (int k = 0; k < N; ++k) info->rank_history[k] = pd.rb > 0 ? ints[k + 2] : 0;
    if (info->sigma_history) {
      if (pd.rb > 0) std::memcpy(info->sigma_history, ctx->h_sigma, sizeof(double) * (size_t)N * kSigmaStride);
      else std::memset(info->sigma_history, 0, sizeof(double) * (size_t)N * kSigmaStride);
    }
    info->jacobi_sweeps = pd.rb > 0 ? ints[w.N + 8] : 0;
    for (int i = 0; i < 3; ++i) info->chol2_cycles[i] = pd.rb > 0 ? scal[4 + i] : 0.0;
  }
  if (flags & 1) return fail(ctx, LRC_ERR_NUMERIC, "shifted Cholesky failed after all escalations");
  if (flags & 2) return fail(ctx, LRC_ERR_NUMERIC, "non-finite singular value in the core SVD");
  if (pd.rb > 0 && pd.where == LRC_MEM_HOST) {   // HOST outputs only now: untouched on error
    CK(cudaMemcpy2DAsync(pd.U_out, sizeof(double) * pd.ld_u, pd.UN, sizeof(double) * w.LDU,
                         sizeof(double) * pd.cap, pd.M, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(pd.V_out, sizeof(double) * pd.ld_v, pd.VN, sizeof(double) * pd.cap,
                         sizeof(double) * pd.cap, pd.n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return LRC_OK;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* lrc_version(void) { return "liblrcheb 0.1 (sm_100a, fp64)"; }

lrc_status lrc_create(lrc_ctx** out, int device, void* cuda_stream) {
  if (!out) return LRC_ERR_ARG;
  *out = nullptr;
  lrc_ctx* ctx = new (std::nothrow) lrc_ctx();
  if (!ctx) return LRC_ERR_NOMEM;
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { g_create_err = cudaGetErrorString(e); delete ctx; return LRC_ERR_CUDA; }
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete ctx; return LRC_ERR_CUDA; }
    ctx->own_stream = true;
  }
  if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_k1, cudaEventDisableTiming) != cudaSuccess) {
    lrc_destroy(ctx);
    return LRC_ERR_CUDA;
  }
  for (int i = 0; i < 4; ++i)
    if (cudaEventCreate(&ctx->ev[i]) != cudaSuccess) { lrc_destroy(ctx); return LRC_ERR_CUDA; }
  cudaError_t pe = spmm_prepare();
  if (pe == cudaSuccess) pe = ts_prepare();
  if (pe == cudaSuccess) pe = small_prepare();
  if (pe != cudaSuccess) {
    g_create_err = std::string("kernel attribute setup: ") + cudaGetErrorString(pe);
    lrc_destroy(ctx);
    return LRC_ERR_CUDA;
  }
  *out = ctx;
  return LRC_OK;
}

void lrc_destroy(lrc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  drop_graph(ctx);
  free_ws(ctx->ws);
  if (!ctx->borrowed) {
    dfree(ctx->row_ptr); dfree(ctx->col_idx);
    for (int t = 0; t < kMaxT; ++t) dfree(ctx->vals[t]);
  }
  dfree(ctx->tmpA); dfree(ctx->tmpB); dfree(ctx->tmpC);
  dfree(ctx->gmU); dfree(ctx->gmV); dfree(ctx->gmI); dfree(ctx->gmP); dfree(ctx->gmG);
  dfree(ctx->pvals); dfree(ctx->pcbuf); dfree(ctx->pc_zero);
  dfree(ctx->group_ptr); dfree(ctx->tdesc); dfree(ctx->tlist_u); dfree(ctx->tlist_g); dfree(ctx->tile_ev); dfree(ctx->trec); dfree(ctx->tmeta); dfree(ctx->dtab);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_k1) cudaEventDestroy(ctx->ev_k1);
  if (ctx->bgexec) cudaGraphExecDestroy(ctx->bgexec);
  for (int i = 0; i < 4; ++i) if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  for (cudaEvent_t e : ctx->evpool) cudaEventDestroy(e);
  if (ctx->h_ints) cudaFreeHost(ctx->h_ints);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->h_sigma) cudaFreeHost(ctx->h_sigma);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* lrc_last_error(const lrc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

float lrc_last_kernel_ms(const lrc_ctx* ctx) { return ctx ? ctx->last_kernel_ms : 0.f; }

int64_t lrc_kernel_launches(const lrc_ctx* ctx) { return ctx ? ctx->launches : 0; }

lrc_status lrc_workspace_bytes(lrc_ctx* ctx, int64_t r_B, int64_t rank_cap, int64_t n_iter, uint32_t flags,
                               size_t* bytes) {
  if (!ctx || !bytes) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_workspace_bytes before set_operator + set_params");
  if (r_B < 0 || r_B > 64 || rank_cap < 1 || rank_cap > kMaxRank || n_iter < 1 || n_iter > 100000)
    return fail(ctx, LRC_ERR_ARG, "r_B / rank_cap / n_iter out of range");
  const int rb = std::max((int)r_B, 1), cap = (int)rank_cap;
  const int wmax = (rb + (rb & 1)) + (ctx->G + 1) * (cap + (cap & 1));
  if (ts_pmax_for((int)std::min<int64_t>(ctx->n, wmax)) < 0) return fail(ctx, LRC_ERR_ARG, "Gram width out of range");
  Workspace w;
  ws_shape(ctx, w, rb, cap, (int)n_iter, wmax, (flags & LRC_RECORD_ITERATES) != 0);
  Carver c;
  c.dry = true;
  ws_carve(w, c);
  *bytes = c.used;
  return LRC_OK;
}

lrc_status lrc_set_workspace(lrc_ctx* ctx, void* dev_ptr, size_t bytes) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (dev_ptr && (reinterpret_cast<uintptr_t>(dev_ptr) & 255)) return fail(ctx, LRC_ERR_ARG, "workspace must be 256-byte aligned");
  if (ctx->pending.active) {
    lrc_status ps = finish_solve(ctx, nullptr);
    if (ps != LRC_OK) return ps;
  }
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  drop_graph(ctx);
  free_ws(ctx->ws);
  ctx->gen = next_gen();
  ctx->user_ws = dev_ptr;
  ctx->user_ws_bytes = dev_ptr ? bytes : 0;
  ctx->last_record = false;
  return LRC_OK;
}

lrc_status lrc_set_reserved_sms(lrc_ctx* ctx, int n) {
  if (!ctx) return LRC_ERR_ARG;
  if (n < 0 || n > 64) return fail(ctx, LRC_ERR_ARG, "reserved SMs must be in [0, 64]");
  if (n != ctx->reserved_sms) {
    cudaStreamSynchronize(ctx->stream);
    drop_graph(ctx);
    free_ws(ctx->ws);      // the persistent grid (and its partial buffers) are sized from it
    ctx->gen = next_gen();
    ctx->reserved_sms = n;
  }
  return LRC_OK;
}

void lrc_set_profiling(lrc_ctx* ctx, int on) {
  if (!ctx) return;
  ctx->profiling = on != 0;
  for (int i = 0; i < P_NCLASS; ++i) { ctx->prof_ms[i] = 0.0; ctx->prof_n[i] = 0; }
  ctx->evused = 0;
  ctx->evcls.clear();
}

int lrc_get_profile(const lrc_ctx* ctx, int cls, const char** name, double* ms_total, int64_t* count) {
  if (cls < 0 || cls >= P_NCLASS) return P_NCLASS;
  if (name) *name = kProfNames[cls];
  if (ms_total) *ms_total = ctx ? ctx->prof_ms[cls] : 0.0;
  if (count) *count = ctx ? ctx->prof_n[cls] : 0;
  return P_NCLASS;
}

}  // extern "C"

namespace {

// The shared pattern + T value arrays (validation, node blocks, SpMM tiles, copies); the term
// structure (legacy or general) is set by the caller afterwards.
lrc_status set_operator_impl(lrc_ctx* ctx, int64_t M, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx,
                             int T, const double* const* vals, double rho_f, double lambda_s, lrc_mem where) {
  ctx->err.clear();
  if (M < 1 || M >= (int64_t)1 << 31) return fail(ctx, LRC_ERR_ARG, "M must be in [1, 2^31)");
  if (nnz < 0 || nnz >= (int64_t)1 << 31) return fail(ctx, LRC_ERR_ARG, "nnz must be in [0, 2^31)");
  if (!row_ptr || (nnz > 0 && !col_idx) || !vals) return fail(ctx, LRC_ERR_ARG, "null pointer");
  for (int t = 0; t < T; ++t)
    if (nnz > 0 && !vals[t]) return fail(ctx, LRC_ERR_ARG, "null value array");
  if (!std::isfinite(rho_f) || !std::isfinite(lambda_s)) return fail(ctx, LRC_ERR_ARG, "rho_f, lambda_s must be finite");
  if (where != LRC_MEM_HOST && where != LRC_MEM_DEVICE && where != LRC_MEM_DEVICE_BORROW)
    return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  CK(cudaSetDevice(ctx->device));
  // host copies of the pattern for validation + node-block detection
  std::vector<int32_t> hrp(M + 1), hci(nnz);
  if (where == LRC_MEM_HOST) {
    std::memcpy(hrp.data(), row_ptr, sizeof(int32_t) * (M + 1));
    if (nnz) std::memcpy(hci.data(), col_idx, sizeof(int32_t) * nnz);
  } else {
    CK(cudaMemcpy(hrp.data(), row_ptr, sizeof(int32_t) * (M + 1), cudaMemcpyDeviceToHost));
    if (nnz) CK(cudaMemcpy(hci.data(), col_idx, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
  }
  if (hrp[0] != 0) return fail(ctx, LRC_ERR_ARG, "row_ptr[0] != 0");
  if (hrp[M] != nnz) return fail(ctx, LRC_ERR_ARG, "row_ptr[M] != nnz");
  for (int64_t i = 0; i < M; ++i) {
    if (hrp[i + 1] < hrp[i]) return fail(ctx, LRC_ERR_ARG, "row_ptr not non-decreasing at row " + std::to_string(i));
    for (int32_t e = hrp[i]; e < hrp[i + 1]; ++e) {
      if (hci[e] < 0 || hci[e] >= M) return fail(ctx, LRC_ERR_ARG, "col_idx out of range in row " + std::to_string(i));
      if (e > hrp[i] && hci[e] <= hci[e - 1])
        return fail(ctx, LRC_ERR_ARG, "col_idx not strictly increasing in row " + std::to_string(i));
    }
  }
  // node blocks: runs of consecutive rows with identical column lists (<= kGroupMax rows)
  std::vector<int32_t> groups;
  groups.reserve(M / 4 + 2);
  groups.push_back(0);
  int gsz = 1;
  for (int64_t i = 1; i < M; ++i) {
    const int32_t l0 = hrp[i] - hrp[i - 1], l1 = hrp[i + 1] - hrp[i];
    bool same = (gsz < kGroupMax) && l0 == l1 &&
                (l1 == 0 || std::memcmp(&hci[hrp[i - 1]], &hci[hrp[i]], sizeof(int32_t) * l1) == 0);
    if (same) { ++gsz; }
    else { groups.push_back((int32_t)i); gsz = 1; }
  }
  groups.push_back((int32_t)M);
  // CTA tiles of the fused SpMM: <= kTileBlocks node blocks, <= kSpmmCap nnz,
  // <= kValCap staged doubles, and -- for the shared-memory U path -- the deduplicated set of U rows
  // the tile's column lists touch (<= kUCap rows) with a 16-bit local index per column-list entry.
  // Everything a CTA needs is packed into one kDescInts-word descriptor (one coalesced load).
  // A block that alone exceeds a bound gets its own tile on the L2-gather path (nu = 0).
  std::vector<int32_t> tdesc;
  {
    const int ng = (int)groups.size() - 1;
    std::vector<int32_t> uni, merged;
    std::vector<int> tb;                           // blocks of the open tile
    int64_t tn = 0, tv = 0, tl = 0;
    auto block_cols = [&](int gi, const int32_t*& c, int& L) {
      c = hci.data() + hrp[groups[gi]];
      L = hrp[groups[gi] + 1] - hrp[groups[gi]];
    };
    auto close_tile = [&](bool ushared) {
      std::vector<int32_t> d(kDescInts, 0);
      const int r0 = groups[tb.front()], r1 = groups[tb.back() + 1];
      d[0] = hrp[r0];
      d[1] = hrp[r1] - hrp[r0];
      d[2] = (int)tb.size();
      d[3] = ushared ? (int)uni.size() : 0;
      d[4] = r0;
      d[5] = r1;
      d[6] = 0;                            // staged doubles (three grouped streams, padded rows)
      uint16_t* lx = reinterpret_cast<uint16_t*>(d.data() + kDescLidx);
      int lo = 0;
      for (size_t b = 0; b < tb.size(); ++b) {
        const int gi = tb[b];
        const int32_t* c; int L;
        block_cols(gi, c, L);
        d[8 + b] = groups[gi];
        d[12 + b] = groups[gi + 1] - groups[gi];
        d[16 + b] = L;
        d[6] += 3 * (groups[gi + 1] - groups[gi]) * (L + ((20 - (L & 15)) & 15));
        d[20 + b] = -1;                    // local row of the block's first row in the staged U rows
        if (ushared) {
          auto it = std::lower_bound(uni.begin(), uni.end(), (int32_t)groups[gi]);
          const int g = groups[gi + 1] - groups[gi];
          if (it != uni.end() && *it == groups[gi] && (it - uni.begin()) + g <= (long)uni.size() &&
              *(it + (g - 1)) == groups[gi] + g - 1)
            d[20 + b] = (int32_t)(it - uni.begin());
        }
        if (ushared)
          for (int j = 0; j < L; ++j)
            lx[lo + j] = (uint16_t)(std::lower_bound(uni.begin(), uni.end(), c[j]) - uni.begin());
        lo += L;
      }
      if (ushared)
        for (size_t u = 0; u < uni.size(); ++u) d[kDescUrows + u] = uni[u];
      tdesc.insert(tdesc.end(), d.begin(), d.end());
      tb.clear(); uni.clear(); tn = tv = tl = 0;
    };
    for (int gi = 0; gi < ng; ++gi) {
      const int g = groups[gi + 1] - groups[gi];
      const int32_t* c; int L;
      block_cols(gi, c, L);
      const int64_t gn = (int64_t)g * L;
      const int lp = L + ((20 - (L & 15)) & 15);     // row pitch of the staged values (spmm.cu)
      const int64_t gv = (int64_t)3 * g * lp;
      merged.clear();
      std::set_union(uni.begin(), uni.end(), c, c + L, std::back_inserter(merged));
      const bool fits = (int)tb.size() < kTileBlocks && tn + gn <= kSpmmCap && tv + gv <= kValCap &&
                        tl + L <= kLidxCap && (int)merged.size() <= kUCap && g <= 5;
      if (!fits && !tb.empty()) {
        close_tile(true);
        merged.assign(c, c + L);
      }
      const bool alone_ok = gn <= kSpmmCap && gv <= kValCap && L <= kUCap && L <= kLidxCap && g <= 5;
      if (!alone_ok) {                       // generic long / tall block: L2-gather path, own tile
        tb.push_back(gi);
        close_tile(false);
        continue;
      }
      uni.swap(merged);
      tb.push_back(gi);
      tn += gn; tv += gv; tl += L;
    }
    if (!tb.empty()) close_tile(true);
  }

  CK(cudaStreamSynchronize(ctx->stream));
  drop_graph(ctx);
  free_ws(ctx->ws);
  if (!ctx->borrowed) {
    dfree(ctx->row_ptr); dfree(ctx->col_idx);
    for (int t = 0; t < kMaxT; ++t) dfree(ctx->vals[t]);
  }
  dfree(ctx->group_ptr);
  dfree(ctx->tdesc); dfree(ctx->tlist_u); dfree(ctx->tlist_g); dfree(ctx->tile_ev); dfree(ctx->trec); dfree(ctx->tmeta);
  ctx->tlist_u = ctx->tlist_g = nullptr; ctx->tile_ev = nullptr; ctx->trec = nullptr; ctx->tmeta = nullptr;
  ctx->row_ptr = nullptr; ctx->col_idx = nullptr; ctx->group_ptr = nullptr; ctx->tdesc = nullptr;
  for (int t = 0; t < kMaxT; ++t) ctx->vals[t] = nullptr;
  ctx->op_set = false;
  ctx->par_set = false;   // params depend on nothing here, but workspaces do; keep semantics simple
  ctx->gen = next_gen();

  if (where == LRC_MEM_DEVICE_BORROW) {
    ctx->borrowed = true;
    ctx->row_ptr = const_cast<int*>(row_ptr);
    ctx->col_idx = const_cast<int*>(col_idx);
    for (int t = 0; t < T; ++t) ctx->vals[t] = const_cast<double*>(vals[t]);
  } else {
    ctx->borrowed = false;
    CK(dalloc(&ctx->row_ptr, M + 1));
    CK(dalloc(&ctx->col_idx, nnz));
    CK(cudaMemcpy(ctx->row_ptr, hrp.data(), sizeof(int32_t) * (M + 1), cudaMemcpyHostToDevice));
    if (nnz) CK(cudaMemcpy(ctx->col_idx, hci.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    for (int t = 0; t < T; ++t) {
      CK(dalloc(&ctx->vals[t], nnz));
      if (nnz) CK(cudaMemcpy(ctx->vals[t], vals[t], sizeof(double) * nnz, kind_in(where)));
    }
  }
  CK(dalloc(&ctx->group_ptr, groups.size()));
  CK(cudaMemcpy(ctx->group_ptr, groups.data(), sizeof(int32_t) * groups.size(), cudaMemcpyHostToDevice));
  ctx->ngroups = (int)groups.size() - 1;
  ctx->ntiles = (int)(tdesc.size() / kDescInts);
  {
    // shared-memory-U tiles first (stable): the hot kernel then indexes tiles by blockIdx.x and
    // reads the (e0, nnz) pair of its tile from a side array, in parallel with the descriptor
    std::vector<int32_t> perm;
    for (int t = 0; t < ctx->ntiles; ++t) if (tdesc[(size_t)t * kDescInts + 3] > 0) perm.push_back(t);
    for (int t = 0; t < ctx->ntiles; ++t) if (tdesc[(size_t)t * kDescInts + 3] <= 0) perm.push_back(t);
    std::vector<int32_t> sorted(tdesc.size()), ev(2 * (size_t)ctx->ntiles + 2, 0);
    for (int i = 0; i < ctx->ntiles; ++i) {
      std::copy(tdesc.begin() + (size_t)perm[i] * kDescInts, tdesc.begin() + (size_t)(perm[i] + 1) * kDescInts,
                sorted.begin() + (size_t)i * kDescInts);
      ev[2 * i] = sorted[(size_t)i * kDescInts + 0];
      ev[2 * i + 1] = sorted[(size_t)i * kDescInts + 1];
    }
    tdesc.swap(sorted);
    CK(dalloc(&ctx->tile_ev, ev.size()));
    CK(cudaMemcpy(ctx->tile_ev, ev.data(), sizeof(int32_t) * ev.size(), cudaMemcpyHostToDevice));
  }
  CK(dalloc(&ctx->tdesc, tdesc.size()));
  CK(cudaMemcpy(ctx->tdesc, tdesc.data(), sizeof(int32_t) * tdesc.size(), cudaMemcpyHostToDevice));
  {
    // tile records + U row runs of the persistent TMA SpMM (lrc_internal.cuh) for the shared-memory-U
    // tiles (stored first); not built when some tile exceeds the kernel's bounds (then the launcher
    // keeps the 3-CTA kernel)
    std::vector<int32_t> rec, runs;
    bool ok = true;
    for (int t = 0; t < ctx->ntiles && ok; ++t) {
      const int32_t* d = tdesc.data() + (size_t)t * kDescInts;
      if (d[3] <= 0) break;
      if (d[1] > kTileNnz || d[3] > kTileUrows) { ok = false; break; }
      std::vector<int32_t> R(kRecInts, 0), Q(kMetaInts, 0);
      R[0] = d[0]; R[1] = d[1]; R[2] = d[2]; R[3] = d[3];
      const uint16_t* lx = reinterpret_cast<const uint16_t*>(d + kDescLidx);
      int lo = 0, eb = 0;
      for (int b = 0; b < d[2]; ++b) {
        const int g = d[12 + b], L = d[16 + b];
        if (lo + L > kRecCols) { ok = false; break; }
        R[4 + b] = d[8 + b]; R[8 + b] = g; R[12 + b] = L; R[16 + b] = lo; R[20 + b] = eb; R[24 + b] = d[20 + b];
        for (int j = 0; j < L; ++j) R[kRecHdr + lo + j] = lx[lo + j];
        lo += L;
        eb += g * L;
      }
      int nr = 0;
      for (int u = 0; u < d[3] && ok; ) {
        int v = u + 1;
        while (v < d[3] && d[kDescUrows + v] == d[kDescUrows + v - 1] + 1) ++v;
        if (nr == kMetaRuns) { ok = false; break; }
        Q[4 + 3 * nr] = d[kDescUrows + u]; Q[5 + 3 * nr] = v - u; Q[6 + 3 * nr] = u;
        ++nr;
        u = v;
      }
      Q[0] = d[0]; Q[1] = d[1]; Q[2] = nr;
      rec.insert(rec.end(), R.begin(), R.end());
      runs.insert(runs.end(), Q.begin(), Q.end());
    }
    dfree(ctx->trec); dfree(ctx->tmeta);
    ctx->trec = nullptr; ctx->tmeta = nullptr;
    if (ok && !rec.empty()) {
      CK(dalloc(&ctx->trec, rec.size()));
      CK(cudaMemcpy(ctx->trec, rec.data(), sizeof(int32_t) * rec.size(), cudaMemcpyHostToDevice));
      CK(dalloc(&ctx->tmeta, runs.size()));
      CK(cudaMemcpy(ctx->tmeta, runs.data(), sizeof(int32_t) * runs.size(), cudaMemcpyHostToDevice));
    }
  }
  {
    std::vector<int32_t> lu, lg;
    for (int t = 0; t < ctx->ntiles; ++t) (tdesc[(size_t)t * kDescInts + 3] > 0 ? lu : lg).push_back(t);
    CK(dalloc(&ctx->tlist_u, lu.size()));
    CK(dalloc(&ctx->tlist_g, lg.size()));
    if (!lu.empty()) CK(cudaMemcpy(ctx->tlist_u, lu.data(), sizeof(int32_t) * lu.size(), cudaMemcpyHostToDevice));
    if (!lg.empty()) CK(cudaMemcpy(ctx->tlist_g, lg.data(), sizeof(int32_t) * lg.size(), cudaMemcpyHostToDevice));
    ctx->ntl_u = (int)lu.size();
    ctx->ntl_g = (int)lg.size();
  }
  ctx->meta_bytes = sizeof(int32_t) * tdesc.size();
  ctx->M = M;
  ctx->nnz = nnz;
  ctx->rho = rho_f;
  ctx->lam = lambda_s;
  ctx->op_set = true;
  return LRC_OK;
}

void set_legacy_terms(lrc_ctx* ctx) {
  ctx->general = false; ctx->T = 6; ctx->G = 3; ctx->id_group = 0;
  for (int g = 0; g < kMaxG; ++g) ctx->gl_n[g] = 0;
}

}  // namespace

extern "C" {

lrc_status lrc_set_operator(lrc_ctx* ctx, int64_t M, int64_t nnz, const int32_t* row_ptr,
                            const int32_t* col_idx, const double* const vals[6], double rho_f,
                            double lambda_s, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  if (!std::isfinite(rho_f) || !std::isfinite(lambda_s)) return fail(ctx, LRC_ERR_ARG, "rho_f, lambda_s must be finite");
  lrc_status st = set_operator_impl(ctx, M, nnz, row_ptr, col_idx, 6, vals, rho_f, lambda_s, where);
  if (st == LRC_OK) set_legacy_terms(ctx);
  return st;
}

lrc_status lrc_set_operator_terms(lrc_ctx* ctx, int64_t M, int64_t nnz, const int32_t* row_ptr,
                                  const int32_t* col_idx, int T, const double* const* vals, int G,
                                  const double* coef, int id_group, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (T < 1 || T > kMaxT) return fail(ctx, LRC_ERR_ARG, "T must be in [1, 8]");
  if (G < 1 || G > kMaxG) return fail(ctx, LRC_ERR_ARG, "G must be in [1, 6]");
  if (!coef) return fail(ctx, LRC_ERR_ARG, "null coef");
  if (id_group < 0 || id_group >= G) return fail(ctx, LRC_ERR_ARG, "id_group must name one of the G groups");
  int gl_n[kMaxG] = {}, gl_t[kMaxG][kGroupTerms] = {};
  double gl_c[kMaxG][kGroupTerms] = {};
  for (int t = 0; t < T; ++t)
    for (int g = 0; g < G; ++g) {
      const double c = coef[t * G + g];
      if (!std::isfinite(c)) return fail(ctx, LRC_ERR_ARG, "coefficients must be finite");
      if (c == 0.0) continue;
      if (gl_n[g] == kGroupTerms) return fail(ctx, LRC_ERR_ARG, "at most 6 arrays per right-diagonal group");
      gl_t[g][gl_n[g]] = t; gl_c[g][gl_n[g]] = c; ++gl_n[g];
    }
  lrc_status st = set_operator_impl(ctx, M, nnz, row_ptr, col_idx, T, vals, 0.0, 0.0, where);
  if (st != LRC_OK) return st;
  if (!ctx->trec) {     // general term lists run on the persistent TMA kernel only
    ctx->op_set = false;
    return fail(ctx, LRC_ERR_ARG, "general term lists need an FE-like pattern (node-block tiles <= 900 nnz, <= 90 "
                                  "U rows, <= 4 row runs)");
  }
  ctx->general = true; ctx->T = T; ctx->G = G; ctx->id_group = id_group;
  for (int g = 0; g < kMaxG; ++g) {
    ctx->gl_n[g] = gl_n[g];
    for (int k = 0; k < kGroupTerms; ++k) { ctx->gl_t[g][k] = gl_t[g][k]; ctx->gl_c[g][k] = gl_c[g][k]; }
  }
  return LRC_OK;
}

lrc_status lrc_set_diagonals(lrc_ctx* ctx, int64_t n, int G, const double* diags, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->general) return fail(ctx, LRC_ERR_STATE, "lrc_set_diagonals needs lrc_set_operator_terms first");
  if (G != ctx->G) return fail(ctx, LRC_ERR_SHAPE, "G differs from the operator's term list");
  if (n < 1 || n > 1024) return fail(ctx, LRC_ERR_ARG, "n must be in [1, 1024]");
  if (!diags) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  CK(cudaSetDevice(ctx->device));
  std::vector<double> h((size_t)G * n);
  CK(cudaMemcpy(h.data(), diags, sizeof(double) * h.size(), where == LRC_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  for (double x : h) if (!std::isfinite(x)) return fail(ctx, LRC_ERR_ARG, "diagonals must be finite");
  for (int64_t i = 0; i < n; ++i)
    if (h[(size_t)ctx->id_group * n + i] != 1.0) return fail(ctx, LRC_ERR_ARG, "the id_group diagonal must be all ones");
  CK(cudaStreamSynchronize(ctx->stream));
  if (n != ctx->n || !ctx->dtab) {
    drop_graph(ctx);
    free_ws(ctx->ws);
    dfree(ctx->dtab);
    ctx->dtab = nullptr;
    CK(dalloc(&ctx->dtab, (size_t)kMaxG * n));
  }
  CK(cudaMemcpy(ctx->dtab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  ctx->hdtab = h;
  ctx->pc_set = false;
  ctx->dmu = ctx->dnu = nullptr;
  ctx->n = n;
  ctx->par_set = true;
  return LRC_OK;
}

lrc_status lrc_set_params(lrc_ctx* ctx, int64_t n, const double* d_mu, const double* d_nu, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set) return fail(ctx, LRC_ERR_STATE, "lrc_set_params before lrc_set_operator");
  if (ctx->general) return fail(ctx, LRC_ERR_STATE, "a general term list takes lrc_set_diagonals");
  if (n < 1 || n > 1024) return fail(ctx, LRC_ERR_ARG, "n must be in [1, 1024]");
  if (!d_mu || !d_nu) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  CK(cudaSetDevice(ctx->device));
  std::vector<double> hm(n), hn(n);
  CK(cudaMemcpy(hm.data(), d_mu, sizeof(double) * n, where == LRC_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hn.data(), d_nu, sizeof(double) * n, where == LRC_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(hm[i]) || !std::isfinite(hn[i])) return fail(ctx, LRC_ERR_ARG, "d_mu / d_nu must be finite");
  CK(cudaStreamSynchronize(ctx->stream));
  if (n != ctx->n || !ctx->dtab) {
    drop_graph(ctx);
    free_ws(ctx->ws);
    dfree(ctx->dtab);
    ctx->dtab = nullptr;
    CK(dalloc(&ctx->dtab, (size_t)kMaxG * n));
  }
  // right-diagonal table of the three groups: [1, d_mu, d_nu]
  std::vector<double> h(3 * (size_t)n, 1.0);
  std::copy(hm.begin(), hm.end(), h.begin() + n);
  std::copy(hn.begin(), hn.end(), h.begin() + 2 * n);
  CK(cudaMemcpy(ctx->dtab, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  ctx->hdtab = h;
  ctx->pc_set = false;                             // the preconditioner follows the parameters
  ctx->dmu = ctx->dtab + n;
  ctx->dnu = ctx->dtab + 2 * n;
  ctx->n = n;
  ctx->par_set = true;
  return LRC_OK;
}

// P_T = sum_t c_t A_t * mean(e_t) on the device, applied inside
// the iteration by q steps of an inner Chebyshev semi-iteration on [p_min, p_max].
lrc_status lrc_set_preconditioner(lrc_ctx* ctx, double p_min, double p_max, int64_t inner_steps) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_set_preconditioner before set_operator + parameters");
  if (!(p_min > 0.0) || !(p_max >= p_min) || !std::isfinite(p_max))
    return fail(ctx, LRC_ERR_ARG, "need 0 < p_min <= p_max");
  if (inner_steps < 1 || inner_steps > 1000) return fail(ctx, LRC_ERR_ARG, "inner_steps must be in [1, 1000]");
  CK(cudaSetDevice(ctx->device));
  const int64_t n = ctx->n;
  const int G = ctx->general ? ctx->G : 3;
  if ((int64_t)ctx->hdtab.size() < (int64_t)G * n) return fail(ctx, LRC_ERR_STATE, "parameters not set");
  double mid[kMaxG];
  for (int g = 0; g < G; ++g) {                    // midpoint of each right diagonal's range
    double lo = ctx->hdtab[(size_t)g * n], hi = lo;
    for (int64_t i = 1; i < n; ++i) {
      lo = std::min(lo, ctx->hdtab[(size_t)g * n + i]);
      hi = std::max(hi, ctx->hdtab[(size_t)g * n + i]);
    }
    mid[g] = 0.5 * (lo + hi);
  }
  PvalArgs pa{};
  int T;
  if (!ctx->general) {                             // arrays [A0, A1, A2, Jrho, Jmu, Jlam], e_t means
    T = 6;
    const double e[6] = {1.0, mid[1], ctx->rho * mid[2], ctx->rho, mid[1], ctx->lam};
    for (int t = 0; t < 6; ++t) { pa.v[t] = ctx->vals[t]; pa.e[t] = e[t]; }
  } else {                                         // e_t = sum_g C[t][g] mean(d_g)
    T = ctx->T;
    for (int t = 0; t < T; ++t) { pa.v[t] = ctx->vals[t]; pa.e[t] = 0.0; }
    for (int g = 0; g < ctx->G; ++g)
      for (int k = 0; k < ctx->gl_n[g]; ++k) pa.e[ctx->gl_t[g][k]] += ctx->gl_c[g][k] * mid[g];
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (!ctx->pvals) CK(dalloc(&ctx->pvals, (size_t)std::max<int64_t>(ctx->nnz, 1)));
  if (!ctx->pc_zero) {
    CK(dalloc(&ctx->pc_zero, 256));
    CK(cudaMemset(ctx->pc_zero, 0, sizeof(double) * 256));
  }
  CK(launch_form_pvals(pa, T, (long long)ctx->nnz, ctx->pvals, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->pc_min = p_min; ctx->pc_max = p_max; ctx->pc_q = (int)inner_steps;
  ctx->pc_gen = next_gen();
  ctx->pc_set = true;
  return LRC_OK;
}

}  // extern "C"

namespace {

// ---- lrc_solve in phases (shared with lrc_solve_batch) ------------------------------------------
struct SolveCall {
  const double* B_U; int64_t ld_bu; const double* B_V; int64_t ld_bv;
  double* U_out; int64_t ld_u; double* V_out; int64_t ld_v;
  int rb, N, cap, wmax;
  double gamma;
  bool record;
};

lrc_status solve_validate(lrc_ctx* ctx, const double* B_U, int64_t ld_bu, const double* B_V, int64_t ld_bv,
                          int64_t r_B, const lrc_solve_opts* opts, double* U_out, int64_t ld_u, double* V_out,
                          int64_t ld_v, lrc_mem where, SolveCall& sc) {
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_solve before lrc_set_operator + lrc_set_params");
  if (!opts) return fail(ctx, LRC_ERR_ARG, "null opts");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  const double lmin = opts->lambda_min, lmax = opts->lambda_max;
  if (!(lmin > 0.0) || !(lmax >= lmin) || !std::isfinite(lmax))
    return fail(ctx, LRC_ERR_ARG, "need 0 < lambda_min <= lambda_max (d > c >= 0)");
  if (!(opts->tol >= 0.0) || !std::isfinite(opts->tol)) return fail(ctx, LRC_ERR_ARG, "tol must be finite and >= 0");
  const int64_t M = ctx->M, n = ctx->n;
  if (opts->rank_cap < 1 || opts->rank_cap > std::min<int64_t>(std::min(M, n), kMaxRank))
    return fail(ctx, LRC_ERR_ARG, "rank_cap must be in [1, min(M, n, 128)]");
  if (opts->n_iter < 1 || opts->n_iter > 100000) return fail(ctx, LRC_ERR_ARG, "n_iter must be in [1, 100000]");
  if (opts->restart_every < 0) return fail(ctx, LRC_ERR_ARG, "restart_every must be >= 0");
  if (r_B < 0 || r_B > 64) return fail(ctx, LRC_ERR_ARG, "r_B must be in [0, 64]");
  if (r_B > 0 && (!B_U || !B_V)) return fail(ctx, LRC_ERR_ARG, "null B_U / B_V");
  if (r_B > 0 && (ld_bu < r_B || ld_bv < r_B)) return fail(ctx, LRC_ERR_SHAPE, "ld_bu / ld_bv < r_B");
  const int cap = (int)opts->rank_cap;
  if (!U_out || !V_out) return fail(ctx, LRC_ERR_ARG, "null output");
  if (ld_u < cap || ld_v < cap) return fail(ctx, LRC_ERR_SHAPE, "ld_u / ld_v < rank_cap");
  const int rb = (int)r_B, N = (int)opts->n_iter;
  // widest concatenation: every block padded to an even width (UDesc::pad_even)
  const int wmax = (rb + (rb & 1)) + (ctx->G + 1) * (cap + (cap & 1));
  if (wmax > kMaxW) return fail(ctx, LRC_ERR_ARG, "r_B + (G + 1) rank_cap must be <= 256");
  const int p_need = (int)std::min<int64_t>(n, wmax);
  if (p_need > 112) return fail(ctx, LRC_ERR_ARG, "min(n, r_B + 4 rank_cap) must be <= 112 in this build");
  if (lrc::vside_smem_bytes((int)n, wmax, ts_pmax_for(p_need)) > kSmemLimit)
    return fail(ctx, LRC_ERR_ARG, "n x (r_B + 4 rank_cap) too large for the single-CTA V-side QR");
  if ((opts->flags & LRC_ASYNC) && where != LRC_MEM_DEVICE)
    return fail(ctx, LRC_ERR_ARG, "LRC_ASYNC needs DEVICE inputs and outputs");
  if ((opts->flags & LRC_PRECONDITIONED) && !ctx->pc_set)
    return fail(ctx, LRC_ERR_STATE, "LRC_PRECONDITIONED before lrc_set_preconditioner (or the parameters changed)");
  if (ctx->pending.active) {                         // an LRC_ASYNC solve never waited for
    lrc_status ps = finish_solve(ctx, nullptr);
    if (ps != LRC_OK) return ps;
  }
  sc.B_U = B_U; sc.ld_bu = ld_bu; sc.B_V = B_V; sc.ld_bv = ld_bv;
  sc.U_out = U_out; sc.ld_u = ld_u; sc.V_out = V_out; sc.ld_v = ld_v;
  sc.rb = rb; sc.N = N; sc.cap = cap; sc.wmax = wmax;
  sc.gamma = 2.0 / (lmax + lmin);
  sc.record = (opts->flags & LRC_RECORD_ITERATES) != 0;
  return LRC_OK;
}

// workspace, inputs, omega sequence, state reset and ||B||_F^2, on ctx's stream (ends with ev[1])
lrc_status solve_prologue(lrc_ctx* ctx, const lrc_solve_opts* opts, lrc_mem where, const SolveCall& sc) {
  ctx->warm_start = (opts->flags & LRC_NO_WARM_START) == 0;
  CK(cudaSetDevice(ctx->device));
  lrc_status st = ensure_ws_fit(ctx, std::max(sc.rb, 1), sc.cap, sc.N, sc.wmax, sc.record);
  if (st != LRC_OK) return st;
  ctx->pc_active = (opts->flags & LRC_PRECONDITIONED) != 0;
  if (ctx->pc_active) {
    st = ensure_pc_buffers(ctx);
    if (st != LRC_OK) return st;
  }
  Workspace& w = ctx->ws;
  cudaStream_t s = ctx->stream;
  const int64_t M = ctx->M, n = ctx->n;
  CK(cudaEventRecord(ctx->ev[0], s));
  if (sc.rb > 0) {
    CK(cudaMemcpy2DAsync(w.BUb, sizeof(double) * w.LDB, sc.B_U, sizeof(double) * sc.ld_bu,
                         sizeof(double) * sc.rb, M, kind_in(where), s));
    CK(cudaMemcpy2DAsync(w.BV, sizeof(double) * sc.rb, sc.B_V, sizeof(double) * sc.ld_bv,
                         sizeof(double) * sc.rb, n, kind_in(where), s));
  }
  std::vector<double> om = omega_schedule(opts->lambda_min, opts->lambda_max, sc.N, (int)opts->restart_every);
  CK(cudaMemcpyAsync(w.omega, om.data(), sizeof(double) * sc.N, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(w.ints, 0, sizeof(int) * (w.N + 16), s));
  CK(cudaMemsetAsync(w.scal, 0, sizeof(double) * 8, s));
  CK(cudaMemsetAsync(w.sigma, 0, sizeof(double) * (size_t)(sc.N + 4) * kSigmaStride, s));
  if (sc.rb > 0) {
    const UDesc ub = ucat_desc(w, M, sc.rb, -1, nullptr, -1, ctx->G);
    VDesc vb{};
    vb.nb = 1;
    vb.pad_even = 1;
    vb.b[0] = vblock(w.BV, sc.rb, sc.rb, -1, 1.0, -1, 0);
    st = enqueue_norm2(ctx, ub, vb, 0, s);
    if (st != LRC_OK) return st;
    if (ctx->pc_active) {                          // P^{-1} B_U once per solve (f2)
      st = enqueue_pinv(ctx, w.BUb, const_cast<double*>(pc_pbu(ctx)), 1, (int)M, w.LDB, w.LDB, 0, sc.rb, nullptr, s);
      if (st != LRC_OK) return st;
    }
  }
  CK(cudaEventRecord(ctx->ev[1], s));
  return LRC_OK;
}

// after the iterations (ctx's stream): ev[2], final residual, outputs, ev[3], result mirrors, pending
lrc_status solve_epilogue(lrc_ctx* ctx, const lrc_solve_opts* opts, lrc_mem where, const SolveCall& sc) {
  Workspace& w = ctx->ws;
  cudaStream_t s = ctx->stream;
  State sd = make_state(w);
  const int64_t M = ctx->M, n = ctx->n;
  const int N = sc.N, cap = sc.cap, rb = sc.rb;
  CK(cudaEventRecord(ctx->ev[2], s));
  if (rb > 0) {
    const int slotN = N + 1;   // rk index of X_N
    double* UN = w.Ubuf[(N + 1) % 3];
    double* VN = w.Vbuf[(N + 1) % 3];
    if (!(opts->flags & LRC_SKIP_FINAL_RESIDUAL)) {
      // residual factors: Ucat = [B_U | W0 | W1 | W2], Vcat = [B_V | -V | -d_mu V | -d_nu V]
      SpmmArgs a = spmm_base(ctx);
      a.U = UN; a.ldu = w.LDU; a.d_r = sd.rk + slotN; a.out = w.W3; a.ldo = w.LDU; a.out_off = 0;
      a.out_sstride = (long long)M * w.LDU;
      KL(P_SPMM, s, launch_spmm(SPMM_PLAIN3, a, cap, s));
      const UDesc ur = ucat_desc(w, M, rb, slotN, nullptr, -1, ctx->G);
      VDesc vr{};
      vr.nb = 0;
      vr.pad_even = 1;
      vr.b[vr.nb++] = vblock(w.BV, rb, rb, -1, 1.0, -1, 0);
      for (int g = 0; g < ctx->G; ++g)
        vr.b[vr.nb++] = vblock(VN, cap, 0, slotN, -1.0, g == ctx->id_group ? -1 : g, 0);
      lrc_status st = enqueue_norm2(ctx, ur, vr, 1, s);
      if (st != LRC_OK) return st;
    }
    // outputs: DEVICE outputs by a guarded copy kernel (columns >= rank zeroed; nothing is written
    // when the device flags an error, so the outputs stay untouched on LRC_ERR_NUMERIC); HOST
    // outputs are copied in finish_solve after the flags were checked
    if (where == LRC_MEM_DEVICE) {
      KL(P_MISC, s, launch_copy_out(UN, w.LDU, sc.U_out, (int)sc.ld_u, (int)M, cap, sd.rk + slotN, sd.flags, s));
      KL(P_MISC, s, launch_copy_out(VN, cap, sc.V_out, (int)sc.ld_v, (int)n, cap, sd.rk + slotN, sd.flags, s));
    } else {
      KL(P_MISC, s, launch_zero_cols(UN, (int)M, w.LDU, sd.rk + slotN, 0, cap, s));
      KL(P_MISC, s, launch_zero_cols(VN, (int)n, cap, sd.rk + slotN, 0, cap, s));
    }
  } else if (where == LRC_MEM_HOST) {
    for (int64_t i = 0; i < M; ++i) std::memset(sc.U_out + i * sc.ld_u, 0, sizeof(double) * cap);
    for (int64_t i = 0; i < n; ++i) std::memset(sc.V_out + i * sc.ld_v, 0, sizeof(double) * cap);
  } else {
    CK(cudaMemset2DAsync(sc.U_out, sizeof(double) * sc.ld_u, 0, sizeof(double) * cap, M, s));
    CK(cudaMemset2DAsync(sc.V_out, sizeof(double) * sc.ld_v, 0, sizeof(double) * cap, n, s));
  }
  CK(cudaEventRecord(ctx->ev[3], s));
  // results -> pinned host mirrors (read by finish_solve after the stream synchronises)
  CK(ensure_pinned(ctx, w.N));
  CK(cudaMemcpyAsync(ctx->h_ints, w.ints, sizeof(int) * (w.N + 16), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ctx->h_scal, w.scal, sizeof(double) * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ctx->h_sigma, w.sigma, sizeof(double) * (size_t)N * kSigmaStride, cudaMemcpyDeviceToHost, s));
  Pending& pd = ctx->pending;
  pd.active = true;
  pd.N = N; pd.rb = rb; pd.cap = cap; pd.M = M; pd.n = n; pd.opt_flags = opts->flags; pd.record = sc.record;
  pd.where = where; pd.U_out = sc.U_out; pd.V_out = sc.V_out; pd.ld_u = sc.ld_u; pd.ld_v = sc.ld_v;
  pd.UN = w.Ubuf[(N + 1) % 3]; pd.VN = w.Vbuf[(N + 1) % 3];
  return LRC_OK;
}

// capture (or reuse) a graph of `body` on stream s; body() enqueues the work, ctx counts its kernels
template <typename F>
lrc_status run_graph(lrc_ctx* ctx, cudaStream_t s, cudaGraphExec_t& gexec, bool reuse, int64_t& gkernels, F&& body) {
  if (!reuse) {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    ctx->capturing = true;
    ctx->capture_count = 0;
    lrc_status es = body();
    ctx->capturing = false;
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (es != LRC_OK) { if (g) cudaGraphDestroy(g); return es; }
    if (ce != cudaSuccess) return fail(ctx, LRC_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&gexec, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) { gexec = nullptr; return fail(ctx, LRC_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce)); }
    gkernels = ctx->capture_count;
  }
  CK(cudaGraphLaunch(gexec, s));
  ctx->launches += gkernels;
  return LRC_OK;
}

}  // namespace

extern "C" {

lrc_status lrc_solve(lrc_ctx* ctx, const double* B_U, int64_t ld_bu, const double* B_V, int64_t ld_bv,
                     int64_t r_B, const lrc_solve_opts* opts, double* U_out, int64_t ld_u,
                     double* V_out, int64_t ld_v, lrc_mem where, lrc_solve_info* info) {
  if (!ctx) return LRC_ERR_ARG;
  SolveCall sc;
  lrc_status st = solve_validate(ctx, B_U, ld_bu, B_V, ld_bv, r_B, opts, U_out, ld_u, V_out, ld_v, where, sc);
  if (st != LRC_OK) return st;
  st = solve_prologue(ctx, opts, where, sc);
  if (st != LRC_OK) return st;
  cudaStream_t s = ctx->stream;
  if (sc.rb > 0) {
    const bool use_graph = (opts->flags & LRC_NO_GRAPH) == 0 && !ctx->profiling;
    GraphKey key;
    key.gen = ctx->gen; key.N = sc.N; key.rb = sc.rb; key.cap = sc.cap; key.gamma = sc.gamma; key.tol = opts->tol;
    key.flags = opts->flags & (LRC_RECORD_ITERATES | LRC_NO_WARM_START | LRC_PRECONDITIONED);
    key.pc_gen = ctx->pc_active ? ctx->pc_gen : 0;
    auto body = [&]() -> lrc_status {
      for (int k = 0; k < sc.N; ++k) {
        lrc_status e = enqueue_iteration(ctx, k, sc.rb, sc.cap, sc.gamma, opts->tol, sc.record);
        if (e != LRC_OK) return e;
      }
      return LRC_OK;
    };
    if (use_graph) {
      const bool reuse = ctx->gexec && ctx->gkey == key;
      st = run_graph(ctx, s, ctx->gexec, reuse, ctx->graph_kernels, body);
      if (st != LRC_OK) { drop_graph(ctx); return st; }
      ctx->gkey = key;
    } else {
      st = body();
      if (st != LRC_OK) return st;
    }
  }
  st = solve_epilogue(ctx, opts, where, sc);
  if (st != LRC_OK) return st;
  if (opts->flags & LRC_ASYNC) return LRC_OK;     // lrc_solve_wait completes the call
  return finish_solve(ctx, info);
}

// Batched lockstep solve of S subsets sharing one operator (Algorithm 1's loop
// over the subsets): per iteration one batched fused SpMM on ctxs[0]'s stream reads the
// operator once for all S U factors, then every subset's truncation runs on its own context's
// stream (V-side assembly forked to the side streams, overlapping the SpMM).  Captured once into a
// CUDA graph over the S streams.
lrc_status lrc_solve_batch(lrc_ctx* const* ctxs, int S, const double* const* B_U, const int64_t* ld_bu,
                           const double* const* B_V, const int64_t* ld_bv, int64_t r_B,
                           const lrc_solve_opts* opts, double* const* U_out, const int64_t* ld_u,
                           double* const* V_out, const int64_t* ld_v, lrc_mem where, lrc_solve_info* infos) {
  if (!ctxs || S < 1 || S > kMaxSub || !ctxs[0] || !B_U || !B_V || !ld_bu || !ld_bv || !U_out || !V_out || !ld_u || !ld_v)
    return LRC_ERR_ARG;
  lrc_ctx* c0 = ctxs[0];
  lrc_ctx* const ctx = c0;   // errors are reported on the first context
  if (!opts) return fail(c0, LRC_ERR_ARG, "null opts");
  if (opts->flags & (LRC_ASYNC | LRC_NO_GRAPH | LRC_RECORD_ITERATES | LRC_PRECONDITIONED))
    return fail(c0, LRC_ERR_ARG, "lrc_solve_batch: LRC_ASYNC / LRC_NO_GRAPH / LRC_RECORD_ITERATES / "
                                 "LRC_PRECONDITIONED not supported");
  if (r_B < 1) return fail(c0, LRC_ERR_ARG, "lrc_solve_batch: r_B must be >= 1");
  for (int q = 0; q < S; ++q) {
    lrc_ctx* c = ctxs[q];
    if (!c) return fail(c0, LRC_ERR_ARG, "null context");
    for (int p = 0; p < q; ++p) if (ctxs[p] == c) return fail(c0, LRC_ERR_ARG, "contexts must be distinct");
    if (!c->op_set || !c0->op_set) return fail(c0, LRC_ERR_STATE, "lrc_solve_batch before lrc_set_operator");
    bool same = c->device == c0->device && c->M == c0->M && c->nnz == c0->nnz && c->row_ptr == c0->row_ptr &&
                c->col_idx == c0->col_idx && c->rho == c0->rho && c->lam == c0->lam;
    for (int t = 0; t < kMaxT; ++t) same = same && c->vals[t] == c0->vals[t];
    same = same && c->general == c0->general && c->T == c0->T && c->G == c0->G;
    if (!same) return fail(c0, LRC_ERR_ARG, "lrc_solve_batch: contexts must borrow the same operator arrays");
  }
  std::vector<SolveCall> sc(S);
  for (int q = 0; q < S; ++q) {
    lrc_status st = solve_validate(ctxs[q], B_U[q], ld_bu[q], B_V[q], ld_bv[q], r_B, opts, U_out[q], ld_u[q],
                                   V_out[q], ld_v[q], where, sc[q]);
    if (st != LRC_OK) return st;
  }
  for (int q = 0; q < S; ++q) {
    lrc_status st = solve_prologue(ctxs[q], opts, where, sc[q]);
    if (st != LRC_OK) return st;
  }
  const int N = sc[0].N, rb = sc[0].rb, cap = sc[0].cap;
  const double gamma = sc[0].gamma, tol = opts->tol;
  cudaStream_t s0 = c0->stream;
  // the capture stream waits for every subset's prologue
  for (int q = 1; q < S; ++q) {
    CK(cudaEventRecord(ctxs[q]->ev_join, ctxs[q]->stream));
    CK(cudaStreamWaitEvent(s0, ctxs[q]->ev_join, 0));
  }
  auto body = [&]() -> lrc_status {
    for (int q = 1; q < S; ++q) {                        // bring the subset streams into the capture
      CK(cudaEventRecord(c0->ev_fork, s0));
      CK(cudaStreamWaitEvent(ctxs[q]->stream, c0->ev_fork, 0));
    }
    for (int k = 0; k < N; ++k) {
      // U_k / V_k of every subset final: record each subset's fork point, join into the SpMM stream
      for (int q = 0; q < S; ++q) {
        CK(cudaEventRecord(ctxs[q]->ev_fork, ctxs[q]->stream));
        if (q > 0) CK(cudaStreamWaitEvent(s0, ctxs[q]->ev_fork, 0));
      }
      SpmmArgs a = iteration_spmm_args(c0, k, gamma);
      a.nsub = S;
      for (int q = 0; q < S; ++q) {
        const SpmmArgs aq = iteration_spmm_args(ctxs[q], k, gamma);
        a.Us[q] = aq.U; a.outs[q] = aq.out; a.d_rs[q] = aq.d_r;
      }
      KL(P_SPMM, s0, launch_spmm(SPMM_S2STEP, a, cap, s0));
      CK(cudaEventRecord(c0->ev_k1, s0));
      for (int q = 0; q < S; ++q) {
        if (q > 0) CK(cudaStreamWaitEvent(ctxs[q]->stream, c0->ev_k1, 0));
        lrc_status e = enqueue_iteration_trunc(ctxs[q], k, rb, cap, gamma, tol, false);
        if (e != LRC_OK) return e;
      }
    }
    for (int q = 1; q < S; ++q) {                        // join the subset streams
      CK(cudaEventRecord(ctxs[q]->ev_join, ctxs[q]->stream));
      CK(cudaStreamWaitEvent(s0, ctxs[q]->ev_join, 0));
    }
    return LRC_OK;
  };
  // graph cache (on ctxs[0]): the contexts, their generations and the solve shape
  std::vector<int64_t> key;
  key.push_back(S); key.push_back(N); key.push_back(rb); key.push_back(cap);
  key.push_back((int64_t)(opts->flags & LRC_NO_WARM_START));
  int64_t gb, tb;
  std::memcpy(&gb, &gamma, 8); std::memcpy(&tb, &tol, 8);
  key.push_back(gb); key.push_back(tb);
  for (int q = 0; q < S; ++q) { key.push_back((int64_t)(uintptr_t)ctxs[q]); key.push_back(ctxs[q]->gen); }
  const bool reuse = c0->bgexec && c0->bkey == key;
  lrc_status st = run_graph(c0, s0, c0->bgexec, reuse, c0->bgraph_kernels, body);
  if (st != LRC_OK) { if (c0->bgexec) cudaGraphExecDestroy(c0->bgexec); c0->bgexec = nullptr; c0->bkey.clear(); return st; }
  c0->bkey = key;
  // every subset stream waits for the batched iterations, then runs its own epilogue
  CK(cudaEventRecord(c0->ev_join, s0));
  for (int q = 1; q < S; ++q) CK(cudaStreamWaitEvent(ctxs[q]->stream, c0->ev_join, 0));
  for (int q = 0; q < S; ++q) {
    st = solve_epilogue(ctxs[q], opts, where, sc[q]);
    if (st != LRC_OK) return st;
  }
  lrc_status worst = LRC_OK;
  for (int q = 0; q < S; ++q) {
    st = finish_solve(ctxs[q], infos ? infos + q : nullptr);
    if (st != LRC_OK && worst == LRC_OK) worst = st;
  }
  return worst;
}

// Wait for the solve enqueued last on ctx, fill info, copy HOST outputs (only when no error was
// flagged on the device) and return the call's status.
lrc_status lrc_solve_wait(lrc_ctx* ctx, lrc_solve_info* info) {
  if (!ctx) return LRC_ERR_ARG;
  if (!ctx->pending.active) return fail(ctx, LRC_ERR_STATE, "no solve pending on this context");
  CK(cudaSetDevice(ctx->device));
  return finish_solve(ctx, info);
}

lrc_status lrc_apply_lowrank(lrc_ctx* ctx, const double* U, int64_t ld_u, int64_t r, double* W,
                             int64_t ld_w, uint32_t mode, double gamma, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set) return fail(ctx, LRC_ERR_STATE, "lrc_apply_lowrank before lrc_set_operator");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  if (r < 1 || r > kMaxRank) return fail(ctx, LRC_ERR_ARG, "r must be in [1, 128]");
  if (!U || !W) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (mode > LRC_APPLY_S2STEP) return fail(ctx, LRC_ERR_ARG, "bad mode");
  const int nout = (mode == LRC_APPLY_SIX) ? ctx->T : ctx->G;   // per array / per right-diagonal group
  if (ld_u < r || ld_w < nout * r) return fail(ctx, LRC_ERR_SHAPE, "leading dimension too small");
  if (ctx->general && mode != LRC_APPLY_SIX && (r > 64 || (where == LRC_MEM_DEVICE && ((ld_u & 1) || (reinterpret_cast<uintptr_t>(U) & 15)))))
    return fail(ctx, LRC_ERR_ARG, "general term lists: r <= 64 and 16-byte aligned U rows (even ld)");
  CK(cudaSetDevice(ctx->device));
  const int64_t M = ctx->M;
  cudaStream_t s = ctx->stream;
  const double* Ud = U;
  double* Wd = W;
  int ldu = (int)ld_u, ldw = (int)ld_w;
  if (where == LRC_MEM_HOST) {
    const int lde = (int)(r + (r & 1));            // even: 16-byte rows for the TMA path
    lrc_status st = ensure_tmp(ctx, &ctx->tmpA, &ctx->tmpA_sz, (size_t)M * lde);
    if (st != LRC_OK) return st;
    st = ensure_tmp(ctx, &ctx->tmpB, &ctx->tmpB_sz, (size_t)M * nout * r);
    if (st != LRC_OK) return st;
    CK(cudaMemcpy2DAsync(ctx->tmpA, sizeof(double) * lde, U, sizeof(double) * ld_u, sizeof(double) * r, M, cudaMemcpyHostToDevice, s));
    Ud = ctx->tmpA; ldu = lde;
    Wd = ctx->tmpB; ldw = nout * (int)r;
  }
  SpmmArgs a = spmm_base(ctx);
  a.U = Ud; a.ldu = ldu; a.d_r = nullptr; a.r_fixed = (int)r; a.out = Wd; a.ldo = ldw; a.out_off = 0;
  a.gamma = gamma;
  CK(cudaEventRecord(ctx->ev[0], s));
  if (mode == LRC_APPLY_SIX) {
    for (int t = 0; t < ctx->T; ++t) {
      a.single_t = t;
      a.out_off = t * (int)r;
      KL(P_SPMM, s, launch_spmm(SPMM_SINGLE, a, (int)r, s));
    }
  } else {
    KL(P_SPMM, s, launch_spmm(mode == LRC_APPLY_S2STEP ? SPMM_S2STEP : SPMM_PLAIN3, a, (int)r, s));
  }
  CK(cudaEventRecord(ctx->ev[1], s));
  if (where == LRC_MEM_HOST)
    CK(cudaMemcpy2DAsync(W, sizeof(double) * ld_w, Wd, sizeof(double) * ldw, sizeof(double) * nout * r, M, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  prof_collect(ctx);
  cudaEventElapsedTime(&ctx->last_kernel_ms, ctx->ev[0], ctx->ev[1]);
  return LRC_OK;
}

lrc_status lrc_apply_dense(lrc_ctx* ctx, const double* S, int64_t ld_s, int64_t ncols, double* Y,
                           int64_t ld_y, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_apply_dense before set_operator + set_params");
  if (ctx->general) return fail(ctx, LRC_ERR_STATE, "lrc_apply_dense: the operator of P:30-36 only");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  if (ncols != ctx->n) return fail(ctx, LRC_ERR_SHAPE, "ncols must equal n of lrc_set_params");
  if (ncols < 1 || ncols > 256) return fail(ctx, LRC_ERR_ARG, "ncols must be in [1, 256]");
  if (!S || !Y) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (ld_s < ncols || ld_y < ncols) return fail(ctx, LRC_ERR_SHAPE, "leading dimension too small");
  CK(cudaSetDevice(ctx->device));
  const int64_t M = ctx->M;
  cudaStream_t s = ctx->stream;
  const double* Sd = S;
  double* Yd = Y;
  int lds = (int)ld_s, ldy = (int)ld_y;
  if (where == LRC_MEM_HOST) {
    lrc_status st = ensure_tmp(ctx, &ctx->tmpA, &ctx->tmpA_sz, (size_t)M * ncols);
    if (st != LRC_OK) return st;
    st = ensure_tmp(ctx, &ctx->tmpB, &ctx->tmpB_sz, (size_t)M * ncols);
    if (st != LRC_OK) return st;
    CK(cudaMemcpy2DAsync(ctx->tmpA, sizeof(double) * ncols, S, sizeof(double) * ld_s, sizeof(double) * ncols, M, cudaMemcpyHostToDevice, s));
    Sd = ctx->tmpA; lds = (int)ncols;
    Yd = ctx->tmpB; ldy = (int)ncols;
  }
  SpmmArgs a = spmm_base(ctx);
  a.U = Sd; a.ldu = lds; a.d_r = nullptr; a.r_fixed = (int)ncols; a.out = Yd; a.ldo = ldy;
  a.dmu = ctx->dmu; a.dnu = ctx->dnu;
  CK(cudaEventRecord(ctx->ev[0], s));
  KL(P_SPMM, s, launch_spmm(SPMM_DENSE, a, (int)ncols, s));
  CK(cudaEventRecord(ctx->ev[1], s));
  if (where == LRC_MEM_HOST)
    CK(cudaMemcpy2DAsync(Y, sizeof(double) * ld_y, Yd, sizeof(double) * ldy, sizeof(double) * ncols, M, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  prof_collect(ctx);
  cudaEventElapsedTime(&ctx->last_kernel_ms, ctx->ev[0], ctx->ev[1]);
  return LRC_OK;
}

lrc_status lrc_truncate(lrc_ctx* ctx, const double* U, int64_t ld_u, const double* V, int64_t ld_v,
                        int64_t wdt, double tol, int64_t cap, double* U_out, double* V_out,
                        int64_t* rank, double* sigma, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_truncate before set_operator + set_params");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  if (wdt < 1 || wdt > kMaxW) return fail(ctx, LRC_ERR_ARG, "w must be in [1, 256]");
  if (cap < 1 || cap > std::min<int64_t>(kMaxRank, std::min(ctx->M, ctx->n))) return fail(ctx, LRC_ERR_ARG, "cap must be in [1, min(M, n, 128)]");
  if (!(tol >= 0.0)) return fail(ctx, LRC_ERR_ARG, "tol must be >= 0");
  if (!U || !V || !U_out || !V_out || !rank) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (ld_u < wdt || ld_v < wdt) return fail(ctx, LRC_ERR_SHAPE, "leading dimension too small");
  const int64_t M = ctx->M, n = ctx->n;
  const int w = (int)wdt, capi = (int)cap;
  const int p_need = (int)std::min<int64_t>(n, w);
  if (p_need > 112) return fail(ctx, LRC_ERR_ARG, "min(n, w) must be <= 112 in this build");
  if (lrc::vside_smem_bytes((int)n, w, ts_pmax_for(p_need)) > kSmemLimit)
    return fail(ctx, LRC_ERR_ARG, "n x w too large for the single-CTA V-side QR");
  CK(cudaSetDevice(ctx->device));
  // a workspace for this call's width (an existing one is reused when it is compatible)
  lrc_status st = ensure_ws_fit(ctx, std::max(ctx->ws.rb, 1), capi, std::max(ctx->ws.N, 1), w, false);
  if (st != LRC_OK) return st;
  Workspace& ws = ctx->ws;
  cudaStream_t s = ctx->stream;
  // inputs
  st = ensure_tmp(ctx, &ctx->tmpA, &ctx->tmpA_sz, (size_t)M * w);
  if (st != LRC_OK) return st;
  st = ensure_tmp(ctx, &ctx->tmpB, &ctx->tmpB_sz, (size_t)n * w + (size_t)n * capi);
  if (st != LRC_OK) return st;
  st = ensure_tmp(ctx, &ctx->tmpC, &ctx->tmpC_sz, (size_t)M * capi);
  if (st != LRC_OK) return st;
  CK(cudaMemcpy2DAsync(ctx->tmpA, sizeof(double) * w, U, sizeof(double) * ld_u, sizeof(double) * w, M, kind_in(where), s));
  CK(cudaMemcpy2DAsync(ctx->tmpB, sizeof(double) * w, V, sizeof(double) * ld_v, sizeof(double) * w, n, kind_in(where), s));
  State sd = make_state(ws);
  const int slot = ws.N + 2;
  CK(cudaMemsetAsync(ws.ints, 0, sizeof(int) * (ws.N + 16), s));
  CK(cudaMemsetAsync(ws.sigma, 0, sizeof(double) * (size_t)(ws.N + 4) * kSigmaStride, s));
  UDesc ud{};
  ud.nb = 1;
  ud.b[0] = ublock(ctx->tmpA, w, w, -1);
  VDesc vd{};
  vd.nb = 1;
  vd.b[0] = vblock(ctx->tmpB, w, w, -1, 1.0, -1, 0);
  double* Vnew = ctx->tmpB + (size_t)n * w;
  st = enqueue_truncation(ctx, ud, vd, nullptr, 0, tol, capi, slot, ws.N, ctx->tmpC, capi, Vnew, capi, s, false);
  if (st != LRC_OK) return st;
  KL(P_MISC, s, launch_zero_cols(ctx->tmpC, (int)M, capi, sd.rk + slot, 0, capi, s));
  int hr = 0, flags = 0;
  CK(cudaMemcpyAsync(&hr, sd.rk + slot, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&flags, sd.flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  std::vector<double> sg(kSigmaStride);
  CK(cudaMemcpyAsync(sg.data(), ws.sigma + (size_t)ws.N * kSigmaStride, sizeof(double) * kSigmaStride, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  prof_collect(ctx);
  ctx->last_record = false;   // tmp state overwrote the iterate bookkeeping slots
  if (flags & 1) return fail(ctx, LRC_ERR_NUMERIC, "shifted Cholesky failed after all escalations");
  if (flags & 2) return fail(ctx, LRC_ERR_NUMERIC, "non-finite singular value in the core SVD");
  CK(cudaMemcpyAsync(U_out, ctx->tmpC, sizeof(double) * M * capi, kind_out(where), s));   // outputs only on success
  CK(cudaMemcpyAsync(V_out, Vnew, sizeof(double) * n * capi, kind_out(where), s));
  CK(cudaStreamSynchronize(s));
  *rank = hr;
  if (sigma) std::memcpy(sigma, sg.data(), sizeof(double) * p_need);
  return LRC_OK;
}

lrc_status lrc_get_iterate(lrc_ctx* ctx, int64_t k, double* U, double* V, int64_t* rank, lrc_mem where) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->last_record || !ctx->ws.Uh) return fail(ctx, LRC_ERR_STATE, "no recorded iterates (solve with LRC_RECORD_ITERATES)");
  if (k < 1 || k > ctx->last_N) return fail(ctx, LRC_ERR_ARG, "k must be in [1, n_iter]");
  if (!U || !V || !rank) return fail(ctx, LRC_ERR_ARG, "null pointer");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  CK(cudaSetDevice(ctx->device));
  Workspace& w = ctx->ws;
  cudaStream_t s = ctx->stream;
  const int cap = ctx->last_cap;
  const size_t M = (size_t)ctx->M, n = (size_t)ctx->n;
  int hr = 0;
  CK(cudaMemcpyAsync(&hr, w.ints + (k + 1), sizeof(int), cudaMemcpyDeviceToHost, s));
  double* Uk = w.Uh + (size_t)(k - 1) * M * w.LDU;
  KL(P_MISC, s, launch_zero_cols(Uk, (int)M, w.LDU, w.ints + (k + 1), 0, cap, s));
  const double* Vk = w.Vh + (size_t)(k - 1) * n * cap;
  CK(cudaMemcpy2DAsync(U, sizeof(double) * cap, Uk, sizeof(double) * w.LDU, sizeof(double) * cap, M, kind_out(where), s));
  CK(cudaMemcpyAsync(V, Vk, sizeof(double) * n * cap, kind_out(where), s));
  CK(cudaStreamSynchronize(s));
  *rank = hr;
  return LRC_OK;
}

}  // extern "C"

// =============================================================================================
// GMREST -- truncated restarted GMRES (restarted
// once after 6 iterations P:546; reading R14).  The same building blocks as ChebyshevT: the
// fused SpMM (PLAIN mode), the truncation operator T of P:544 (V-side QR, CholeskyQR2 + Jacobi), the
// honest residual; plus Frobenius inner products of low-rank matrices, <U1 V1^T, U2 V2^T> =
// tr((U1^T U2)(V2^T V1)), whose M-level part U1^T U2 is a Gram pass over [U1 | U2] with T = I.
// Host-driven: the Arnoldi coefficients decide the next linear combination, so each step reads a few
// scalars back (no graph).
// =============================================================================================
namespace {

struct LR {                 // a low-rank matrix s * U V^T held in device buffers, rank in st.rk[slot]
  double* U; double* V; int slot; double scale; int rank;
};

lrc_status gm_rank_sigma(lrc_ctx* ctx, int slot, int sigma_row, int& rank, double& fro) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  int r = 0;
  double sg[kSigmaStride];
  CK(cudaMemcpyAsync(&r, st.rk + slot, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(sg, st.sigma + (size_t)sigma_row * kSigmaStride, sizeof(sg), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double f = 0.0;
  for (int i = 0; i < r; ++i) f += sg[i] * sg[i];
  rank = r;
  fro = std::sqrt(f);
  return LRC_OK;
}

// out = T_{tau,cap}(sum_b scale_b * U_b V_b^T) over the given low-rank terms; out.scale = 1
lrc_status gm_truncate(lrc_ctx* ctx, const std::vector<LR>& terms, double tau, int cap, LR& out, int sigma_row,
                       double& fro) {
  Workspace& w = ctx->ws;
  UDesc ud{};
  VDesc vd{};
  ud.pad_even = 1; vd.pad_even = 1;
  for (const LR& t : terms) {
    ud.b[ud.nb++] = ublock(t.U, w.LDU, 0, t.slot);
    vd.b[vd.nb++] = vblock(t.V, cap, 0, t.slot, t.scale, -1, 0);
  }
  lrc_status st = enqueue_truncation(ctx, ud, vd, nullptr, 0, tau, cap, out.slot, sigma_row, out.U, w.LDU, out.V, cap,
                                     ctx->stream, false);
  if (st != LRC_OK) return st;
  out.scale = 1.0;
  return gm_rank_sigma(ctx, out.slot, sigma_row, out.rank, fro);
}

// out = T(L(x)) (x.scale folded into the V side), through the grouped fused SpMM
lrc_status gm_apply(lrc_ctx* ctx, const LR& x, double tau, int cap, LR& out, int sigma_row, double& fro) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  cudaStream_t s = ctx->stream;
  SpmmArgs a = spmm_base(ctx);
  a.U = x.U; a.ldu = w.LDU; a.d_r = st.rk + x.slot; a.out = w.W3; a.ldo = w.LDU; a.out_off = 0;
  a.out_sstride = (long long)ctx->M * w.LDU;
  KL(P_SPMM, s, launch_spmm(SPMM_PLAIN3, a, cap, s));
  UDesc ud{};
  VDesc vd{};
  ud.pad_even = 1; vd.pad_even = 1;
  for (int g = 0; g < ctx->G; ++g) {
    ud.b[ud.nb++] = ublock(w.W3 + (size_t)g * ctx->M * w.LDU, w.LDU, 0, x.slot);
    vd.b[vd.nb++] = vblock(x.V, cap, 0, x.slot, x.scale, g == ctx->id_group ? -1 : g, 0);
  }
  lrc_status r = enqueue_truncation(ctx, ud, vd, nullptr, 0, tau, cap, out.slot, sigma_row, out.U, w.LDU, out.V, cap,
                                    s, false);
  if (r != LRC_OK) return r;
  out.scale = 1.0;
  return gm_rank_sigma(ctx, out.slot, sigma_row, out.rank, fro);
}

// <a, b>_F of two low-rank matrices (ranks known on the host)
lrc_status gm_inner(lrc_ctx* ctx, const LR& a, const LR& b, int cap, double& out) {
  out = 0.0;
  if (a.rank == 0 || b.rank == 0) return LRC_OK;
  Workspace& w = ctx->ws;
  State st = make_state(w);
  cudaStream_t s = ctx->stream;
  const int ra = a.rank + (a.rank & 1), rbk = b.rank + (b.rank & 1);
  const int wdt = ra + rbk, pmax = ts_pmax_for(wdt);
  TsArgs ta{};
  ta.M = (int)ctx->M;
  ta.u.nb = 2; ta.u.pad_even = 1;
  ta.u.b[0] = ublock(a.U, w.LDU, 0, a.slot);
  ta.u.b[1] = ublock(b.U, w.LDU, 0, b.slot);
  ta.rk = st.rk;
  ta.T = ctx->gmI; ta.ldt = kMaxP;        // identity: X = [U_a | U_b], G = X^T X
  ta.d_p = nullptr; ta.p_fixed = wdt;
  ta.partials = ctx->gmP;
  KL(P_TS_GRAM, s, launch_ts(0, ta, pmax, w.grid, s));
  KL(P_REDUCE, s, launch_gram_reduce(ctx->gmP, w.grid, pmax, ctx->gmG, s));
  std::vector<double> G((size_t)pmax * pmax), Va((size_t)ctx->n * cap), Vb((size_t)ctx->n * cap);
  CK(cudaMemcpyAsync(G.data(), ctx->gmG, sizeof(double) * G.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(Va.data(), a.V, sizeof(double) * Va.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(Vb.data(), b.V, sizeof(double) * Vb.size(), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // tr((U_a^T U_b)(V_b^T V_a)) = sum_{i,j} (U_a^T U_b)[i][j] (V_a^T V_b)[i][j]
  double acc = 0.0;
  for (int i = 0; i < a.rank; ++i)
    for (int j = 0; j < b.rank; ++j) {
      double vv = 0.0;
      for (int64_t q = 0; q < ctx->n; ++q) vv += Va[(size_t)q * cap + i] * Vb[(size_t)q * cap + j];
      acc += G[(size_t)i * pmax + ra + j] * vv;
    }
  out = acc * a.scale * b.scale;
  return LRC_OK;
}

// y = argmin || beta e1 - H y ||  (H (k+1) x k upper Hessenberg, row-major ld m) by Givens rotations
void gm_lsq(const std::vector<double>& Hin, int m, int k, double beta, std::vector<double>& y) {
  std::vector<double> H(Hin), g(k + 1, 0.0);
  g[0] = beta;
  for (int j = 0; j < k; ++j) {
    const double a = H[(size_t)j * m + j], b = H[(size_t)(j + 1) * m + j];
    const double r = std::hypot(a, b);
    const double c = r > 0 ? a / r : 1.0, sn = r > 0 ? b / r : 0.0;
    for (int q = j; q < k; ++q) {
      const double x = H[(size_t)j * m + q], z = H[(size_t)(j + 1) * m + q];
      H[(size_t)j * m + q] = c * x + sn * z;
      H[(size_t)(j + 1) * m + q] = -sn * x + c * z;
    }
    const double gx = g[j], gz = g[j + 1];
    g[j] = c * gx + sn * gz;
    g[j + 1] = -sn * gx + c * gz;
  }
  y.assign(k, 0.0);
  for (int j = k - 1; j >= 0; --j) {
    double acc = g[j];
    for (int q = j + 1; q < k; ++q) acc -= H[(size_t)j * m + q] * y[q];
    const double d = H[(size_t)j * m + j];
    y[j] = d != 0.0 ? acc / d : 0.0;
  }
}

// honest ||B - L(X)||_F^2 -> scal[1] (as the solve epilogue)
lrc_status gm_residual2(lrc_ctx* ctx, const LR& x, int rb, int cap, double& r2) {
  Workspace& w = ctx->ws;
  State st = make_state(w);
  cudaStream_t s = ctx->stream;
  UDesc ud{};
  VDesc vd{};
  ud.pad_even = 1; vd.pad_even = 1;
  ud.b[ud.nb++] = ublock(w.BUb, w.LDB, rb, -1);
  vd.b[vd.nb++] = vblock(w.BV, rb, rb, -1, 1.0, -1, 0);
  if (x.rank > 0) {
    SpmmArgs a = spmm_base(ctx);
    a.U = x.U; a.ldu = w.LDU; a.d_r = st.rk + x.slot; a.out = w.W3; a.ldo = w.LDU; a.out_off = 0;
    a.out_sstride = (long long)ctx->M * w.LDU;
    KL(P_SPMM, s, launch_spmm(SPMM_PLAIN3, a, cap, s));
    for (int g = 0; g < ctx->G; ++g) {
      ud.b[ud.nb++] = ublock(w.W3 + (size_t)g * ctx->M * w.LDU, w.LDU, 0, x.slot);
      vd.b[vd.nb++] = vblock(x.V, cap, 0, x.slot, -x.scale, g == ctx->id_group ? -1 : g, 0);
    }
  }
  lrc_status r = enqueue_norm2(ctx, ud, vd, 1, s);
  if (r != LRC_OK) return r;
  double sc[8];
  CK(cudaMemcpyAsync(sc, w.scal, sizeof(sc), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  r2 = sc[1];
  return LRC_OK;
}

}  // namespace

extern "C" {

lrc_status lrc_solve_gmres(lrc_ctx* ctx, const double* B_U, int64_t ld_bu, const double* B_V, int64_t ld_bv,
                           int64_t r_B, const lrc_gmres_opts* opts, double* U_out, int64_t ld_u, double* V_out,
                           int64_t ld_v, lrc_mem where, lrc_gmres_info* info) {
  if (!ctx) return LRC_ERR_ARG;
  ctx->err.clear();
  if (!ctx->op_set || !ctx->par_set) return fail(ctx, LRC_ERR_STATE, "lrc_solve_gmres before set_operator + params");
  if (!opts) return fail(ctx, LRC_ERR_ARG, "null opts");
  if (!valid_mem(where)) return fail(ctx, LRC_ERR_ARG, "bad lrc_mem");
  const int64_t M = ctx->M, n = ctx->n;
  const int cap = (int)opts->rank_cap, m = (int)opts->restart, maxc = (int)opts->max_cycles;
  if (cap < 1 || cap > std::min<int64_t>(std::min(M, n), 64)) return fail(ctx, LRC_ERR_ARG, "rank_cap must be in [1, min(M, n, 64)]");
  if (m < 1 || m > 32 || maxc < 1 || maxc > 1000) return fail(ctx, LRC_ERR_ARG, "restart in [1, 32], max_cycles in [1, 1000]");
  if (!(opts->trunc_tol >= 0.0) || !(opts->tol >= 0.0)) return fail(ctx, LRC_ERR_ARG, "tolerances must be >= 0");
  if (r_B < 1 || r_B > 64 || !B_U || !B_V || ld_bu < r_B || ld_bv < r_B) return fail(ctx, LRC_ERR_ARG, "bad B factors");
  if (!U_out || !V_out || ld_u < cap || ld_v < cap) return fail(ctx, LRC_ERR_ARG, "bad outputs");
  const int rb = (int)r_B;
  const int wmax = std::max((rb + (rb & 1)) + ctx->G * (cap + (cap & 1)), (ctx->G) * (cap + (cap & 1)));
  if (wmax > kMaxW || std::min<int64_t>(n, wmax) > 112) return fail(ctx, LRC_ERR_ARG, "r_B + G rank_cap too wide");
  if (ctx->pending.active) {
    lrc_status ps = finish_solve(ctx, nullptr);
    if (ps != LRC_OK) return ps;
  }
  CK(cudaSetDevice(ctx->device));
  // slots: 0 X, 1 W, 2 T (scratch), 3 .. 3 + m: the Krylov basis; sigma rows likewise
  lrc_status st = ensure_ws_fit(ctx, rb, cap, m + 8, wmax, false);
  if (st != LRC_OK) return st;
  Workspace& w = ctx->ws;
  cudaStream_t s = ctx->stream;
  const size_t need = (size_t)(m + 1);
  if (ctx->gm_cap < need || !ctx->gmU) {
    dfree(ctx->gmU); dfree(ctx->gmV);
    ctx->gmU = ctx->gmV = nullptr; ctx->gm_cap = 0;
    CK(dalloc(&ctx->gmU, need * M * w.LDU));
    CK(dalloc(&ctx->gmV, need * n * cap));
    ctx->gm_cap = need;
  }
  if (!ctx->gmI) {
    std::vector<double> I((size_t)kMaxP * kMaxP, 0.0);
    for (int i = 0; i < kMaxP; ++i) I[(size_t)i * kMaxP + i] = 1.0;
    CK(dalloc(&ctx->gmI, I.size()));
    CK(cudaMemcpy(ctx->gmI, I.data(), sizeof(double) * I.size(), cudaMemcpyHostToDevice));
    CK(dalloc(&ctx->gmP, (size_t)148 * kMaxP * kMaxP));
    CK(dalloc(&ctx->gmG, (size_t)kMaxP * kMaxP));
  }
  State sd = make_state(w);
  CK(cudaMemsetAsync(w.ints, 0, sizeof(int) * (w.N + 16), s));
  CK(cudaMemsetAsync(w.scal, 0, sizeof(double) * 8, s));
  CK(cudaMemsetAsync(w.sigma, 0, sizeof(double) * (size_t)(w.N + 4) * kSigmaStride, s));
  CK(cudaMemcpy2DAsync(w.BUb, sizeof(double) * w.LDB, B_U, sizeof(double) * ld_bu, sizeof(double) * rb, M, kind_in(where), s));
  CK(cudaMemcpy2DAsync(w.BV, sizeof(double) * rb, B_V, sizeof(double) * ld_bv, sizeof(double) * rb, n, kind_in(where), s));
  CK(cudaMemcpyAsync(sd.rk + 0, &rb, sizeof(int), cudaMemcpyHostToDevice, s));     // slot 0 := r_B for B
  // ||B||_F
  double b2 = 0.0;
  {
    UDesc ub = ucat_desc(w, M, rb, -1, nullptr, -1, ctx->G);
    VDesc vb{};
    vb.nb = 1; vb.pad_even = 1;
    vb.b[0] = vblock(w.BV, rb, rb, -1, 1.0, -1, 0);
    st = enqueue_norm2(ctx, ub, vb, 0, s);
    if (st != LRC_OK) return st;
    double sc[8];
    CK(cudaMemcpyAsync(sc, w.scal, sizeof(sc), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    b2 = sc[0];
  }
  const double bnorm = std::sqrt(b2);
  const double tau = opts->trunc_tol;
  LR X{w.Ubuf[0], w.Vbuf[0], 0, 1.0, 0};
  CK(cudaMemsetAsync(sd.rk + 0, 0, sizeof(int), s));                               // X = 0
  LR Wv{w.Ubuf[1], w.Vbuf[1], 1, 1.0, 0};
  LR Tm{w.Ubuf[2], w.Vbuf[2], 2, 1.0, 0};
  std::vector<LR> Vb(m + 1);
  for (int j = 0; j <= m; ++j)
    Vb[j] = LR{ctx->gmU + (size_t)j * M * w.LDU, ctx->gmV + (size_t)j * n * cap, 3 + j, 1.0, 0};
  std::vector<int> steps;
  std::vector<double> cres;
  double rho = bnorm > 0 ? 1.0 : 0.0;
  int cycles = 0;
  const int srow = m + 6;           // sigma row for the scratch truncations
  for (int c = 0; c < maxc && bnorm > 0; ++c) {
    cycles = c + 1;
    // R0 = T(B - L(X)) into the basis slot 0
    double beta = 0.0;
    {
      UDesc ud{};
      VDesc vd{};
      ud.pad_even = 1; vd.pad_even = 1;
      ud.b[ud.nb++] = ublock(w.BUb, w.LDB, rb, -1);
      vd.b[vd.nb++] = vblock(w.BV, rb, rb, -1, 1.0, -1, 0);
      if (X.rank > 0) {
        SpmmArgs a = spmm_base(ctx);
        a.U = X.U; a.ldu = w.LDU; a.d_r = sd.rk + X.slot; a.out = w.W3; a.ldo = w.LDU; a.out_off = 0;
        a.out_sstride = (long long)M * w.LDU;
        KL(P_SPMM, s, launch_spmm(SPMM_PLAIN3, a, cap, s));
        for (int g = 0; g < ctx->G; ++g) {
          ud.b[ud.nb++] = ublock(w.W3 + (size_t)g * M * w.LDU, w.LDU, 0, X.slot);
          vd.b[vd.nb++] = vblock(X.V, cap, 0, X.slot, -X.scale, g == ctx->id_group ? -1 : g, 0);
        }
      }
      st = enqueue_truncation(ctx, ud, vd, nullptr, 0, tau, cap, Vb[0].slot, srow, Vb[0].U, w.LDU, Vb[0].V, cap, s, false);
      if (st != LRC_OK) return st;
      st = gm_rank_sigma(ctx, Vb[0].slot, srow, Vb[0].rank, beta);
      if (st != LRC_OK) return st;
    }
    if (beta == 0.0) { rho = 0.0; break; }
    Vb[0].scale = 1.0 / beta;
    std::vector<double> H((size_t)(m + 1) * m, 0.0);
    int k = 0;
    for (int j = 0; j < m; ++j) {
      double fro = 0.0;
      st = gm_apply(ctx, Vb[j], tau, cap, Wv, srow, fro);
      if (st != LRC_OK) return st;
      double hmax = 0.0;
      for (int i = 0; i <= j; ++i) {
        double h = 0.0;
        st = gm_inner(ctx, Wv, Vb[i], cap, h);
        if (st != LRC_OK) return st;
        H[(size_t)i * m + j] = h;
        hmax = std::max(hmax, std::fabs(h));
        LR mi = Vb[i];
        mi.scale = -h * Vb[i].scale;
        st = gm_truncate(ctx, {Wv, mi}, tau, cap, Tm, srow, fro);
        if (st != LRC_OK) return st;
        std::swap(Wv.U, Tm.U); std::swap(Wv.V, Tm.V); std::swap(Wv.slot, Tm.slot);
        Wv.rank = Tm.rank; Wv.scale = 1.0;
      }
      H[(size_t)(j + 1) * m + j] = fro;
      k = j + 1;
      if (fro <= 1e-14 * std::max(hmax, fro)) { H[(size_t)(j + 1) * m + j] = 0.0; break; }   // breakdown (R14)
      // V_{j+1} = W / h_{j+1,j}: move W's factors into the basis slot
      CK(cudaMemcpyAsync(Vb[j + 1].U, Wv.U, sizeof(double) * M * w.LDU, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(Vb[j + 1].V, Wv.V, sizeof(double) * n * cap, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(sd.rk + Vb[j + 1].slot, sd.rk + Wv.slot, sizeof(int), cudaMemcpyDeviceToDevice, s));
      Vb[j + 1].rank = Wv.rank;
      Vb[j + 1].scale = 1.0 / fro;
    }
    std::vector<double> y;
    gm_lsq(H, m, k, beta, y);
    for (int j = 0; j < k; ++j) {             // X = T(... T(X + y_1 V_1) ...)
      LR vj = Vb[j];
      vj.scale = y[j] * Vb[j].scale;
      double fro = 0.0;
      st = gm_truncate(ctx, {X, vj}, tau, cap, Tm, srow, fro);
      if (st != LRC_OK) return st;
      std::swap(X.U, Tm.U); std::swap(X.V, Tm.V); std::swap(X.slot, Tm.slot);
      X.rank = Tm.rank; X.scale = 1.0;
    }
    steps.push_back(k);
    double r2 = 0.0;
    st = gm_residual2(ctx, X, rb, cap, r2);
    if (st != LRC_OK) return st;
    rho = std::sqrt(r2) / bnorm;
    cres.push_back(rho);
    if (rho <= opts->tol) break;
  }
  // outputs (columns >= rank zeroed)
  KL(P_MISC, s, launch_zero_cols(X.U, (int)M, w.LDU, sd.rk + X.slot, 0, cap, s));
  KL(P_MISC, s, launch_zero_cols(X.V, (int)n, cap, sd.rk + X.slot, 0, cap, s));
  CK(cudaMemcpy2DAsync(U_out, sizeof(double) * ld_u, X.U, sizeof(double) * w.LDU, sizeof(double) * cap, M, kind_out(where), s));
  CK(cudaMemcpy2DAsync(V_out, sizeof(double) * ld_v, X.V, sizeof(double) * cap, sizeof(double) * cap, n, kind_out(where), s));
  int flags = 0;
  CK(cudaMemcpyAsync(&flags, sd.flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  ctx->last_record = false;
  if (info) {
    info->cycles = cycles;
    info->rank = X.rank;
    info->rel_residual = rho;
    info->b_norm = bnorm;
    for (int c = 0; c < (int)steps.size() && info->inner_steps; ++c) info->inner_steps[c] = steps[c];
    for (int c = 0; c < (int)cres.size() && info->cycle_residuals; ++c) info->cycle_residuals[c] = cres[c];
  }
  if (flags & 1) return fail(ctx, LRC_ERR_NUMERIC, "shifted Cholesky failed after all escalations");
  if (flags & 2) return fail(ctx, LRC_ERR_NUMERIC, "non-finite singular value in the core SVD");
  return LRC_OK;
}

}  // extern "C"
