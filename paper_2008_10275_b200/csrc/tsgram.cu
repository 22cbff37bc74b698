// a3 / a4 / a6 -- tall-skinny fp64 DMMA kernels of the truncation (
// truncation operator T of PAPER.md P:544).
//
// All three M-level passes of the truncation have the same shape: a row tile of a logical
// concatenation of strided blocks (M x w, up to five blocks, widths read from device-resident
// ranks and padded to even) is multiplied by a small w x p matrix T held in L2, on the fp64 tensor
// pipe (mma.sync.m8n8k4.f64, "DMMA"), and the p-wide tile X = U_tile T is then either
//   GRAM  : contracted with itself, G += X^T X (upper 8x8 tiles in 2x2 register blocks, DMMA),
//           accumulated in registers across the CTA's tiles and written once as a per-CTA partial
//           (deterministic fixed-order reduction in gram_reduce_kernel); optionally X itself is
//           written out (pass 1 keeps Y), or
//   STORE : written out (U_{k+1}, row-major).
// Pass 1: U = Ucat = [B_U | W0' | W1 | W2 | U_{k-1}], T = R_V^T (lower trapezoidal), X = Y stored.
// Pass 2: U = Y, T = R1^{-1} (upper triangular).  Basis pass: U = Y, T = W_r Sigma_r^{-1}.
//
// Tile: 128 rows x p, 16 warps, warp w owns rows [8w, 8w+8) (one 8-row DMMA tile) and all p
// columns.  The K loop streams 32-column chunks of U and 32-row chunks of T through a 3-stage
// shared-memory ring (16-byte cp.async when every block is 16-byte aligned, else 8-byte; zero fill
// past M / w) whose hand-offs are mbarriers.  The X tile of the Gram epilogue is parked in two of
// the (then idle) stages.
#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kThreads = 512;   // 16 warps
constexpr int kWarps = kThreads / 32;
constexpr int kBM = 128;        // rows per tile
// k chunk: 32 for the Gram passes, 36 for the basis pass (p = 100 -> 3 chunks instead of 4; the Gram
// kernels run out of registers with the wider chunk plan).  The U chunk's shared-memory row stride is
// 36 doubles in both cases (== 4 mod 16: conflict-free fragment loads).
template <int MODE> struct BKof { static constexpr int v = MODE == 1 ? 36 : 32; };
constexpr int kSU = 36;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}


// mbarrier helpers for the stage handshakes of the chunk ring
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
// arrives once all of this thread's earlier cp.async copies have landed
__device__ __forceinline__ void mb_arrive_cp(unsigned long long* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_addr(b)), "r"(parity) : "memory");
}

// column offsets of the Ucat blocks (off[nb] = w)
__device__ __forceinline__ int ucat_offsets(const TsArgs& a, int (&off)[kMaxUBlocks + 1]) {
  int o = 0;
#pragma unroll
  for (int bi = 0; bi < kMaxUBlocks; ++bi) {
    off[bi] = o;
    if (bi < a.u.nb) {
      const int wd = a.u.b[bi].w_fixed + (a.u.b[bi].w_idx >= 0 ? a.rk[a.u.b[bi].w_idx] : 0);
      o += a.u.pad_even ? wd + (wd & 1) : wd;
    }
  }
  off[kMaxUBlocks] = o;
  return o;
}

template <int PT, int BK>
struct TsShape {
  static constexpr int PMAX = PT * 8;
  static constexpr int SX = PMAX + 4;                    // T chunk / X tile row stride
  static constexpr int STAGE = kBM * kSU + BK * SX;      // doubles per pipeline stage
  static constexpr int NSTAGE = 3;
  static constexpr int SMEM = NSTAGE * STAGE;
  static constexpr int XH = (kBM / 2) * SX;              // half X tile (64 rows), fits one stage
  static_assert(XH <= STAGE, "half X tile must fit a stage");
  static constexpr int PT2 = (PT + 1) / 2;               // 2x2 super tiles of the Gram
  static constexpr int NS = PT2 * (PT2 + 1) / 2;
  static constexpr int SPW = (NS + kWarps - 1) / kWarps;  // super tiles per warp
  static constexpr int HP = PMAX / 2;                    // 16-byte pieces per T row
};

// Per-thread copy plan of one chunk (tile rows m0.., logical Ucat columns k0..k0+kBK) into a stage.
//   Ucat, 16-byte mode: thread copies column pair 2*(tid&15) of rows (tid>>4) + 32q, q = 0..3
//   Ucat,  8-byte mode: thread copies column tid&31 of rows (tid>>5) + 16q, q = 0..7
//   T: warp wp copies T rows k0+2wp, k0+2wp+1; lane the 16-byte pieces lane, lane+32 (< HP)
// The copies are issued in 8 parts interleaved with the DMMA steps of the previous chunk, so no
// warp ever stalls the tensor pipe on a block of address arithmetic.
struct ChunkPlan {
  const double* ub;   // Ucat source of this thread's column at row m0 (null: column past w)
  int ld;
  const double* ub2;  // the thread's extra copy (columns 32..35 of the chunk), null if none
  int ld2;
  int m0, k0;
  unsigned st;        // stage base (shared address)
};

__device__ __forceinline__ const double* col_src(const TsArgs& a, int col, int m0, int w, const int* off, int& ld) {
  ld = 0;
  if (col >= w) return nullptr;
  int bi = 0;
#pragma unroll
  for (int q = 1; q < kMaxUBlocks; ++q) bi += (col >= off[q]);
  ld = a.u.b[bi].ld;
  return a.u.b[bi].p + (size_t)m0 * ld + (col - off[bi]);
}

// Chunk columns 0..31: 16-byte mode -> pair (tid & 15) of rows (tid >> 4) + 32q; 8-byte mode ->
// column (tid & 31) of rows (tid >> 5) + 16q.  Columns 32..35: 16-byte mode -> pair 16 + (tid & 1)
// of row tid >> 1 (threads < 256); 8-byte mode -> column 32 + (tid & 3) of row tid >> 2.
template <int PT, int BK>
__device__ __forceinline__ ChunkPlan plan_chunk(const TsArgs& a, unsigned stage, int m0, int k0, int w,
                                                const int* off, int tid) {
  ChunkPlan c;
  c.m0 = m0; c.k0 = k0; c.st = stage;
  c.ub = col_src(a, k0 + (a.u16 ? (tid & 15) * 2 : (tid & 31)), m0, w, off, c.ld);
  c.ub2 = nullptr; c.ld2 = 0;
  if (BK > 32 && (!a.u16 || tid < 256))
    c.ub2 = col_src(a, k0 + 32 + (a.u16 ? (tid & 1) * 2 : (tid & 3)), m0, w, off, c.ld2);
  return c;
}

template <int PT, int BK>
__device__ __forceinline__ void issue_part(const TsArgs& a, const ChunkPlan& c, int part, int w, int tid) {
  using S = TsShape<PT, BK>;
  if (a.u16) {
    if (part < 4) {
      const int i = (tid >> 4) + 32 * part, j = (tid & 15) * 2;
      const bool ok = c.ub != nullptr && (c.m0 + i < a.M);
      const double* src = ok ? c.ub + (size_t)i * c.ld : a.u.b[0].p;
      const unsigned sa = c.st + 8u * (i * kSU + j);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
    }
  } else {
    const int i = (tid >> 5) + 16 * part, j = tid & 31;
    const bool ok = c.ub != nullptr && (c.m0 + i < a.M);
    const double* src = ok ? c.ub + (size_t)i * c.ld : a.u.b[0].p;
    const unsigned sa = c.st + 8u * (i * kSU + j);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 8 : 0));
  }
  if (BK > 32 && part == 4) {   // U chunk columns 32..35
    if (a.u16) {
      if (tid < 256) {
        const int i = tid >> 1, j = 32 + (tid & 1) * 2;
        const bool ok = c.ub2 != nullptr && (c.m0 + i < a.M);
        const double* src = ok ? c.ub2 + (size_t)i * c.ld2 : a.u.b[0].p;
        const unsigned sa = c.st + 8u * (i * kSU + j);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 16 : 0));
      }
    } else {
      const int i = tid >> 2, j = 32 + (tid & 3);
      const bool ok = c.ub2 != nullptr && (c.m0 + i < a.M);
      const double* src = ok ? c.ub2 + (size_t)i * c.ld2 : a.u.b[0].p;
      const unsigned sa = c.st + 8u * (i * kSU + j);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 8 : 0));
    }
  }
  if (part >= 4) {   // T chunk rows 0..31 (warp wp: rows 2wp, 2wp+1)
    const int q = part - 4;
    const int wp = tid >> 5, lane = tid & 31;
    const int row = 2 * wp + (q >> 1), piece = lane + 32 * (q & 1);
    if (piece < S::HP) {
      const int cr = c.k0 + row;
      const bool ok = cr < w;
      const double* g = ok ? a.T + (size_t)cr * a.ldt + 2 * piece : a.T;
      const unsigned sa = c.st + 8u * (kBM * kSU + row * S::SX + 2 * piece);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
    }
  }
  if (BK > 32 && part == 5 && tid < 4 * 64) {   // T chunk rows 32..35
    const int row = 32 + (tid >> 6), piece = tid & 63;
    if (piece < S::HP) {
      const int cr = c.k0 + row;
      const bool ok = cr < w;
      const double* g = ok ? a.T + (size_t)cr * a.ldt + 2 * piece : a.T;
      const unsigned sa = c.st + 8u * (kBM * kSU + row * S::SX + 2 * piece);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 16 : 0));
    }
  }
}

// One chunk (BK columns of the logical Ucat / rows of T) of a warp's 8-row X slice, with the set of
// active n-tiles of every k4 step known at compile time: KIND 0 = all PT n-tiles (the bulk of the
// K range), KIND 1 = chunk KC of a lower-trapezoidal T (T1 = R_V^T: n-tile n is zero for rows
// < 8n), KIND 2 = chunk KC of an upper-triangular T (R1^{-1}: n-tile n is zero for rows >= 8n + 8).
// Skipped DMMAs are not emitted at all (a predicated-off DMMA still occupies the tensor pipe), and
// there is no per-k-step dispatch.  nka = active k4 steps of the chunk (the zero tail past w is
// skipped); issue(kk) interleaves the next chunk's copy issue with the DMMA steps.
template <int PT, int BK, int KIND, int KC, typename Issue>
__device__ __forceinline__ void chunk_mma(double (&x0)[PT][2], const double* sa, const double* st, int nka,
                                          Issue&& issue) {
  constexpr int SX = PT * 8 + 4;
#pragma unroll
  for (int kk = 0; kk < BK; kk += 4) {
    if (kk / 4 < nka) {
      const double a0 = sa[kk];
      const double* bt = st + kk * SX;
      constexpr int dummy = 0;
      (void)dummy;
#pragma unroll
      for (int n = 0; n < PT; ++n) {
        const int k = KC * BK + kk;                       // compile-time for KIND 1, 2
        const bool on = KIND == 0 ? true : (KIND == 1 ? (8 * n <= k + 3) : (8 * n + 8 > k));
        if (on) dmma884(x0[n], a0, bt[n * 8]);
      }
    }
    issue(kk);
  }
}

// Gram contribution of the parked 128-row X tile to one 2x2 super tile (I0, J0) of G (8x8 tiles):
// KIND 0 full, 1 diagonal (the lower tile is skipped), 2 last column of odd PT (J0+1 absent),
// 3 last diagonal of odd PT (one tile).
template <int KIND, int SX>
__device__ __forceinline__ void gram_tile(double (&acc)[4][2], const double* xh0, const double* xh1, int I0,
                                          int J0, int tig, int gid) {
#pragma unroll 4
  for (int k = 0; k < kBM; k += 4) {
    const double* xr = (k < 64 ? xh0 : xh1) + ((k & 63) + tig) * SX + gid;
    const double a0 = xr[I0 * 8], b0 = xr[J0 * 8];
    if constexpr (KIND == 0) {
      const double a1 = xr[(I0 + 1) * 8], b1 = xr[(J0 + 1) * 8];
      dmma884(acc[0], a0, b0); dmma884(acc[1], a0, b1); dmma884(acc[2], a1, b0); dmma884(acc[3], a1, b1);
    } else if constexpr (KIND == 1) {
      const double a1 = xr[(I0 + 1) * 8], b1 = xr[(J0 + 1) * 8];
      dmma884(acc[0], a0, b0); dmma884(acc[1], a0, b1); dmma884(acc[3], a1, b1);
    } else if constexpr (KIND == 2) {
      const double a1 = xr[(I0 + 1) * 8];
      dmma884(acc[0], a0, b0); dmma884(acc[2], a1, b0);
    } else {
      dmma884(acc[0], a0, b0);
    }
  }
}

template <int PT, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
ts_kernel(TsArgs a) {
  constexpr int kBK = BKof<MODE>::v;
  using S = TsShape<PT, kBK>;
  constexpr int PMAX = S::PMAX, SX = S::SX;

  // block column offsets in shared memory (keeps them out of the register budget)
  __shared__ int off[kMaxUBlocks + 1];
  int w;
  {
    int o[kMaxUBlocks + 1];
    w = ucat_offsets(a, o);
    if (threadIdx.x <= kMaxUBlocks) off[threadIdx.x] = o[threadIdx.x];
  }
  const int p = a.d_p ? *a.d_p : a.p_fixed;
  const int ntiles = (a.M + kBM - 1) / kBM;
  if (w <= 0 || p <= 0 || (int)blockIdx.x >= ntiles) {
    if (MODE == 0) {   // still publish a zero partial so the reduction is well defined
      double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
      for (int e = threadIdx.x; e < PMAX * PMAX; e += kThreads) part[e] = 0.0;
    }
    return;
  }

  extern __shared__ double sm[];
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;

  // Gram super tiles (I2, J2), I2 <= J2, of this warp
  double gacc[S::SPW][4][2];
  int sI[S::SPW], sJ[S::SPW];
#pragma unroll
  for (int s = 0; s < S::SPW; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) gacc[s][q][0] = gacc[s][q][1] = 0.0;
    int t = warp + kWarps * s, I = 0;
    if (t >= S::NS) { sI[s] = -1; sJ[s] = -1; continue; }
    while (t >= S::PT2 - I) { t -= S::PT2 - I; ++I; }
    sI[s] = I; sJ[s] = I + t;
  }

  const int nk = (w + kBK - 1) / kBK;
  // Chunks of all this CTA's tiles form one sequence g = 0, 1, ...; chunk g lives in stage g % 3.
  // Chunk g+1 is in flight while g is computed and g+2 is issued during the second half of g's DMMA
  // steps, except that at most the next tile's chunk 0 is prefetched across a tile boundary: the X
  // tile of the epilogue is parked (as two 64-row halves) in the two stages that chunk does not use.
  // Stage hand-offs are mbarriers instead of CTA barriers: full[s] completes when every thread's
  // copies of the chunk in stage s have landed (cp.async arrive-on), empty[s] when every warp has
  // contracted it; use count u of a stage -> parity u & 1.
  __shared__ __align__(8) unsigned long long full[3], empty[3];
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) { mb_init(&full[i], kThreads); mb_init(&empty[i], kWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  auto produce_wait = [&](int h) { if (h >= 3) mb_wait(&empty[h % 3], ((h / 3) - 1) & 1); };
  int g = 0, issued = 0;
  __syncthreads();   // off[], barriers
  {
    const ChunkPlan c0 = plan_chunk<PT, kBK>(a, sbase, blockIdx.x * kBM, 0, w, off, tid);
#pragma unroll
    for (int part = 0; part < 8; ++part) issue_part<PT, kBK>(a, c0, part, w, tid);
    mb_arrive_cp(&full[0]);
  }
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int m0 = tile * kBM;
    const bool has_next = tile + (int)gridDim.x < ntiles;
    double x0[PT][2];
#pragma unroll
    for (int n = 0; n < PT; ++n) x0[n][0] = x0[n][1] = 0.0;

    for (int kc = 0; kc < nk; ++kc, ++g) {
      // tile start: the previous tile's X halves are fully consumed (the direct-store basis pass
      // parks no X tile)
      if (kc == 0 && !(MODE == 1 && a.o16)) __syncthreads();
      if (issued == g) {
        // (tile start without prefetch) chunk g+1 now, before computing g
        int nm0 = -1, nk0 = 0;
        if (kc + 1 < nk) { nm0 = m0; nk0 = (kc + 1) * kBK; }
        else if (has_next) { nm0 = m0 + gridDim.x * kBM; nk0 = 0; }
        if (nm0 >= 0) {
          produce_wait(g + 1);
          const ChunkPlan c1 = plan_chunk<PT, kBK>(a, sbase + 8u * S::STAGE * ((g + 1) % 3), nm0, nk0, w, off, tid);
#pragma unroll
          for (int part = 0; part < 8; ++part) issue_part<PT, kBK>(a, c1, part, w, tid);
          mb_arrive_cp(&full[(g + 1) % 3]);
          issued = g + 1;
        }
      }
      mb_wait(&full[g % 3], (g / 3) & 1);   // chunk g has landed
      // chunk g+2 (this tile's kc+2, or the next tile's chunk 0) is issued during the DMMA steps
      int pm0 = -1, pk0 = 0;
      if (issued == g + 1) {
        if (kc + 2 < nk) { pm0 = m0; pk0 = (kc + 2) * kBK; }
        else if (kc + 2 == nk && has_next) { pm0 = m0 + gridDim.x * kBM; pk0 = 0; }
      }
      ChunkPlan c2;
      if (pm0 >= 0) c2 = plan_chunk<PT, kBK>(a, sbase + 8u * S::STAGE * ((g + 2) % 3), pm0, pk0, w, off, tid);
      const double* s_u = sm + (g % 3) * S::STAGE;
      const double* s_t = s_u + kBM * kSU;
      const int k0 = kc * kBK;
      const double* sa = s_u + (warp * 8 + gid) * kSU + tig;
      const double* st = s_t + tig * SX + gid;
      const int nka = max(0, min(kBK / 4, (w - k0 + 3) / 4));
      // second half of the chunk: issue chunk g+2 (the stage of chunk g-1 is (almost surely) free)
      constexpr int kIssue0 = kBK - 16;   // the last four k4 steps issue two parts each
      auto issue = [&](int kk) {
        if (pm0 >= 0 && kk >= kIssue0) {
          if (kk == kIssue0) produce_wait(g + 2);
          issue_part<PT, kBK>(a, c2, 2 * ((kk - kIssue0) / 4), w, tid);
          issue_part<PT, kBK>(a, c2, 2 * ((kk - kIssue0) / 4) + 1, w, tid);
        }
      };
      if constexpr (MODE == 0) {
        if (a.t_lower && k0 + 3 < 8 * (PT - 1)) {
          switch (kc) {
            case 0: chunk_mma<PT, kBK, 1, 0>(x0, sa, st, nka, issue); break;
            case 1: chunk_mma<PT, kBK, 1, 1>(x0, sa, st, nka, issue); break;
            case 2: chunk_mma<PT, kBK, 1, 2>(x0, sa, st, nka, issue); break;
            default: chunk_mma<PT, kBK, 1, 3>(x0, sa, st, nka, issue); break;
          }
        } else if (a.t_upper && kc < 4) {
          switch (kc) {
            case 0: chunk_mma<PT, kBK, 2, 0>(x0, sa, st, nka, issue); break;
            case 1: chunk_mma<PT, kBK, 2, 1>(x0, sa, st, nka, issue); break;
            case 2: chunk_mma<PT, kBK, 2, 2>(x0, sa, st, nka, issue); break;
            default: chunk_mma<PT, kBK, 2, 3>(x0, sa, st, nka, issue); break;
          }
        } else {
          chunk_mma<PT, kBK, 0, 0>(x0, sa, st, nka, issue);
        }
      } else {
        chunk_mma<PT, kBK, 0, 0>(x0, sa, st, nka, issue);
      }
      if (pm0 >= 0) { mb_arrive_cp(&full[(g + 2) % 3]); issued = g + 2; }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[g % 3]);   // this warp is done with stage g % 3
    }
    if (MODE == 0 && a.yout) {
      // Y = this X tile straight from the accumulators (all PMAX columns; the ones >= p are exact
      // zeros): fire-and-forget 16-byte evict-first stores, full 32-byte sectors per quad
      const int row = m0 + warp * 8 + gid;
      if (row < a.M) {
        double* yr = a.yout + (size_t)row * a.ldy + 2 * tig;
#pragma unroll
        for (int n = 0; n < PT; ++n) __stcs(reinterpret_cast<double2*>(yr + n * 8), make_double2(x0[n][0], x0[n][1]));
      }
    }
    if (MODE == 1 && a.o16) {
      // rows of U_{k+1} straight from the accumulators (16-byte evict-first stores, full sectors);
      // the padded (solver) mode also writes the zero pad column of an odd rank
      const int pw = p + (a.u.pad_even ? (p & 1) : 0);
      const int row = m0 + warp * 8 + gid;
      if (row < a.M) {
        double* orow = a.out + (size_t)row * a.ldo;
#pragma unroll
        for (int n = 0; n < PT; ++n) {
          const int c = n * 8 + 2 * tig;
          if (c + 1 < pw) __stcs(reinterpret_cast<double2*>(orow + c), make_double2(x0[n][0], x0[n][1]));
          else if (c < pw) __stcs(orow + c, x0[n][0]);
        }
      }
      continue;
    }
    // X tile -> the two stages not holding the next tile's chunk 0 (chunk g, if issued)
    __syncthreads();   // every warp is done with the last chunk
    double* xh0 = sm + ((g + 1) % 3) * S::STAGE;   // rows 0..63
    double* xh1 = sm + ((g + 2) % 3) * S::STAGE;   // rows 64..127
    {
      double* xr = (warp < 8 ? xh0 : xh1) + ((warp & 7) * 8 + gid) * SX;
#pragma unroll
      for (int n = 0; n < PT; ++n)
        *reinterpret_cast<double2*>(xr + n * 8 + 2 * tig) = make_double2(x0[n][0], x0[n][1]);
    }
    __syncthreads();
    if constexpr (MODE == 0) {
#pragma unroll
      for (int s = 0; s < S::SPW; ++s) {
        if (sI[s] < 0) continue;
        const int I0 = 2 * sI[s], J0 = 2 * sJ[s];
        // odd PT: the last super row/column is half; the kind is warp-uniform and fixed, so each
        // kind runs its own loop (no predicated-off DMMAs)
        const bool i1 = I0 + 1 < PT, j1 = J0 + 1 < PT;
        const int kind = (sI[s] == sJ[s]) ? (i1 ? 1 : 3) : (j1 ? 0 : 2);
        if (kind == 0) gram_tile<0, SX>(gacc[s], xh0, xh1, I0, J0, tig, gid);
        else if (kind == 1) gram_tile<1, SX>(gacc[s], xh0, xh1, I0, J0, tig, gid);
        else if (kind == 2) gram_tile<2, SX>(gacc[s], xh0, xh1, I0, J0, tig, gid);
        else gram_tile<3, SX>(gacc[s], xh0, xh1, I0, J0, tig, gid);
      }
    } else {
      // rows of U_{k+1}: 16-byte stores when the output rows are 16-byte aligned
      const int pw = p + (a.u.pad_even ? (p & 1) : 0);   // padded (solver) mode also writes the zero pad column
      if (a.o16) {
        constexpr int HP = S::HP;
        for (int e = tid; e < kBM * HP; e += kThreads) {
          const int i = e / HP, j = 2 * (e - (e / HP) * HP);
          const int m = m0 + i;
          const double* xr = (i < 64 ? xh0 : xh1) + (i & 63) * SX + j;
          if (m < a.M && j < pw) {
            if (j + 1 < pw) __stcs(reinterpret_cast<double2*>(a.out + (size_t)m * a.ldo + j), *reinterpret_cast<const double2*>(xr));
            else __stcs(a.out + (size_t)m * a.ldo + j, xr[0]);
          }
        }
      } else {
        for (int e = tid; e < kBM * PMAX; e += kThreads) {
          const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
          const int m = m0 + i;
          if (m < a.M && j < pw) a.out[(size_t)m * a.ldo + j] = ((i < 64 ? xh0 : xh1) + (i & 63) * SX)[j];
        }
      }
    }
    // the next tile's first barrier protects the X halves before chunk g+1 overwrites one of them
  }

  if constexpr (MODE == 0) {
    double* part = a.partials + (size_t)blockIdx.x * PMAX * PMAX;
    // lower 8x8 tiles are never computed: zero them so the reduction reads defined data
    for (int e = tid; e < PMAX * PMAX; e += kThreads) {
      const int i = e / PMAX, j = e - (e / PMAX) * PMAX;
      if ((i >> 3) > (j >> 3)) part[e] = 0.0;
    }
#pragma unroll
    for (int s = 0; s < S::SPW; ++s) {
      if (sI[s] >= 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int I = 2 * sI[s] + (q >> 1), J = 2 * sJ[s] + (q & 1);
          if (I < PT && J < PT && I <= J) {
            const int row = I * 8 + gid, col = J * 8 + 2 * tig;
            part[row * PMAX + col] = gacc[s][q][0];
            part[row * PMAX + col + 1] = gacc[s][q][1];
          }
        }
      }
    }
  }
}

template <int PT, int MODE>
cudaError_t launch_pt(const TsArgs& a, int grid, cudaStream_t s) {
  ts_kernel<PT, MODE><<<grid, kThreads, sizeof(double) * TsShape<PT, BKof<MODE>::v>::SMEM, s>>>(a);
  return cudaGetLastError();
}

template <int PT, int MODE>
cudaError_t prep_pt() {
  return cudaFuncSetAttribute(ts_kernel<PT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(sizeof(double) * TsShape<PT, BKof<MODE>::v>::SMEM));
}

template <int MODE, int PT>
struct Dispatch {
  static cudaError_t launch(const TsArgs& a, int pt, int grid, cudaStream_t s) {
    if (pt == PT) return launch_pt<PT, MODE>(a, grid, s);
    return Dispatch<MODE, PT - 1>::launch(a, pt, grid, s);
  }
  static cudaError_t prep() {
    cudaError_t e = prep_pt<PT, MODE>();
    return e != cudaSuccess ? e : Dispatch<MODE, PT - 1>::prep();
  }
};
template <int MODE>
struct Dispatch<MODE, 0> {
  static cudaError_t launch(const TsArgs&, int, int, cudaStream_t) { return cudaErrorInvalidValue; }
  static cudaError_t prep() { return cudaSuccess; }
};

__global__ void gram_reduce_kernel(const double* __restrict__ partials, int nblocks, int pmax,
                                   double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int n2 = pmax * pmax;
  if (e >= n2) return;
  const int i = e / pmax, j = e - (e / pmax) * pmax;
  if (i > j) return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b) s += partials[(size_t)b * n2 + e];   // fixed order
  G[i * pmax + j] = s;
  G[j * pmax + i] = s;
}

}  // namespace

cudaError_t ts_prepare() {
  cudaError_t e = Dispatch<0, 16>::prep();
  return e != cudaSuccess ? e : Dispatch<1, 16>::prep();
}

int ts_pmax_for(int p) {
  if (p < 1 || p > 128) return -1;
  return 8 * ((p + 7) / 8);
}

int ts_grid_for(int M, int reserved) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int ntiles = (M + kBM - 1) / kBM;
  int g = sms - (reserved > 0 ? reserved : 0);
  if (g < 1) g = 1;
  return ntiles < g ? (ntiles > 0 ? ntiles : 1) : g;
}

cudaError_t launch_ts(int mode, const TsArgs& a0, int pmax, int grid, cudaStream_t s) {
  if (pmax % 8 || pmax < 8 || pmax > 128) return cudaErrorInvalidValue;
  TsArgs a = a0;
  bool u16 = a.u.pad_even != 0;
  for (int bi = 0; bi < a.u.nb; ++bi)
    u16 = u16 && (a.u.b[bi].ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.u.b[bi].p) & 15) == 0);
  a.u16 = u16 ? 1 : 0;
  a.o16 = (mode == 1 && a.out && a.ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(a.out) & 15) == 0) ? 1 : 0;
  return mode == 0 ? Dispatch<0, 16>::launch(a, pmax / 8, grid, s)
                   : Dispatch<1, 16>::launch(a, pmax / 8, grid, s);
}

cudaError_t launch_gram_reduce(const double* partials, int nblocks, int pmax, double* G,
                               cudaStream_t s) {
  const int n2 = pmax * pmax;
  gram_reduce_kernel<<<(n2 + 255) / 256, 256, 0, s>>>(partials, nblocks, pmax, G);
  return cudaGetLastError();
}

}  // namespace lrc
