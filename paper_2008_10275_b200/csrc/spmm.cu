// a1 -- fused six-array CSR SpMM (`equation_intro_mat1`).
//
// One pass over the shared CSR pattern reads each of the six fp64 value arrays once and the shared
// column indices once per node block, and produces the operator grouped by right diagonal (exact,
// Kronecker identity I(x)(A0+rho Jrho+lam Jlam) + Dmu(x)(A1+Jmu) + Dnu(x)(rho A2)):
//     W0 = (A0 + rho Jrho + lam Jlam) U,  W1 = (A1 + Jmu) U,  W2 = rho A2 U,
// with the Chebyshev-step epilogue W0' = U - gamma W0 fused (S2STEP).  The D_mu / D_nu scaling
// of the terms lives on the V side (n rows), never on the M side (vside kernel).
//
// Mapping: rows come in node blocks -- runs of <= 8 consecutive rows with
// identical column lists (the 5 field rows of an FE node share one list), detected at
// set_operator -- packed into CTA tiles of <= 4 blocks / kSpmmCap nnz / kUCap deduplicated U rows,
// each described by a 1 KB host-built descriptor (U-path tiles stored first).  The hot kernel
// (spmm_u_kernel, 8 warps, 3 CTAs/SM) loads the tile's six contiguous value segments into
// registers (evict-first), stages the tile's deduplicated U rows in shared memory (TMA bulk copies
// behind an mbarrier), combines the six arrays into the three grouped streams in a conflict-free
// [slot][j] layout, and gives each warp one (node block, 32-column slice) contraction on the fp64
// tensor pipe (m16n8k4 DMMA, computed transposed so stores are full sectors).  Tiles whose rows do
// not fit the U-path bounds take the general spmm_kernel (L2 gather).  spmm_dense_kernel is the
// config-5 dense variant.
#include <algorithm>
#include <type_traits>

#include "lrc_internal.cuh"

namespace lrc {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPre = 4;                 // U gather prefetch depth

template <int MODE>
struct Nacc { static constexpr int v = (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) ? 3 : 1; };
template <int MODE>
struct Nstage { static constexpr int v = (MODE == SPMM_SINGLE) ? 1 : 3; };

// Staged values are laid out [slot][j] (slot = row*NV + stream, j = column-list entry) with a row
// pitch == 4 (mod 16) doubles: the staging stores (consecutive j) and the DMMA fragment loads
// (8 slots x 4 entries) are both bank-conflict free.
__device__ __forceinline__ int row_pitch(int L) { return L + ((20 - (L & 15)) & 15); }

template <int MODE>
__device__ __forceinline__ void stage_entry(const SpmmArgs& a, int idx, double* dst, int lp, double cs) {
  if constexpr (MODE == SPMM_SINGLE) {
    dst[0] = cs * __ldcs(a.v[a.single_t] + idx);
  } else {
    const double v0 = __ldcs(a.v[0] + idx), v1 = __ldcs(a.v[1] + idx), v2 = __ldcs(a.v[2] + idx);
    const double v3 = __ldcs(a.v[3] + idx), v4 = __ldcs(a.v[4] + idx), v5 = __ldcs(a.v[5] + idx);
    dst[0] = fma(a.lam, v5, fma(a.rho, v3, v0));   // A0 + rho Jrho + lam Jlam
    dst[lp] = v1 + v4;                             // A1 + Jmu
    dst[2 * lp] = a.rho * v2;                      // rho A2
  }
}

// One warp: rows [row0, row0 + gs) of a node block (their staged entries at
// vals[((qo + q) * NV + t) * lp + j]), columns c = c0 + lane, over the jn staged column-list entries.
template <int MODE, int GM>
__device__ __forceinline__ void block_task(const SpmmArgs& a, int r, int c, int row0, int gs, int qo,
                                           int jn, int lp, const double* vals, const int* cols,
                                           double (&acc)[GM][Nacc<MODE>::v]) {
  constexpr int NV = Nstage<MODE>::v;
  const bool act = c < r;
  double dmu_c = 0.0, dnu_c = 0.0;
  if constexpr (MODE == SPMM_DENSE) {
    if (act) { dmu_c = a.dmu[c]; dnu_c = a.dnu[c]; }
  }
  double ring[kPre];
#pragma unroll
  for (int d = 0; d < kPre; ++d) ring[d] = (d < jn && act) ? __ldg(a.U + (size_t)cols[d] * a.ldu + c) : 0.0;
  for (int j0 = 0; j0 < jn; j0 += kPre) {
#pragma unroll
    for (int t = 0; t < kPre; ++t) {
      const int j = j0 + t;
      if (j >= jn) break;
      const double u = ring[t];
      const int jp = j + kPre;
      ring[t] = (jp < jn && act) ? __ldg(a.U + (size_t)cols[jp] * a.ldu + c) : 0.0;
      const double* vj = vals + qo * NV * lp + j;
#pragma unroll
      for (int q = 0; q < GM; ++q) {
        if (q < gs) {
          if constexpr (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) {
            acc[q][0] = fma(vj[(q * 3 + 0) * lp], u, acc[q][0]);
            acc[q][1] = fma(vj[(q * 3 + 1) * lp], u, acc[q][1]);
            acc[q][2] = fma(vj[(q * 3 + 2) * lp], u, acc[q][2]);
          } else if constexpr (MODE == SPMM_DENSE) {
            const double coef = fma(dnu_c, vj[(q * 3 + 2) * lp], fma(dmu_c, vj[(q * 3 + 1) * lp], vj[(q * 3) * lp]));
            acc[q][0] = fma(coef, u, acc[q][0]);
          } else {
            acc[q][0] = fma(vj[q * lp], u, acc[q][0]);
          }
        }
      }
    }
  }
  (void)row0;
}

__device__ __forceinline__ void dmma1684(double (&d)[4], double a0, double a1, double b) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// Hot modes (S2STEP / PLAIN3) on the fp64 tensor pipe: a node sub-block of gs <= 5 rows is the
// dense contraction  [3 gs x L] (rows q*3 + stream, staged values) x [L x 32] (gathered U rows),
// done as m16n8k4 DMMA over 4-entry k steps with the next step's U gather in flight.  Writes the
// three grouped outputs (and the S2STEP epilogue) straight from the accumulator fragments.
template <int MODE>
__device__ __forceinline__ void block_task_mma(const SpmmArgs& a, int r, int n0, int row0, int gs, int qo,
                                               int L, int lp, const double* vals, const int* cols,
                                               int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int nrow = gs * 3;
  const int ra = gid, rb = gid + 8;
  double acc[4][4];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0;
  // prologue: gather for k step 0
  double bnext[4];
  {
    const int j = tig;
    const bool jv = j < L;
    const double* urow = a.U + (size_t)(jv ? cols[j] : 0) * a.ldu;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int c = n0 + nt * 8 + gid;
      bnext[nt] = (jv && c < r) ? __ldg(urow + c) : 0.0;
    }
  }
  for (int k0 = 0; k0 < L; k0 += 4) {
    double b[4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) b[nt] = bnext[nt];
    {
      const int j = k0 + 4 + tig;
      const bool jv = j < L;
      const double* urow = a.U + (size_t)(jv ? cols[j] : 0) * a.ldu;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = n0 + nt * 8 + gid;
        bnext[nt] = (jv && c < r) ? __ldg(urow + c) : 0.0;
      }
    }
    const int j = k0 + tig;
    const bool jv = j < L;
    const double* vj = vals + qo * 3 * lp + j;
    const double a0 = (jv && ra < nrow) ? vj[ra * lp] : 0.0;
    const double a1 = (jv && rb < nrow) ? vj[rb * lp] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) dmma1684(acc[nt], a0, a1, b[nt]);
  }
  // epilogue: fragment (R, C) -> output row row0 + R/3, stream R%3, column n0 + nt*8 + 2 tig + {0,1}
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int R = h ? rb : ra;
    if (R >= nrow) continue;
    const int q = R / 3, st = R - (R / 3) * 3;
    const size_t row = (size_t)(row0 + q);
    double* orow = a.out + st * (a.out_sstride ? a.out_sstride : r) + row * a.ldo + a.out_off;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = n0 + nt * 8 + 2 * tig + e;
        if (c < r) {
          double v = acc[nt][h * 2 + e];
          if (MODE == SPMM_S2STEP && st == 0) v = fma(-a.gamma, v, __ldg(a.U + row * a.ldu + c));
          __stcs(orow + c, v);
        } else if (c == r && (r & 1) && a.out_sstride) {
          __stcs(orow + c, 0.0);          // zero pad column of the (even-padded) Ucat block
        }
      }
    }
  }
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  while (!mbar_try(b, parity)) {}
}


__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// warm L2 with a global range (no shared memory, no completion tracking): the producer of the TMA
// kernel runs this a few tiles ahead of its shared-memory stages so more HBM traffic is in flight
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// rows of U (r columns, ldu even, 16-byte aligned) -> s_u (row stride ust even) in 16-byte chunks
__device__ __forceinline__ void stage_u_rows(const SpmmArgs& a, int r, const int* ids, int nu, double* su,
                                             int ust, int tid, int nthreads) {
  // one warp per U row, lanes over the row (no per-copy integer division)
  const int lane = tid & 31, wp = tid >> 5, nw = nthreads >> 5;
  if (a.u_aligned16) {
    const int nch = (r + 1) >> 1;   // an odd r copies one element of padding (r + 1 <= ldu)
    for (int u = wp; u < nu; u += nw) {
      const double* src = a.U + (size_t)ids[u] * a.ldu;
      for (int ch = lane; ch < nch; ch += 32) cp_async16(su + u * ust + 2 * ch, src + 2 * ch);
    }
  } else {
    for (int u = wp; u < nu; u += nw) {
      const double* src = a.U + (size_t)ids[u] * a.ldu;
      for (int c = lane; c < r; c += 32) cp_async8(su + u * ust + c, src + c);
    }
  }
}

// Same contraction with the tile's deduplicated U rows already in shared memory (row stride ust),
// computed transposed so stores are full sectors:  D^T (32 cols x 3 gs) = U_tile^T (32 x L) Vals^T.
// m16n8k4: M = 16 U columns (A = U^T from s_u, lcols[j] = local row of entry j), N = 8 row*3+stream
// slots (B = staged values), K = 4 column-list entries.  lrow0 = local row of the block's first row
// in s_u (for the S2STEP epilogue), -1 if absent.
template <int MODE>
__device__ __forceinline__ void block_task_mma_smem(const SpmmArgs& a, int r, int n0, int row0, int gs,
                                                    int qo, int L, int lp, const double* vals,
                                                    const unsigned short* lcols, const double* s_u, int ust,
                                                    int lrow0, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int nrow = gs * 3;
  double acc[2][2][4];   // [m tile (16 cols)][n tile (8 slots)][frag]
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.0;
  for (int k0 = 0; k0 < L; k0 += 4) {
    const int j = k0 + tig;
    const bool jv = j < L;
    const double* vj = vals + qo * 3 * lp + j;
    const double b0 = (jv && gid < nrow) ? vj[gid * lp] : 0.0;
    const double b1 = (jv && gid + 8 < nrow) ? vj[(gid + 8) * lp] : 0.0;
    const double* urow = s_u + (jv ? lcols[j] : 0) * ust;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int cA = n0 + mt * 16 + gid, cB = cA + 8;
      const double a0 = (jv && cA < r) ? urow[cA] : 0.0;
      const double a1 = (jv && cB < r) ? urow[cB] : 0.0;
      dmma1684(acc[mt][0], a0, a1, b0);
      dmma1684(acc[mt][1], a0, a1, b1);
    }
  }
  // epilogue: frag (m, n) -> column n0 + mt*16 + m, slot R = nt*8 + n = q*3 + stream
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int R = nt * 8 + 2 * tig + e;
      if (R >= nrow) continue;
      const int q = R / 3, st = R - (R / 3) * 3;
      const size_t row = (size_t)(row0 + q);
      double* orow = a.out + st * (a.out_sstride ? a.out_sstride : r) + row * a.ldo + a.out_off;
      const double* urow_self = (lrow0 >= 0) ? s_u + (lrow0 + qo + q) * ust : a.U + row * a.ldu;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
#pragma unroll
        for (int hm = 0; hm < 2; ++hm) {
          const int c = n0 + mt * 16 + gid + hm * 8;
          if (c < r) {
            double v = acc[mt][nt][hm * 2 + e];
            if (MODE == SPMM_S2STEP && st == 0) v = fma(-a.gamma, v, urow_self[c]);
            __stcs(orow + c, v);
          } else if (c == r && (r & 1) && a.out_sstride) {
            __stcs(orow + c, 0.0);        // zero pad column of the (even-padded) Ucat block
          }
        }
      }
    }
  }
}

// block_task_mma_smem without per-step predicates (spmm_u_kernel): the staged values are
// zero-filled up to the next multiple of 4 column-list entries, the local U row index is clamped,
// and out-of-range slots / U columns only feed accumulator entries that are never stored.
template <int MODE>
__device__ __forceinline__ void block_task_mma_fast(const SpmmArgs& a, int r, int n0, int row0, int gs,
                                                    int qo, int L, int lp, const double* vals,
                                                    const unsigned short* lcols, const double* s_u, int ust,
                                                    int lrow0, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  const int nrow = gs * 3;
  double acc[2][2][4];   // [m tile (16 cols)][n tile (8 slots)][frag]
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.0;
  const int L4 = (L + 3) & ~3;
  const double* vb = vals + (qo * 3 + gid) * lp + tig;
  const double* ub = s_u + n0 + gid;
  const unsigned short* lc = lcols + tig;
  const int lmax = L - 1 - tig;
#pragma unroll 2
  for (int k0 = 0; k0 < L4; k0 += 4) {
    const double b0 = vb[k0], b1 = vb[8 * lp + k0];
    const double* urow = ub + (int)lc[min(k0, lmax)] * ust;
    const double a00 = urow[0], a01 = urow[8], a10 = urow[16], a11 = urow[24];
    dmma1684(acc[0][0], a00, a01, b0);
    dmma1684(acc[0][1], a00, a01, b1);
    dmma1684(acc[1][0], a10, a11, b0);
    dmma1684(acc[1][1], a10, a11, b1);
  }
  // epilogue: frag (m, n) -> column n0 + mt*16 + m, slot R = nt*8 + n = q*3 + stream.  A lane's
  // four values of one slot sit in one output row at columns n0 + gid + {0, 8, 16, 24}; the S2
  // update out0 = U - gamma W0 is applied branch-free (alpha, beta) from the staged U row.
  const long long sst = a.out_sstride ? a.out_sstride : r;
  const bool full = n0 + 32 <= r;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int R = nt * 8 + 2 * tig + e;
      if (R >= nrow) continue;
      const int q = R / 3, st = R - q * 3;
      double* orow = a.out + st * sst + (size_t)(row0 + q) * a.ldo + a.out_off + n0 + gid;
      const bool s2 = (MODE == SPMM_S2STEP) && st == 0;
      const double alpha = s2 ? -a.gamma : 1.0, beta = s2 ? 1.0 : 0.0;
      const double* us = s_u + (MODE == SPMM_S2STEP ? (lrow0 + qo + q) * ust : 0) + n0 + gid;
      if (full) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int hm = 0; hm < 2; ++hm) {
            const int o = mt * 16 + hm * 8;
            const double u = (MODE == SPMM_S2STEP) ? us[o] : 0.0;
            __stcs(orow + o, fma(alpha, acc[mt][nt][hm * 2 + e], beta * u));
          }
      } else {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int hm = 0; hm < 2; ++hm) {
            const int o = mt * 16 + hm * 8, c = n0 + gid + o;
            if (c < r) {
              const double u = (MODE == SPMM_S2STEP) ? us[o] : 0.0;
              __stcs(orow + o, fma(alpha, acc[mt][nt][hm * 2 + e], beta * u));
            } else if (c == r && (r & 1) && a.out_sstride) {
              __stcs(orow + o, 0.0);        // zero pad column of the (even-padded) Ucat block
            }
          }
      }
    }
  }
}

template <int MODE, int GM>
__device__ __forceinline__ void block_store(const SpmmArgs& a, int r, int c, int row0, int gs,
                                            const double (&acc)[GM][Nacc<MODE>::v]) {
  if (c >= r) return;
#pragma unroll
  for (int q = 0; q < GM; ++q) {
    if (q < gs) {
      const size_t row = (size_t)(row0 + q);
      double* orow = a.out + row * a.ldo + a.out_off;
      const long long sst = a.out_sstride ? a.out_sstride : r;
      if (MODE != SPMM_SINGLE && MODE != SPMM_DENSE && a.out_sstride && (r & 1) && c + 1 == r) {
        __stcs(orow + r, 0.0); __stcs(orow + sst + r, 0.0); __stcs(orow + 2 * sst + r, 0.0);
      }
      if constexpr (MODE == SPMM_S2STEP) {
        const double uk = __ldg(a.U + row * a.ldu + c);
        __stcs(orow + c, fma(-a.gamma, acc[q][0], uk));
        __stcs(orow + sst + c, acc[q][1]);
        __stcs(orow + 2 * sst + c, acc[q][2]);
      } else if constexpr (MODE == SPMM_PLAIN3) {
        __stcs(orow + c, acc[q][0]);
        __stcs(orow + sst + c, acc[q][1]);
        __stcs(orow + 2 * sst + c, acc[q][2]);
      } else {
        __stcs(orow + c, acc[q][0]);
      }
    }
  }
}

template <int MODE, int GM>
__device__ __forceinline__ void zero_acc(double (&acc)[GM][Nacc<MODE>::v]) {
#pragma unroll
  for (int q = 0; q < GM; ++q)
#pragma unroll
    for (int t = 0; t < Nacc<MODE>::v; ++t) acc[q][t] = 0.0;
}

template <int MODE, int GM>
__global__ void __launch_bounds__(kThreads, 2)
spmm_kernel(SpmmArgs a, int ust) {
  const int r = a.d_r ? *a.d_r : a.r_fixed;
  if (r <= 0) return;
  constexpr int NV = Nstage<MODE>::v;
  constexpr int NACC = Nacc<MODE>::v;
  extern __shared__ double smem_dyn[];
  constexpr bool HOT = (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3);
  double* s_v = smem_dyn;                                     // [kValCap]
  double* s_u = smem_dyn + kValCap;                           // [kUCap][ust]   (HOT modes)
  int* s_col = reinterpret_cast<int*>(smem_dyn + kValCap + (HOT ? kUCap * ust : 0));   // [kSpmmCap]
  __shared__ int s_desc[kDescInts];
  __shared__ int s_bstart[kGroupMax + 1], s_vbase[kGroupMax], s_cbase[kGroupMax];
  __shared__ int s_L[kGroupMax], s_g[kGroupMax], s_js[kGroupMax], s_row0[kGroupMax];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int CT = (r + 31) >> 5;                               // 32-column slices

  double cs = 1.0;
  if constexpr (MODE == SPMM_SINGLE)
    cs = a.gen ? 1.0 : ((a.single_t == 2 || a.single_t == 3) ? a.rho : (a.single_t == 5 ? a.lam : 1.0));

  // one coalesced load of the tile's packed descriptor
  const int t = a.tlist ? a.tlist[blockIdx.x] : blockIdx.x;
  for (int i = tid; i < kDescInts; i += kThreads) s_desc[i] = __ldg(a.tdesc + (size_t)t * kDescInts + i);
  __syncthreads();
  const int e0 = s_desc[0], tot = s_desc[1], nb = s_desc[2];
  const int rbeg = s_desc[4], rend = s_desc[5];
  const unsigned short* s_lx = reinterpret_cast<const unsigned short*>(s_desc + kDescLidx);

  // staged path only if the whole tile fits the value stage (s_desc[6] = staged doubles at NV = 3);
  // a single block longer or taller than that takes the chunked long path below
  if (tot <= kSpmmCap && s_desc[6] <= kValCap) {
    if (tid == 0) {
      int vb = 0, cb = 0, eb = 0;
      for (int b = 0; b < nb; ++b) {
        const int g = s_desc[12 + b], L = s_desc[16 + b];
        s_bstart[b] = eb;
        s_row0[b] = s_desc[8 + b]; s_g[b] = g; s_L[b] = L;
        s_js[b] = row_pitch(L);
        s_vbase[b] = vb; s_cbase[b] = cb;
        vb += g * NV * s_js[b];
        cb += L;
        eb += g * L;
      }
      s_bstart[nb] = tot;
    }
    __syncthreads();
    const int nu = HOT ? s_desc[3] : 0;
    // ---- the tile's deduplicated U rows -> shared memory (cp.async, overlaps the value stream)
    if (HOT && nu > 0) {
      stage_u_rows(a, r, s_desc + kDescUrows, nu, s_u, ust, tid, kThreads);
      asm volatile("cp.async.commit_group;\n" ::);
    }
    // ---- stage: coalesced over the tile's contiguous nnz range.  Every thread first issues all the
    //      loads of its (<= kStg) entries, then combines and stores them, so the DRAM latency is
    //      paid once per tile rather than once per entry.
    constexpr int kStg = (kSpmmCap + kThreads - 1) / kThreads;
    constexpr int NRAW = (MODE == SPMM_SINGLE) ? 1 : 6;
    double raw[kStg][NRAW];
#pragma unroll
    for (int k = 0; k < kStg; ++k) {
      const int e = tid + k * kThreads;
      if (e < tot) {
        if constexpr (MODE == SPMM_SINGLE) {
          raw[k][0] = __ldcs(a.v[a.single_t] + e0 + e);
        } else {
#pragma unroll
          for (int v = 0; v < 6; ++v) raw[k][v] = __ldcs(a.v[v] + e0 + e);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kStg; ++k) {
      const int e = tid + k * kThreads;
      if (e < tot) {
        int b = 0;
#pragma unroll
        for (int kk = 1; kk < kGroupMax; ++kk) b += (kk < nb && e >= s_bstart[kk]);
        const int L = s_L[b];
        const int rel = e - s_bstart[b];
        const int q = rel / L, j = rel - (rel / L) * L;
        const int lp = s_js[b];
        double* dst = s_v + s_vbase[b] + q * NV * lp + j;
        if constexpr (MODE == SPMM_SINGLE) {
          dst[0] = cs * raw[k][0];
        } else {
          dst[0] = fma(a.lam, raw[k][5], fma(a.rho, raw[k][3], raw[k][0]));   // A0 + rho Jrho + lam Jlam
          dst[lp] = raw[k][1] + raw[k][4];                                   // A1 + Jmu
          dst[2 * lp] = a.rho * raw[k][2];                                    // rho A2
        }
        if (q == 0 && !(HOT && nu > 0)) s_col[s_cbase[b] + j] = __ldcs(a.col_idx + e0 + e);
      }
    }
    if (HOT && nu > 0) asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    // ---- compute: one warp per (node block, 32-column slice)
    for (int task = warp; task < nb * CT; task += kWarps) {
      const int b = task / CT, ct = task - (task / CT) * CT;
      const int c = ct * 32 + lane;
      const int g = s_g[b];
      if constexpr (HOT) {
        for (int qo = 0; qo < g; qo += 5) {
          if (nu > 0)
            block_task_mma_smem<MODE>(a, r, ct * 32, s_row0[b] + qo, min(5, g - qo), qo, s_L[b], s_js[b],
                                      s_v + s_vbase[b], s_lx + s_cbase[b], s_u, ust, s_desc[20 + b], lane);
          else
            block_task_mma<MODE>(a, r, ct * 32, s_row0[b] + qo, min(5, g - qo), qo, s_L[b], s_js[b],
                                 s_v + s_vbase[b], s_col + s_cbase[b], lane);
        }
      } else {
        for (int qo = 0; qo < g; qo += GM) {
          const int gs = min(GM, g - qo);
          double acc[GM][NACC];
          zero_acc<MODE, GM>(acc);
          block_task<MODE, GM>(a, r, c, s_row0[b] + qo, gs, qo, s_L[b], s_js[b], s_v + s_vbase[b],
                               s_col + s_cbase[b], acc);
          block_store<MODE, GM>(a, r, c, s_row0[b] + qo, gs, acc);
        }
      }
    }
  } else {
    // ---- one block longer than the stage (generic long rows): chunks of its column list; the
    //      whole CTA stages, warp ct < CT accumulates column slice ct
    const int g = rend - rbeg;
    const int L = s_desc[16];
    const int jc = min(kSpmmCap, kValCap / (g * NV) - 16);   // row_pitch(jc) * g * NV <= kValCap
    for (int qo = 0; qo < g; qo += GM) {
      const int gs = min(GM, g - qo);
      double acc[GM][NACC];
      zero_acc<MODE, GM>(acc);
      for (int j0 = 0; j0 < L; j0 += jc) {
        const int jn = min(jc, L - j0);
        const int lp = row_pitch(jn);
        __syncthreads();
        for (int e = tid; e < g * jn; e += kThreads) {
          const int q = e / jn, j = e - (e / jn) * jn;
          stage_entry<MODE>(a, e0 + q * L + j0 + j, s_v + q * NV * lp + j, lp, cs);
          if (q == 0) s_col[j] = __ldcs(a.col_idx + e0 + j0 + j);
        }
        __syncthreads();
        if (warp < CT) block_task<MODE, GM>(a, r, warp * 32 + lane, rbeg + qo, gs, qo, jn, lp, s_v, s_col, acc);
      }
      if (warp < CT) block_store<MODE, GM>(a, r, warp * 32 + lane, rbeg + qo, gs, acc);
    }
  }
}


// Lean hot kernel (S2STEP / PLAIN3) for the shared-memory-U tiles only: same stages as the U path of
// spmm_kernel without the gather / scalar code, so it fits 3 CTAs per SM (registers and ~76 KB smem).
template <int MODE>
__global__ void __launch_bounds__(kThreads, 3)
spmm_u_kernel(SpmmArgs a, int ust) {
  const int r = a.d_r ? *a.d_r : a.r_fixed;
  if (r <= 0) return;
  extern __shared__ double smem_dyn[];
  double* s_v = smem_dyn;                        // [kValCap]
  double* s_u = smem_dyn + kValCap;              // [kUCap][ust]
  __shared__ __align__(16) int s_desc[kDescInts];
  __shared__ int s_bstart[kTileBlocks + 1], s_vbase[kTileBlocks], s_lp[kTileBlocks];
  __shared__ float s_invL[kTileBlocks];
  __shared__ __align__(8) unsigned long long ubar;   // U-row bulk copies (TMA) complete here
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool ubulk = a.u_aligned16 != 0;
  if (tid == 0 && ubulk) {
    mbar_init(&ubar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  const int CT = (r + 31) >> 5;
  // U tiles are stored first (tile = blockIdx.x); the value loads need only (e0, tot), fetched in
  // parallel with the descriptor, so they are issued before the descriptor arrives
  const int t = blockIdx.x;
  const int2 et = __ldg(reinterpret_cast<const int2*>(a.tile_ev) + t);
  const int e0 = et.x, tot = et.y;
  if (tid < kDescInts / 4)
    *reinterpret_cast<int4*>(s_desc + 4 * tid) = __ldg(reinterpret_cast<const int4*>(a.tdesc + (size_t)t * kDescInts) + tid);
  constexpr int kStg = (kSpmmCap + kThreads - 1) / kThreads;
  double raw[kStg][6];
#pragma unroll
  for (int k = 0; k < kStg; ++k) {
    const int e = tid + k * kThreads;
    if (e < tot) {
#pragma unroll
      for (int v = 0; v < 6; ++v) raw[k][v] = __ldcs(a.v[v] + e0 + e);
    } else {
#pragma unroll
      for (int v = 0; v < 6; ++v) raw[k][v] = 0.0;
    }
  }
  __syncthreads();
  const int nb = s_desc[2], nu = s_desc[3];
  if (ubulk) {
    // the tile's deduplicated U rows by TMA bulk copies (one per row, warp 0): this traffic stays off
    // the LSU path the value loads and the contraction's shared-memory loads share
    if (warp == 0) {
      const unsigned ubytes = (unsigned)((r + 1) >> 1) * 16u;
      const int nuc = nu;
      if (lane == 0) mbar_expect_tx(&ubar, ubytes * (unsigned)nuc);
      __syncwarp();
      for (int u = lane; u < nuc; u += 32)
        bulk_g2s(s_u + u * ust, a.U + (size_t)s_desc[kDescUrows + u] * a.ldu, ubytes, &ubar);
    }
  } else {
    stage_u_rows(a, r, s_desc + kDescUrows, nu, s_u, ust, tid, kThreads);
    asm volatile("cp.async.commit_group;\n" ::);
  }
  if (tid == 0) {
    int vb = 0, eb = 0;
    for (int b = 0; b < nb; ++b) {
      const int g = s_desc[12 + b], L = s_desc[16 + b];
      s_bstart[b] = eb; s_lp[b] = row_pitch(L); s_vbase[b] = vb; s_invL[b] = 1.0f / (float)L;
      vb += g * 3 * s_lp[b];
      eb += g * L;
    }
    s_bstart[nb] = tot;
  }
  __syncthreads();                               // block table
#pragma unroll
  for (int k = 0; k < kStg; ++k) {
    const int e = tid + k * kThreads;
    if (e < tot) {
      int b = 0;
#pragma unroll
      for (int kk = 1; kk < kTileBlocks; ++kk) b += (kk < nb && e >= s_bstart[kk]);
      const int L = s_desc[16 + b];
      const int rel = e - s_bstart[b];
      // q = rel / L exactly: (rel + 1/2) / L is >= 1/(2L) away from an integer, far above the
      // float rounding error for rel, L <= 1024
      const int q = __float2int_rz(((float)rel + 0.5f) * s_invL[b]), j = rel - q * L;
      const int lp = s_lp[b];
      double* dst = s_v + s_vbase[b] + q * 3 * lp + j;
      dst[0] = fma(a.lam, raw[k][5], fma(a.rho, raw[k][3], raw[k][0]));   // A0 + rho Jrho + lam Jlam
      dst[lp] = raw[k][1] + raw[k][4];                                   // A1 + Jmu
      dst[2 * lp] = a.rho * raw[k][2];                                    // rho A2
    }
  }
  // zero the staged entries L .. round4(L)-1 of every slot (the contraction runs in steps of 4)
  for (int b = 0; b < nb; ++b) {
    const int g = s_desc[12 + b], L = s_desc[16 + b], lp = s_lp[b];
    for (int i = tid; i < g * 3 * 4; i += kThreads) {
      const int j = L + (i & 3);
      if (j < ((L + 3) & ~3)) s_v[s_vbase[b] + (i >> 2) * lp + j] = 0.0;
    }
  }
  if (ubulk) mbar_wait(&ubar, 0);
  else asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  const unsigned short* lx = reinterpret_cast<const unsigned short*>(s_desc + kDescLidx);
  int cb = 0;
  for (int b = 0, task0 = 0; b < nb; ++b) {
    const int g = s_desc[12 + b], L = s_desc[16 + b];
    for (int ct = 0; ct < CT; ++ct, ++task0) {
      if ((task0 % kWarps) != warp) continue;
      const int lrow0 = s_desc[20 + b];
      for (int qo = 0; qo < g; qo += 5) {
        if (MODE == SPMM_S2STEP && lrow0 < 0)   // the block's own U rows are not staged (no diagonal)
          block_task_mma_smem<MODE>(a, r, ct * 32, s_desc[8 + b] + qo, min(5, g - qo), qo, L, s_lp[b],
                                    s_v + s_vbase[b], lx + cb, s_u, ust, lrow0, lane);
        else
          block_task_mma_fast<MODE>(a, r, ct * 32, s_desc[8 + b] + qo, min(5, g - qo), qo, L, s_lp[b],
                                    s_v + s_vbase[b], lx + cb, s_u, ust, lrow0, lane);
      }
    }
    cb += L;
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent TMA-fed hot kernel (S2STEP / PLAIN3), one CTA per SM, warp-specialised:
//   producer warp : per tile, by cp.async.bulk (completion on the stage's mbarrier): the tile's
//                   deduplicated U rows as a few contiguous row runs (a 2-deep ring) FIRST -- a U stage
//                   frees only when the tile two back is done, so this copy is the tile's critical
//                   path and must not queue behind value copies -- then the 1 KB tile record (block
//                   geometry + local U-row index per column-list entry) and the six raw value
//                   segments of the NEXT tile (a 3-deep ring used LRC_SPMM_RAW_AHEAD - 1 tiles ahead);
//   consumer warps: NG groups of kTCons warps; group g takes every NG-th tile of the CTA.  A warp
//                   owns (node block, 32-column slice) tasks; the 6 -> 3 value combination happens in
//                   the B-fragment loads (three LDS + two FMA per element, branch-free), the U
//                   fragments come from the staged rows, and the contraction runs on the fp64 tensor
//                   pipe (m16n8k4, transposed so the stores are full sectors).  A warp signals the
//                   stages' empty barriers when it is done with the tile; no CTA-wide barrier.
// ---------------------------------------------------------------------------------------------
#ifndef LRC_SPMM_RAW_STAGES
#define LRC_SPMM_RAW_STAGES 3
#endif
#ifndef LRC_SPMM_U_STAGES
#define LRC_SPMM_U_STAGES 2
#endif
constexpr int kTStages = LRC_SPMM_RAW_STAGES;   // raw value / record stages
constexpr int kUStages = LRC_SPMM_U_STAGES;     // U row stages
#ifndef LRC_SPMM_CONS
#define LRC_SPMM_CONS 12
#endif
#ifndef LRC_SPMM_PREFETCH
#define LRC_SPMM_PREFETCH 4
#endif
#ifndef LRC_SPMM_MT
#define LRC_SPMM_MT 2
#endif
constexpr int kTCons = LRC_SPMM_CONS;     // consumer warps (the operator of P:30-36)
constexpr int kTMt = LRC_SPMM_MT;         // 16-column m-tiles per consumer task (columns per task = 16 kTMt)
constexpr int kTConsGen = 8;              // consumer warps for general term lists (more registers)
constexpr int kRawStride = ((kTileNnz + 3 + 3) / 16) * 16 + 12;   // doubles per raw array per stage (>= kTileNnz + 3, == 12 mod 16)
static_assert(kRawStride >= kTileNnz + 3 && kRawStride % 16 == 12, "raw stage stride");
constexpr int kTUrowMax = kTileUrows;     // staged U rows per tile
constexpr int kTLdMax = 64;               // U leading dimension supported (r <= 64)
constexpr int kTPrefetch = LRC_SPMM_PREFETCH;   // raw values warmed into L2 this many tiles ahead (0: off)
#ifndef LRC_SPMM_NOPRED
#define LRC_SPMM_NOPRED 1
#endif
#ifndef LRC_SPMM_UPREFETCH
#define LRC_SPMM_UPREFETCH 0
#endif
constexpr int kTUPrefetch = LRC_SPMM_UPREFETCH;  // U row runs warmed into L2 this many tiles ahead (0: off)

// raw value stages for nT value arrays (3 up to six arrays, 2 beyond: shared memory)
__host__ __device__ __forceinline__ int tma_raw_stages(int nT) { return nT <= 6 ? kTStages : 2; }

constexpr int kTmaSmemMax = 232448 - 2048;      // opt-in dynamic shared memory granted to the TMA kernel
// dynamic shared memory of the TMA kernel for nT value arrays and U rows of leading dimension ldu
size_t tma_smem(int nT, int ldu = kTLdMax) {
  const int nsr = tma_raw_stages(nT);
  return sizeof(double) * ((size_t)nsr * nT * kRawStride + (size_t)kUStages * kTUrowMax * ldu) +
         sizeof(int) * (size_t)nsr * kRecInts;
}

// GEN = false: the operator of P:30-36 (six arrays, the three groups of DESIGN.md K1, fixed combination);
// GEN = true: a general term list: nT arrays, G groups, group g = sum of up to
// kGroupTerms arrays with coefficients, slots (row q, group g) = q G + g in NT n-tiles of 8.
// PAIR: the m index of an m-tile maps to U columns (2 gid, 2 gid + 1) instead of (gid, gid + 8), so a
// lane's two A-fragment elements, its S2 operand and its two outputs of a slot are one 16-byte access
// each (needs 16-byte aligned output rows; the host decides).
template <int MODE, bool GEN, int NT, int NCW_, int KCG = 4, bool PAIR = false>
__global__ void __launch_bounds__((NCW_ + 1) * 32, 1)
spmm_tma_kernel(SpmmArgs a) {
  // subsets batched in this pass (one read of the operator for several subsets' U)
  const int S = a.nsub > 1 ? a.nsub : 1;
  int rmax = 0;
  for (int q = 0; q < S; ++q) {
    const int* dr = S > 1 ? a.d_rs[q] : a.d_r;
    rmax = max(rmax, dr ? *dr : a.r_fixed);
  }
  if (rmax <= 0) return;
  extern __shared__ __align__(16) double smem_dyn[];
  const int nT = GEN ? a.T : 6;                   // value arrays
  const int nsr = tma_raw_stages(nT);             // raw value stages
  const int G = GEN ? a.G : 3;                    // output groups
  double* s_raw = smem_dyn;                                                   // [stage][nT][kRawStride]
  double* s_ub = s_raw + (size_t)nsr * nT * kRawStride;                       // [ustage][kTUrowMax * ldu]
  const int ldu_s = a.ldu;                        // U stage row stride (even, <= kTLdMax)
  int* s_rec = reinterpret_cast<int*>(s_ub + (size_t)kUStages * kTUrowMax * ldu_s);   // [stage][kRecInts]
  // raw/record stages per tile i (ring of kTStages), U stages per work item m = i * S + subset
  // (ring of kUStages)
  __shared__ __align__(8) unsigned long long full_r[kTStages], empty_r[kTStages], full_u[kUStages], empty_u[kUStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NCW = NCW_;
  const int ldu = a.ldu;
  int rsub[kMaxSub];                              // ranks of the subsets (read once)
#pragma unroll
  for (int q = 0; q < kMaxSub; ++q) {
    const int* dr = S > 1 ? a.d_rs[q] : a.d_r;
    rsub[q] = (q < S) ? (dr ? *dr : a.r_fixed) : 0;
  }
  const int CT = (rmax + 16 * kTMt - 1) / (16 * kTMt);
  const int tpt = kTileBlocks * CT;              // (virtual) tasks per work item: blocks x CT column slices
  if (tid == 0) {
    for (int q = 0; q < nsr; ++q) { mbar_init(&full_r[q], 1); mbar_init(&empty_r[q], NCW); }
    for (int q = 0; q < kUStages; ++q) { mbar_init(&full_u[q], 1); mbar_init(&empty_u[q], NCW); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int Gd = gridDim.x, ntl = a.ntl_u;
  const int nmine = ((int)blockIdx.x < ntl) ? (ntl - (int)blockIdx.x + Gd - 1) / Gd : 0;
  const int nwork = nmine * S;

  if (warp == NCW) {
    // ------------------------------------------------------------------------------- producer
    // work item m: first the U rows of m (stage m % kUStages, last used by item m - kUStages), then
    // the record + raw values of every tile up to two ahead of m's tile (stage last used by tile - 3).
    // The per-tile metadata (first nnz, nnz, U row runs; tmeta) of 32 consecutive tiles of this CTA
    // sits in registers (lane l: tile 32 b + l), loaded one batch ahead: no global-load latency on
    // the producer's per-tile path.
    int4 cur[kMetaInts / 4], nxt[kMetaInts / 4];
    auto load_batch = [&](int b, int4 (&dst)[kMetaInts / 4]) {
      const int j = 32 * b + lane;
      if (j < nmine) {
        const int4* src = reinterpret_cast<const int4*>(a.tmeta + (size_t)(blockIdx.x + j * Gd) * kMetaInts);
#pragma unroll
        for (int w = 0; w < kMetaInts / 4; ++w) dst[w] = __ldg(src + w);
      } else {
#pragma unroll
        for (int w = 0; w < kMetaInts / 4; ++w) dst[w] = make_int4(0, 0, 0, 0);
      }
    };
    int bcur = 0;
    load_batch(0, cur);
    load_batch(1, nxt);
    // word W of local tile j (j in the current or the next batch), broadcast from its lane
    auto meta = [&](int j, auto wc) -> int {
      constexpr int W = decltype(wc)::value;
      const int4 vc = cur[W / 4], vn = nxt[W / 4];
      const int xc = (W % 4 == 0) ? vc.x : (W % 4 == 1) ? vc.y : (W % 4 == 2) ? vc.z : vc.w;
      const int xn = (W % 4 == 0) ? vn.x : (W % 4 == 1) ? vn.y : (W % 4 == 2) ? vn.z : vn.w;
      return __shfl_sync(0xffffffffu, (j >> 5) == bcur ? xc : xn, j & 31);
    };
    using W0 = std::integral_constant<int, 0>;
    using W1 = std::integral_constant<int, 1>;
    using W2 = std::integral_constant<int, 2>;
    int ri = 0;                                   // next tile whose record + raw values are issued
    for (int m = 0; m < nwork; ++m) {
      const int i = m / S, q = m - i * S;
      if ((i >> 5) != bcur && q == 0) {           // next batch of metadata
#pragma unroll
        for (int w = 0; w < kMetaInts / 4; ++w) cur[w] = nxt[w];
        ++bcur;
        load_batch(bcur + 1, nxt);
      }
      // this lane's U row run (lanes 8 .. 8 + nrun - 1)
      const int nrun = meta(i, W2{});
      int rv[3 * kMetaRuns];
      rv[0] = meta(i, std::integral_constant<int, 4>{});  rv[1] = meta(i, std::integral_constant<int, 5>{});
      rv[2] = meta(i, std::integral_constant<int, 6>{});  rv[3] = meta(i, std::integral_constant<int, 7>{});
      rv[4] = meta(i, std::integral_constant<int, 8>{});  rv[5] = meta(i, std::integral_constant<int, 9>{});
      rv[6] = meta(i, std::integral_constant<int, 10>{}); rv[7] = meta(i, std::integral_constant<int, 11>{});
      rv[8] = meta(i, std::integral_constant<int, 12>{}); rv[9] = meta(i, std::integral_constant<int, 13>{});
      rv[10] = meta(i, std::integral_constant<int, 14>{}); rv[11] = meta(i, std::integral_constant<int, 15>{});
      const int myr = lane - 16;
      int rg = 0, rl = 0, rs = 0;
#pragma unroll
      for (int k = 0; k < kMetaRuns; ++k)
        if (myr == k && k < nrun) { rg = rv[3 * k]; rl = rv[3 * k + 1]; rs = rv[3 * k + 2]; }
      const int us = m % kUStages;
      // everything the copy needs is ready before the wait: the issue follows the stage's release at once
      unsigned ub = (unsigned)rl * (unsigned)ldu * 8u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ub += __shfl_xor_sync(0xffffffffu, ub, o);
      const double* Usrc0 = S > 1 ? a.Us[q] : a.U;
      double* udst = s_ub + (size_t)us * kTUrowMax * ldu_s + (size_t)rs * ldu;
      const double* usrc = Usrc0 + (size_t)rg * ldu;
      if (m >= kUStages) mbar_wait(&empty_u[us], ((m / kUStages) - 1) & 1);
      {
        if (lane == 0) mbar_expect_tx(&full_u[us], ub);
        __syncwarp();
        const double* Usrc = Usrc0;
        if (rl > 0) bulk_g2s(udst, usrc, (unsigned)rl * (unsigned)ldu * 8u, &full_u[us]);
        // warm the U row runs of a later tile into L2: the first touch of a U row (written evict-first
        // by the basis pass) is a DRAM read, and the U copy is the tile's critical path
        if (kTUPrefetch > 0 && i + kTUPrefetch < nmine) {
          const int ip = i + kTUPrefetch;
          const int nrp = meta(ip, W2{});
          int pv[2 * kMetaRuns];
          pv[0] = meta(ip, std::integral_constant<int, 4>{});  pv[1] = meta(ip, std::integral_constant<int, 5>{});
          pv[2] = meta(ip, std::integral_constant<int, 7>{});  pv[3] = meta(ip, std::integral_constant<int, 8>{});
          pv[4] = meta(ip, std::integral_constant<int, 10>{}); pv[5] = meta(ip, std::integral_constant<int, 11>{});
          pv[6] = meta(ip, std::integral_constant<int, 13>{}); pv[7] = meta(ip, std::integral_constant<int, 14>{});
          int pg = 0, pl = 0;
#pragma unroll
          for (int k = 0; k < kMetaRuns; ++k)
            if (myr == k && k < nrp) { pg = pv[2 * k]; pl = pv[2 * k + 1]; }
          if (pl > 0) bulk_prefetch_l2(Usrc + (size_t)pg * ldu, (unsigned)pl * (unsigned)ldu * 8u);
        }
      }
#ifndef LRC_SPMM_RAW_AHEAD
#define LRC_SPMM_RAW_AHEAD 2
#endif
      for (; ri < nmine && ri <= i + nsr - (nsr >= 3 ? LRC_SPMM_RAW_AHEAD : 1); ++ri) {   // at least one tile ahead
        const int tr = blockIdx.x + ri * Gd, sr = ri % nsr;
        const int e0 = meta(ri, W0{}), tot = meta(ri, W1{});
        int pe0 = 0, ptot = 0;
        if (kTPrefetch > 0 && ri + kTPrefetch < nmine) { pe0 = meta(ri + kTPrefetch, W0{}); ptot = meta(ri + kTPrefetch, W1{}); }
        if (ri >= nsr) mbar_wait(&empty_r[sr], ((ri / nsr) - 1) & 1);
        if (kTPrefetch > 0 && ptot > 0 && lane < nT) {   // warm L2 further ahead
          const int p0 = pe0 & ~1, p1 = (pe0 + ptot) & ~1;
          if (p1 > p0) bulk_prefetch_l2(a.v[lane] + p0, 8u * (unsigned)(p1 - p0));
        }
        const int e0a = e0 & ~1, end = e0 + tot, endc = end & ~1;
        double* raw = s_raw + (size_t)sr * nT * kRawStride;
        if (lane == 0) {
          if (end & 1)   // odd tail element: plain load (a bulk copy never reads past the tile)
            for (int v = 0; v < nT; ++v) raw[v * kRawStride + (end - 1 - e0a)] = __ldg(a.v[v] + end - 1);
          mbar_expect_tx(&full_r[sr], (unsigned)nT * 8u * (unsigned)(endc - e0a) + 4u * kRecInts);
        }
        __syncwarp();
        if (lane < nT) {
          if (endc > e0a) bulk_g2s(raw + lane * kRawStride, a.v[lane] + e0a, 8u * (unsigned)(endc - e0a), &full_r[sr]);
        } else if (lane == 8) {
          bulk_g2s(s_rec + sr * kRecInts, a.trec + (size_t)tr * kRecInts, 4u * kRecInts, &full_r[sr]);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------------------- consumers
  // the CTA's tasks form one sequence (work item m, task) = m * tpt + task, dealt round-robin to the
  // consumer warps; a task is one (node block, 32-column slice) of a work item; the virtual tasks
  // (fewer than 4 blocks, or columns past this subset's rank) only arrive on the stage barriers
  const int gid = lane >> 2, tig = lane & 3;
  // Every warp walks all work items in order and waits on every stage phase (a warp that skipped an
  // item could see a stage's barrier two phases behind and take the stale parity for a completed one);
  // it arrives once per item on the U stage's empty barrier and once per tile on the raw stage's.
  // lane constants of the operator of P:30-36: slot nt*8 + gid = 3 q + group st combines the arrays
  // (A0, Jrho, Jlam) / (A1, Jmu) / (A2) with the coefficients (1, rho, lam) / (1, 1) / (rho)
  int lc_ao[2][3];
  double lc_co[2][3];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int slot = nt * 8 + gid, st = slot - (slot / 3) * 3;
    lc_ao[nt][0] = (st == 0 ? 0 : (st == 1 ? 1 : 2)) * kRawStride;
    lc_ao[nt][1] = (st == 0 ? 3 : (st == 1 ? 4 : 2)) * kRawStride;
    lc_ao[nt][2] = (st == 0 ? 5 : (st == 1 ? 4 : 2)) * kRawStride;
    lc_co[nt][0] = st == 2 ? a.rho : 1.0;
    lc_co[nt][1] = st == 0 ? a.rho : (st == 1 ? 1.0 : 0.0);
    lc_co[nt][2] = st == 0 ? a.lam : 0.0;
  }
  // item counters kept incrementally (no per-item divisions): tile i, subset q, raw stage sr and its
  // phase pr, U stage us and its phase pu, rot = (m * tpt) mod NCW
  int i = 0, q = 0, sr = 0, us = 0, rot = 0;
  unsigned pr = 0, pu = 0;
  for (int m = 0; m < nwork; ++m) {
    mbar_wait(&full_r[sr], pr);
    mbar_wait(&full_u[us], pu);
    for (int task = warp - rot + (warp < rot ? NCW : 0); task < tpt; task += NCW) {
    const int* R = s_rec + sr * kRecInts;
    const double* raw = s_raw + (size_t)sr * nT * kRawStride;
    const double* su = s_ub + (size_t)us * kTUrowMax * ldu_s;
    int r = rsub[0];
#pragma unroll
    for (int k = 1; k < kMaxSub; ++k) if (q == k) r = rsub[k];
    const double* Uq = S > 1 ? a.Us[q] : a.U;
    double* outq = S > 1 ? a.outs[q] : a.out;
    const long long sst = a.out_sstride ? a.out_sstride : r;
    const int nb = R[2];
    const int off = R[0] & 1;                      // the stage starts at the even element before e0
    // CT <= 2 for 32-column tasks (r <= 64): no integer division on the task path
    const int b = (kTMt == 2) ? (CT == 2 ? task >> 1 : task) : task / CT;
    const int n0 = (task - b * CT) * (16 * kTMt);
    if (b < nb && n0 < r) {
      const int row0 = R[4 + b], g = R[8 + b], L = R[12 + b], cb = kRecHdr + R[16 + b], nbase = R[20 + b];
      const int lrow0 = R[24 + b];
      // B operand (staged values, combined in the load): slot = nt*8 + gid -> (row q, group st);
      // KC arrays per group with coefficients (legacy: the fixed combination of P:30-36)
      constexpr int KC = GEN ? KCG : 3;
      int po[NT][KC];
      double co[NT][KC];
      bool sv[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int slot = nt * 8 + gid, q = slot / G, st = slot - q * G;
        sv[nt] = q < g;
        const int o = off + nbase + (sv[nt] ? q * L : 0) + tig;
        if constexpr (GEN) {
          const int gs = sv[nt] ? st : 0;
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const bool on = k < a.gl_n[gs];
            po[nt][k] = (on ? a.gl_t[gs][k] : 0) * kRawStride + o;
            co[nt][k] = on ? a.gl_c[gs][k] : 0.0;
          }
        } else {
          // the lane's arrays and coefficients were fixed at kernel start (lc_ao, lc_co)
#pragma unroll
          for (int k = 0; k < 3; ++k) { po[nt][k] = lc_ao[nt < 2 ? nt : 0][k] + o; co[nt][k] = lc_co[nt < 2 ? nt : 0][k]; }
        }
      }
      // A operand (U^T): columns n0 + mt*16 + gid (+8), entry j = k0 + tig -> staged U row R[cb + j]
      int cc[kTMt][2];
      bool vv[kTMt][2];
#pragma unroll
      for (int mt = 0; mt < kTMt; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          cc[mt][h] = PAIR ? n0 + 16 * mt + 2 * gid + h : n0 + gid + 16 * mt + 8 * h;
          vv[mt][h] = cc[mt][h] < r;
        }
      const int jmax = L - 1;
      double acc[kTMt][NT][4];
#pragma unroll
      for (int mt = 0; mt < kTMt; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.0;
      const int L4 = (L + 3) & ~3;
#define LRC_TMA_STEP(U_OFF, K0)                                                           \
  {                                                                                  \
    const int k0 = (K0);                                                             \
    const double* u = su + (U_OFF);                                                  \
        double xf[kTMt][2];                                                         \
_Pragma("unroll")                                                                   \
        for (int mt = 0; mt < kTMt; ++mt) {                                         \
          if constexpr (PAIR && LRC_SPMM_NOPRED) {                                  \
            /* no column predicate: an A element of a column >= r only reaches accumulator rows   \
               that are never stored, and the read stays inside the dynamic shared memory */     \
            const double2 t2 = *reinterpret_cast<const double2*>(u + cc[mt][0]);    \
            xf[mt][0] = t2.x;                                                       \
            xf[mt][1] = t2.y;                                                       \
          } else if constexpr (PAIR) {                                              \
            const double2 t2 = vv[mt][0] ? *reinterpret_cast<const double2*>(u + cc[mt][0]) \
                                         : make_double2(0.0, 0.0);                  \
            xf[mt][0] = t2.x;                                                       \
            xf[mt][1] = vv[mt][1] ? t2.y : 0.0;                                     \
          } else {                                                                  \
            xf[mt][0] = vv[mt][0] ? u[cc[mt][0]] : 0.0;                             \
            xf[mt][1] = vv[mt][1] ? u[cc[mt][1]] : 0.0;                             \
          }                                                                         \
        }                                                                           \
        const bool jv = k0 + tig < L;                                               \
        double bv[NT];                                                              \
_Pragma("unroll")                                                                   \
        for (int nt = 0; nt < NT; ++nt) {                                           \
          double v = co[nt][0] * raw[po[nt][0] + k0];                               \
_Pragma("unroll")                                                                   \
          for (int k = 1; k < KC; ++k) v = fma(co[nt][k], raw[po[nt][k] + k0], v);  \
          /* an absent slot (sv false) only feeds output columns that are never stored */        \
          bv[nt] = (jv && (sv[nt] || (PAIR && LRC_SPMM_NOPRED))) ? v : 0.0;         \
        }                                                                           \
_Pragma("unroll")                                                                   \
        for (int nt = 0; nt < NT; ++nt) {                                           \
_Pragma("unroll")                                                                   \
          for (int mt = 0; mt < kTMt; ++mt) dmma1684(acc[mt][nt], xf[mt][0], xf[mt][1], bv[nt]); \
        }                                                                           \
  }
      if (L4 <= 48) {
        // node blocks of <= 12 k4 steps (interior FE nodes: L = 45): this lane's staged U row offset of
        // every step first, so no step waits on an index load before its U fragment loads
        int uo[12];
#pragma unroll
        for (int t = 0; t < 12; ++t) uo[t] = R[cb + min(4 * t + tig, jmax)] * ldu;
#pragma unroll
        for (int t = 0; t < 12; ++t) {
          if (4 * t >= L4) break;
          LRC_TMA_STEP(uo[t], 4 * t)
        }
      } else {
#pragma unroll 2
        for (int kk = 0; kk < L4; kk += 4) LRC_TMA_STEP(R[cb + min(kk + tig, jmax)] * ldu, kk)
      }
#undef LRC_TMA_STEP
      // epilogue: frag (m, n) -> column n0 + mt*16 + gid (+8), slot nt*8 + 2 tig + e = G q + group
      const bool full_cols = n0 + 16 * kTMt <= r;
      const int s2g = GEN ? a.id_group : 0;       // the identity-diagonal group carries U - g W
      if constexpr (PAIR) {
        // paired mapping: the 64-bit bases and the per-m-tile column predicates are formed once per
        // task; a slot (nt, e) then costs one select, one 32-bit offset and the 16-byte accesses
        double* ob = outq + ((long long)row0 * a.ldo + a.out_off + n0 + 2 * gid);
        const double* ubs = (lrow0 >= 0) ? su + lrow0 * ldu + n0 + 2 * gid
                                         : Uq + ((size_t)row0 * ldu + n0 + 2 * gid);
        bool ok[kTMt], two[kTMt];
#pragma unroll
        for (int mt = 0; mt < kTMt; ++mt) {
          const int c = n0 + 2 * gid + 16 * mt;
          ok[mt] = full_cols || c < r;
          two[mt] = full_cols || c + 1 < r;
        }
        const bool padz = a.out_sstride != 0;     // (even-padded Ucat block) zero pad column of an odd r
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int Rs = nt * 8 + 2 * tig + e;
            if (Rs >= G * g) continue;
            const int q = Rs / G, st = Rs - q * G;
            double* orow = ob + ((long long)st * sst + q * a.ldo);
            const bool s2 = (MODE == SPMM_S2STEP) && st == s2g;
            const double* us_ = ubs + q * ldu;
#pragma unroll
            for (int mt = 0; mt < kTMt; ++mt) {
              if (ok[mt]) {
                double v0 = acc[mt][nt][e], v1 = acc[mt][nt][2 + e];
                if (s2) {
                  const double2 uu = *reinterpret_cast<const double2*>(us_ + 16 * mt);
                  v0 = fma(-a.gamma, v0, uu.x);
                  v1 = fma(-a.gamma, v1, uu.y);
                }
                if (two[mt] || padz) __stcs(reinterpret_cast<double2*>(orow + 16 * mt), make_double2(v0, two[mt] ? v1 : 0.0));
                else __stcs(orow + 16 * mt, v0);
              }
            }
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < (PAIR ? 0 : NT); ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int Rs = nt * 8 + 2 * tig + e;
          if (Rs >= G * g) continue;
          const int q = Rs / G, st = Rs - q * G;
          const size_t row = (size_t)(row0 + q);
          const bool s2 = (MODE == SPMM_S2STEP) && st == s2g;
          double* orow = outq + st * sst + row * a.ldo + a.out_off + n0 + gid;
          // the block's own U row (S2 epilogue) from the staged rows when present
          const double* us_ = (lrow0 >= 0) ? su + (size_t)(lrow0 + q) * ldu + n0 + gid : Uq + row * ldu + n0 + gid;
#pragma unroll
          for (int mt = 0; mt < kTMt; ++mt)
#pragma unroll
            for (int hm = 0; hm < 2; ++hm) {
              const int o = mt * 16 + hm * 8, c = n0 + gid + o;
              if (full_cols || c < r) {
                double v = acc[mt][nt][hm * 2 + e];
                if (s2) v = fma(-a.gamma, v, us_[o]);
                __stcs(orow + o, v);
              } else if (c == r && (r & 1) && a.out_sstride) {
                __stcs(orow + o, 0.0);        // zero pad column of the (even-padded) Ucat block
              }
            }
        }
      }
    }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty_u[us]);
      if (q == S - 1) mbar_arrive(&empty_r[sr]);
    }
    rot += tpt;
    while (rot >= NCW) rot -= NCW;
    if (++us == kUStages) { us = 0; pu ^= 1u; }
    if (++q == S) {
      q = 0; ++i;
      if (++sr == nsr) { sr = 0; pr ^= 1u; }
    }
  }
}

// Config-5 dense application Y = sum_t c_t A_t S diag(e_t) (S dense M x ncols, ncols <= 256) on the
// fp64 tensor pipe, shared-memory-U tiles.  Per tile the six value streams are combined once into
// the three grouped streams; S is then processed in 64-column chunks: the chunk of the tile's
// deduplicated S rows is staged (16-byte cp.async), every warp contracts one (node block, 32-column
// half) exactly like the hot kernel (transposed m16n8k4, D = S_chunk^T Vals^T) and combines the three
// streams of D in registers (five quad shuffles) into Y[row][c] = D[c][3q] + d_mu[c] D[c][3q+1] +
// d_nu[c] D[c][3q+2].  The m rows (gid, gid + 8) of an m-tile map to the adjacent columns
// (2 gid, 2 gid + 1): one 16-byte A-fragment load per m-tile and k4 step, one 16-byte store per
// output row and m-tile (128-byte row segments per warp store).  No D slab: ~75 KB of shared memory per CTA.
constexpr int kDenseChunk = 64;
constexpr int kDenseUst = kDenseChunk + 4;          // == 4 mod 16 doubles

template <int MODE>
__global__ void __launch_bounds__(kThreads, 3)
spmm_dense_kernel(SpmmArgs a) {
  const int ncols = a.r_fixed;
  extern __shared__ __align__(16) double smem_dyn[];
  double* s_v = smem_dyn;                                     // [kValCap]
  double* s_u = s_v + kValCap;                                // [kUCap][kDenseUst] (+32 slack)
  __shared__ __align__(16) int s_desc[kDescInts];
  __shared__ int s_bstart[kTileBlocks + 1], s_vbase[kTileBlocks], s_lp[kTileBlocks];
  __shared__ float s_invL[kTileBlocks];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int t = blockIdx.x;
  const int2 et = __ldg(reinterpret_cast<const int2*>(a.tile_ev) + t);
  const int e0 = et.x, tot = et.y;
  if (tid < kDescInts / 4)
    *reinterpret_cast<int4*>(s_desc + 4 * tid) = __ldg(reinterpret_cast<const int4*>(a.tdesc + (size_t)t * kDescInts) + tid);
  constexpr int kStg = (kSpmmCap + kThreads - 1) / kThreads;
  double raw[kStg][6];
#pragma unroll
  for (int k = 0; k < kStg; ++k) {
    const int e = tid + k * kThreads;
    if (e < tot) {
#pragma unroll
      for (int v = 0; v < 6; ++v) raw[k][v] = __ldcs(a.v[v] + e0 + e);
    } else {
#pragma unroll
      for (int v = 0; v < 6; ++v) raw[k][v] = 0.0;
    }
  }
  __syncthreads();
  const int nb = s_desc[2], nu = s_desc[3];
  if (tid == 0) {
    int vb = 0, eb = 0;
    for (int b = 0; b < nb; ++b) {
      const int g = s_desc[12 + b], L = s_desc[16 + b];
      s_bstart[b] = eb; s_lp[b] = row_pitch(L); s_vbase[b] = vb; s_invL[b] = 1.0f / (float)L;
      vb += g * 3 * s_lp[b];
      eb += g * L;
    }
    s_bstart[nb] = tot;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kStg; ++k) {
    const int e = tid + k * kThreads;
    if (e < tot) {
      int b = 0;
#pragma unroll
      for (int kk = 1; kk < kTileBlocks; ++kk) b += (kk < nb && e >= s_bstart[kk]);
      const int L = s_desc[16 + b];
      const int rel = e - s_bstart[b];
      const int q = __float2int_rz(((float)rel + 0.5f) * s_invL[b]), j = rel - q * L;
      const int lp = s_lp[b];
      double* dst = s_v + s_vbase[b] + q * 3 * lp + j;
      dst[0] = fma(a.lam, raw[k][5], fma(a.rho, raw[k][3], raw[k][0]));   // A0 + rho Jrho + lam Jlam
      dst[lp] = raw[k][1] + raw[k][4];                                   // A1 + Jmu
      dst[2 * lp] = a.rho * raw[k][2];                                    // rho A2
    }
  }
  for (int b = 0; b < nb; ++b) {
    const int g = s_desc[12 + b], L = s_desc[16 + b], lp = s_lp[b];
    for (int i = tid; i < g * 3 * 4; i += kThreads) {
      const int j = L + (i & 3);
      if (j < ((L + 3) & ~3)) s_v[s_vbase[b] + (i >> 2) * lp + j] = 0.0;
    }
  }
  const unsigned short* lx = reinterpret_cast<const unsigned short*>(s_desc + kDescLidx);
  for (int c0 = 0; c0 < ncols; c0 += kDenseChunk) {
    const int cw = min(kDenseChunk, ncols - c0);
    __syncthreads();   // previous chunk fully consumed (and the staged values visible)
    if (a.u_aligned16) {
      const int nch = (cw + 1) >> 1;
      for (int u = warp; u < nu; u += kWarps) {
        const double* src = a.U + (size_t)s_desc[kDescUrows + u] * a.ldu + c0;
        for (int ch = lane; ch < nch; ch += 32) cp_async16(s_u + u * kDenseUst + 2 * ch, src + 2 * ch);
      }
    } else {
      for (int u = warp; u < nu; u += kWarps) {
        const double* src = a.U + (size_t)s_desc[kDescUrows + u] * a.ldu + c0;
        for (int c = lane; c < cw; c += 32) cp_async8(s_u + u * kDenseUst + c, src + c);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    const int CT = (cw + 31) >> 5;
    int cb = 0, bprev = 0;
    for (int task = warp; task < nb * CT; task += kWarps) {
      const int b = task / CT, ct = task - (task / CT) * CT;
      for (; bprev < b; ++bprev) cb += s_desc[16 + bprev];
      const int g = s_desc[12 + b], L = s_desc[16 + b], lp = s_lp[b];
      const int n0 = ct * 32;
      const double dm_lo = 0.0;
      (void)dm_lo;
      for (int qo = 0; qo < g; qo += 5) {
        const int gs = min(5, g - qo);
        double acc[2][2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = acc[mt][nt][2] = acc[mt][nt][3] = 0.0;
        const int L4 = (L + 3) & ~3;
        const double* vb = s_v + s_vbase[b] + (qo * 3 + gid) * lp + tig;
        const double* ub = s_u + n0 + 2 * gid;     // paired columns: m rows (gid, gid + 8) <-> columns (2 gid, 2 gid + 1)
        const unsigned short* lc = lx + cb + tig;
        const int lmax = L - 1 - tig;
#pragma unroll 2
        for (int k0 = 0; k0 < L4; k0 += 4) {
          const double b0 = vb[k0], b1 = vb[8 * lp + k0];
          const double* urow = ub + (int)lc[min(k0, lmax)] * kDenseUst;
          const double2 p0 = *reinterpret_cast<const double2*>(urow), p1 = *reinterpret_cast<const double2*>(urow + 16);
          dmma1684(acc[0][0], p0.x, p0.y, b0);
          dmma1684(acc[0][1], p0.x, p0.y, b1);
          dmma1684(acc[1][0], p1.x, p1.y, b0);
          dmma1684(acc[1][1], p1.x, p1.y, b1);
        }
        // Y[row q][c] = D[c][3q] + d_mu[c] D[c][3q+1] + d_nu[c] D[c][3q+2].  Lane (gid, t) holds, per
        // column c = n0 + mt*16 + 2 gid + hm, slots v0 = 2t, v1 = 2t+1, v2 = 8+2t, v3 = 9+2t; each of the
        // five outputs of a quad needs exactly one slot of another lane of the quad (five shuffles):
        //   q0 = t0 (0, 1 | 2 from t1)    q1 = t2 (3 from t1 | 4, 5)    q2 = t3 (6, 7 | 8 from t0)
        //   q3 = t1 (9 from t0 | 10, 11)  q4 = t2 (12, 13 | 14 from t3)
        // The two columns (hm = 0, 1) of a lane are adjacent: one 16-byte store per output row.
        const int base = lane & ~3;
        const int rowq = s_desc[8 + b] + qo;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          double ya[2] = {0.0, 0.0}, yb[2] = {0.0, 0.0};   // row A (every lane), row B (tig == 2: q4)
          const int cl = n0 + mt * 16 + 2 * gid;
          const int c = c0 + cl;
          double dmv[2] = {0.0, 0.0}, dnv[2] = {0.0, 0.0};
          if (cl < cw) { dmv[0] = __ldg(a.dmu + c); dnv[0] = __ldg(a.dnu + c); }
          if (cl + 1 < cw) { dmv[1] = __ldg(a.dmu + c + 1); dnv[1] = __ldg(a.dnu + c + 1); }
#pragma unroll
          for (int hm = 0; hm < 2; ++hm) {
            const double v0 = acc[mt][0][hm * 2], v1 = acc[mt][0][hm * 2 + 1];
            const double v2 = acc[mt][1][hm * 2], v3 = acc[mt][1][hm * 2 + 1];
            const double x1v0 = __shfl_sync(0xffffffffu, v0, base + 1);
            const double x1v1 = __shfl_sync(0xffffffffu, v1, base + 1);
            const double x0v2 = __shfl_sync(0xffffffffu, v2, base + 0);
            const double x0v3 = __shfl_sync(0xffffffffu, v3, base + 0);
            const double x3v2 = __shfl_sync(0xffffffffu, v2, base + 3);
            const double dm = dmv[hm], dn = dnv[hm];
            if (tig == 0) ya[hm] = fma(dn, x1v0, fma(dm, v1, v0));
            else if (tig == 1) ya[hm] = fma(dn, v3, fma(dm, v2, x0v3));
            else if (tig == 2) { ya[hm] = fma(dn, v1, fma(dm, v0, x1v1)); yb[hm] = fma(dn, x3v2, fma(dm, v3, v2)); }
            else ya[hm] = fma(dn, x0v2, fma(dm, v1, v0));
          }
          if (cl >= cw) continue;
          const int qa = tig == 0 ? 0 : (tig == 1 ? 3 : (tig == 2 ? 1 : 2));
          double* oc = a.out + a.out_off + c;
          const bool two = cl + 1 < cw;
          if (qa < gs) {
            double* o = oc + (size_t)(rowq + qa) * a.ldo;
            if (two && a.o_pair) __stcs(reinterpret_cast<double2*>(o), make_double2(ya[0], ya[1]));
            else { __stcs(o, ya[0]); if (two) __stcs(o + 1, ya[1]); }
          }
          if (tig == 2 && 4 < gs) {
            double* o = oc + (size_t)(rowq + 4) * a.ldo;
            if (two && a.o_pair) __stcs(reinterpret_cast<double2*>(o), make_double2(yb[0], yb[1]));
            else { __stcs(o, yb[0]); if (two) __stcs(o + 1, yb[1]); }
          }
        }
      }
    }
  }
}
int ust_for(int rmax) { return ((rmax + 11) / 16) * 16 + 4; }   // >= rmax + 1, == 4 mod 16 (even)

size_t dense_smem() {
  return sizeof(double) * (kValCap + (size_t)kUCap * kDenseUst + 32);
}

size_t smem_for(int mode, int rmax) {
  const bool hot = (mode == SPMM_S2STEP || mode == SPMM_PLAIN3);
  return sizeof(double) * (kValCap + (hot ? (size_t)kUCap * ust_for(rmax) : 0)) + sizeof(int) * kSpmmCap;
}


int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

bool tma_ok(const SpmmArgs& a, int rmax) {
  bool al = a.trec != nullptr && a.tmeta != nullptr && rmax <= kTLdMax && a.ldu <= kTLdMax && (a.ldu % 2 == 0) &&
            a.nsub <= kMaxSub && tma_smem(a.gen ? a.T : 6, a.ldu) <= (size_t)kTmaSmemMax;
  for (int q = 0; q < max(1, a.nsub); ++q) {
    const double* u = a.nsub > 1 ? a.Us[q] : a.U;
    al = al && ((reinterpret_cast<uintptr_t>(u) & 15) == 0);
  }
  for (int v = 0; v < (a.gen ? a.T : 6); ++v) al = al && ((reinterpret_cast<uintptr_t>(a.v[v]) & 15) == 0);
  return al;
}

// 16-byte output accesses of the PAIR column mapping: even row stride / offsets, aligned bases, and a
// group stride known to be even on the host
bool tma_pair_ok(const SpmmArgs& a) {
#ifdef LRC_SPMM_NOPAIR
  return false;
#endif
  bool ok = !a.gen && (a.ldo % 2 == 0) && (a.out_off % 2 == 0);
  if (a.out_sstride) ok = ok && (a.out_sstride % 2 == 0);
  else ok = ok && a.nsub <= 1 && a.d_r == nullptr && (a.r_fixed % 2 == 0);
  for (int q = 0; q < max(1, a.nsub); ++q) {
    const double* o = a.nsub > 1 ? a.outs[q] : a.out;
    ok = ok && ((reinterpret_cast<uintptr_t>(o) & 15) == 0);
  }
  return ok;
}

template <int MODE>
cudaError_t launch_m(const SpmmArgs& a0, int rmax, cudaStream_t s) {
  SpmmArgs a = a0;
  // 16-byte U row copies need 16-byte aligned rows and room for the padding element of an odd r
  a.u_aligned16 = ((reinterpret_cast<uintptr_t>(a.U) & 15) == 0) && (a.ldu % 2 == 0) && (rmax < a.ldu || rmax % 2 == 0);
  a.o_pair = ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0) && (a.ldo % 2 == 0) && (a.out_off % 2 == 0);
  constexpr bool HOT = (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3);
  if constexpr (HOT) {
    // slack: the predicate-free contraction reads up to 32*CT - 1 columns of the last staged U row
    const int ust = ust_for(rmax), slack = max(0, 32 * ((rmax + 31) / 32) - ust);
    const size_t sm_u = sizeof(double) * (kValCap + (size_t)kUCap * ust + slack);
    // persistent TMA-fed kernel: 16-byte aligned value arrays and U rows, tile records available
    if (tma_ok(a, rmax) && a.ntl_u > 0) {
      const int grid = min(a.ntl_u, max(1, sm_count() - max(0, a.reserved_sms)));
      if (!a.gen) {
        if (tma_pair_ok(a))
          spmm_tma_kernel<MODE, false, 2, kTCons, 4, true><<<grid, (kTCons + 1) * 32, tma_smem(6, a.ldu), s>>>(a);
        else
          spmm_tma_kernel<MODE, false, 2, kTCons><<<grid, (kTCons + 1) * 32, tma_smem(6, a.ldu), s>>>(a);
      } else {
        const int nt = (5 * a.G + 7) / 8;          // slots (row, group) of a node block in n-tiles of 8
        int kmax = 0;
        for (int g = 0; g < a.G; ++g) kmax = max(kmax, a.gl_n[g]);
        const int th = (kTConsGen + 1) * 32;
        const size_t sm = tma_smem(a.T, a.ldu);
        if (kmax <= 4) {
          if (nt <= 2) spmm_tma_kernel<MODE, true, 2, kTConsGen, 4><<<grid, th, sm, s>>>(a);
          else if (nt == 3) spmm_tma_kernel<MODE, true, 3, kTConsGen, 4><<<grid, th, sm, s>>>(a);
          else spmm_tma_kernel<MODE, true, 4, kTConsGen, 4><<<grid, th, sm, s>>>(a);
        } else {
          if (nt <= 2) spmm_tma_kernel<MODE, true, 2, kTConsGen, 6><<<grid, th, sm, s>>>(a);
          else if (nt == 3) spmm_tma_kernel<MODE, true, 3, kTConsGen, 6><<<grid, th, sm, s>>>(a);
          else spmm_tma_kernel<MODE, true, 4, kTConsGen, 6><<<grid, th, sm, s>>>(a);
        }
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      if (a.gen) return cudaSuccess;               // general term lists: TMA path only (host checks)
      if (a.ntl_g > 0) {
        a.tlist = a.tlist_g;
        for (int q = 0; q < max(1, a.nsub); ++q) {      // L2-gather tiles: one launch per subset
          SpmmArgs aq = a;
          if (a.nsub > 1) { aq.nsub = 1; aq.U = a.Us[q]; aq.out = a.outs[q]; aq.d_r = a.d_rs[q]; }
          spmm_kernel<MODE, 5><<<a.ntl_g, kThreads, smem_for(MODE, rmax), s>>>(aq, ust_for(rmax));
        }
      }
      return cudaGetLastError();
    }
    if (a.nsub > 1) {                              // no batched path: one pass per subset
      for (int q = 0; q < a.nsub; ++q) {
        SpmmArgs aq = a;
        aq.nsub = 1; aq.U = a.Us[q]; aq.out = a.outs[q]; aq.d_r = a.d_rs[q];
        cudaError_t e = launch_m<MODE>(aq, rmax, s);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    if (sm_u <= 75 * 1024) {                       // 3 CTAs / SM
      if (a.ntl_u > 0) {
        spmm_u_kernel<MODE><<<a.ntl_u, kThreads, sm_u, s>>>(a, ust);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
      }
      if (a.ntl_g > 0) {
        a.tlist = a.tlist_g;
        spmm_kernel<MODE, 5><<<a.ntl_g, kThreads, smem_for(MODE, rmax), s>>>(a, ust_for(rmax));
      }
      return cudaGetLastError();
    }
  }
  if constexpr (MODE == SPMM_DENSE) {
    // shared-memory-S tiles on the tensor pipe, L2-gather tiles on the general kernel
    if (a.ntl_u > 0) {
      a.u_aligned16 = ((reinterpret_cast<uintptr_t>(a.U) & 15) == 0) && (a.ldu % 2 == 0);
      spmm_dense_kernel<MODE><<<a.ntl_u, kThreads, dense_smem(), s>>>(a);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    if (a.ntl_g > 0) {
      a.tlist = a.tlist_g;
      spmm_kernel<MODE, 5><<<a.ntl_g, kThreads, smem_for(MODE, rmax), s>>>(a, ust_for(rmax));
    }
    return cudaGetLastError();
  }
  if (a.ntiles == 0) return cudaSuccess;
  a.tlist = nullptr;
  spmm_kernel<MODE, 5><<<a.ntiles, kThreads, smem_for(MODE, rmax), s>>>(a, ust_for(rmax));
  return cudaGetLastError();
}

template <int MODE>
cudaError_t prep_m() {
  cudaError_t e = cudaFuncSetAttribute(spmm_kernel<MODE, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_for(MODE, kMaxRank));
  if (e != cudaSuccess) return e;
  if constexpr (MODE == SPMM_DENSE) {
    e = cudaFuncSetAttribute(spmm_dense_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dense_smem());
    if (e != cudaSuccess) return e;
  }
  if constexpr (MODE == SPMM_S2STEP || MODE == SPMM_PLAIN3) {
    e = cudaFuncSetAttribute(spmm_u_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 75 * 1024);
    if (e != cudaSuccess) return e;
    const int mx = (int)std::min(std::max(tma_smem(6), tma_smem(kMaxT)), (size_t)kTmaSmemMax);
    e = cudaFuncSetAttribute(spmm_tma_kernel<MODE, false, 2, kTCons>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(spmm_tma_kernel<MODE, false, 2, kTCons, 4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e != cudaSuccess) return e;
#define LRC_TMA_ATTR(NT_, KC_)                                                                          \
    e = cudaFuncSetAttribute(spmm_tma_kernel<MODE, true, NT_, kTConsGen, KC_>,                          \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, mx);                           \
    if (e != cudaSuccess) return e;
    LRC_TMA_ATTR(2, 4) LRC_TMA_ATTR(3, 4) LRC_TMA_ATTR(4, 4) LRC_TMA_ATTR(2, 6) LRC_TMA_ATTR(3, 6) LRC_TMA_ATTR(4, 6)
#undef LRC_TMA_ATTR
    if (e != cudaSuccess) return e;
  }
  return e;
}

}  // namespace

// Kernel attributes are set once per process/device, outside any graph capture.
cudaError_t spmm_prepare() {
  cudaError_t e;
  if ((e = prep_m<SPMM_S2STEP>()) != cudaSuccess) return e;
  if ((e = prep_m<SPMM_PLAIN3>()) != cudaSuccess) return e;
  if ((e = prep_m<SPMM_SINGLE>()) != cudaSuccess) return e;
  return prep_m<SPMM_DENSE>();
}

cudaError_t launch_spmm(int mode, const SpmmArgs& a, int rmax, cudaStream_t s) {
  if (rmax > (mode == SPMM_DENSE ? 256 : kMaxRank)) return cudaErrorInvalidValue;
  switch (mode) {
    case SPMM_S2STEP: return launch_m<SPMM_S2STEP>(a, rmax, s);
    case SPMM_PLAIN3: return launch_m<SPMM_PLAIN3>(a, rmax, s);
    case SPMM_SINGLE: return launch_m<SPMM_SINGLE>(a, rmax, s);
    case SPMM_DENSE: return launch_m<SPMM_DENSE>(a, rmax, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lrc
