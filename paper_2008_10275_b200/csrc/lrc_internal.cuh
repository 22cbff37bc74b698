// Internal declarations shared by the liblrcheb translation units (kernels + C ABI driver).
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Independence").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lrc {

constexpr int kMaxRank = 128;    // rank_cap limit
constexpr int kMaxP = 128;       // max Gram width p = min(n, w)
constexpr int kMaxW = 256;       // max concatenation width w = r_B + 4 r
constexpr int kGroupMax = 8;     // rows per node block in the fused SpMM
constexpr int kSpmmCap = 1024;   // nnz staged per SpMM CTA tile
constexpr int kValCap = 3200;    // staged (combined, row-padded) doubles per SpMM tile
#ifndef LRC_TILE_BLOCKS
#define LRC_TILE_BLOCKS 4
#endif
constexpr int kTileBlocks = LRC_TILE_BLOCKS;   // node blocks per SpMM tile
constexpr int kUCap = 90;        // deduplicated U rows staged in shared memory per SpMM tile
// SpMM tile descriptor (int32 words): [0] e0 (first nnz) [1] tot (nnz) [2] nb (blocks) [3] nu (U rows
// staged; 0 = L2-gather tile) [4] rbeg [5] rend [6] staged doubles (3 streams, padded rows) [7] pad, [8+b] row0, [12+b] g, [16+b] L, [20+b] local U row of the block's
// first row (-1: not staged)
// (b < 4); [24 .. 24+kUCap) U row ids; [kDescLidx ..) uint16 local column indices of the blocks'
// column lists, concatenated (<= kLidxCap entries).
constexpr int kDescInts = 256;
constexpr int kDescUrows = 24;
constexpr int kDescLidx = kDescUrows + kUCap;                 // 114
constexpr int kLidxCap = 2 * (kDescInts - kDescLidx);         // 284
constexpr int kSigmaStride = 128;
// Tile record of the persistent TMA SpMM (int32 words, 1 KB, one per shared-memory-U tile, same order):
// [0] e0 [1] tot [2] nb [3] staged U rows, [4+b] row0, [8+b] g, [12+b] L, [16+b] offset of block b's
// column list in [kRecHdr ..), [20+b] first nnz of block b relative to e0, [24+b] local row of the
// block's first row among the staged U rows (-1: not staged) (b < 4); [kRecHdr ..) the blocks' column
// lists as local (staged) U row indices.
constexpr int kRecInts = 256;
constexpr int kRecHdr = 32;
constexpr int kRecCols = kRecInts - kRecHdr;
constexpr int kTileNnz = 225 * kTileBlocks;      // nnz per tile of the TMA kernel (interior FE node blocks: 5 rows x 45)
constexpr int kTileUrows = 15 * (kTileBlocks + 2);     // staged U rows per tile of the TMA kernel (3 grid rows x (blocks + 2) nodes x 5)
constexpr int kMetaInts = 16;      // per-tile metadata of the TMA kernel: e0, nnz, runs, 0, 4 x (first row,
constexpr int kMetaRuns = 4;       //   rows, local first row) of the staged U row runs

// ------------------------------------------------------------------------------------------
// a1: fused six-array CSR SpMM
// ------------------------------------------------------------------------------------------
enum SpmmMode { SPMM_S2STEP = 0, SPMM_PLAIN3 = 1, SPMM_SINGLE = 2, SPMM_DENSE = 3 };
constexpr int kMaxSub = 4;        // subsets per batched SpMM pass
constexpr int kMaxT = 8;          // value arrays of a general term list
constexpr int kMaxG = 6;          // right-diagonal groups of a general term list
constexpr int kGroupTerms = 6;    // arrays per group

struct SpmmArgs {
  int M;
  int ngroups;
  const int* group_ptr;     // [ngroups+1] first row of each node block
  int ntiles;
  const int* tdesc;         // [ntiles][kDescInts] packed tile descriptors (see spmm.cu)
  const int* tlist_u;       // tiles with shared-memory U rows (nu > 0): 0 .. ntl_u-1 (stored first)
  int ntl_u;
  const int* tile_ev;       // [ntiles][2] first nnz and nnz count of each tile
  const int* trec;          // [ntl_u][kRecInts] tile records of the TMA kernel (null: not available)
  const int* tmeta;         // [ntl_u][kMetaInts] first nnz, nnz and U row runs of the TMA kernel's tiles
  const int* tlist_g;       // L2-gather tiles (nu = 0)
  int ntl_g;
  const int* tlist;         // (set by the launcher) tile list, or null for all tiles
  int u_aligned16;          // (set by the launcher) U rows may be copied in 16-byte chunks
  int o_pair;               // (set by the launcher) output rows admit 16-byte stores at even columns
  const int* row_ptr;
  const int* col_idx;
  const double* v[kMaxT];   // value arrays: A0, A1, A2, Jrho, Jmu, Jlam (legacy) or the T arrays of a term list
  // general term list (gen != 0): T arrays, G output groups, group g = sum over
  // k < gl_n[g] of gl_c[g][k] * array gl_t[g][k]; id_group = the group with the identity diagonal
  int gen, T, G, id_group;
  int gl_n[kMaxG];
  int gl_t[kMaxG][kGroupTerms];
  double gl_c[kMaxG][kGroupTerms];
  double rho, lam;
  const double* U;          // M x r input (row-major, ld ldu)
  int ldu;
  const int* d_r;           // r = d_r ? *d_r : r_fixed   (device-resident rank)
  int r_fixed;
  double* out;              // outputs at out[t*out_sstride + row*ldo + out_off + c] (t = stream)
  int ldo;
  int out_off;
  long long out_sstride;    // element offset between the three output streams; 0 = r (interleaved)
  double gamma;             // S2STEP: out0 = U - gamma * W0
  int single_t;             // SINGLE: output c_t A_t U
  const double* dmu;        // DENSE: per-column scalings
  const double* dnu;
  int reserved_sms;         // persistent hot kernel: SMs left free (concurrent solves)
  // f1 batched application: nsub > 1 subsets' U factors in one pass over the operator (TMA kernel
  // only; same ldu / output layout for all); U / out / d_r above are then unused
  int nsub;
  const double* Us[kMaxSub];
  double* outs[kMaxSub];
  const int* d_rs[kMaxSub];
};
cudaError_t launch_spmm(int mode, const SpmmArgs& a, int rmax, cudaStream_t s);

// ------------------------------------------------------------------------------------------
// a3/a4/a6: tall-skinny DMMA kernels over the logical concatenation Ucat = [A | B]
// ------------------------------------------------------------------------------------------
// Logical concatenation Ucat = [block 0 | ... | block nb-1] of row-major M-row blocks; block width =
// w_fixed + (w_idx >= 0 ? rk[w_idx] : 0) (device-resident ranks).
struct UBlock { const double* p; int ld; int w_fixed; int w_idx; };
constexpr int kMaxUBlocks = 8;    // B_U | G <= 6 groups | U_{k-1}
struct UDesc { UBlock b[kMaxUBlocks]; int nb; int pad_even; };   // pad_even: every block's logical
                                                                   // width rounded up to even (the pad
                                                                   // column holds zeros / finite data
                                                                   // met by a zero row of T)

struct TsArgs {
  int M;
  UDesc u;
  const int* rk;            // device rank array (may be null if no *_idx is used)
  const double* T;          // w x p small right matrix (row-major, ld ldt)
  int ldt;
  const int* d_p;           // p = d_p ? *d_p : p_fixed
  int p_fixed;
  double* partials;         // GRAM: [gridDim.x][pmax*pmax]
  double* out;              // STORE: M x p (ld ldo)
  int ldo;
  int t_lower;              // T[c][i] == 0 for i > c (T1 = R_V^T): skip the zero blocks
  int t_upper;              // T[c][i] == 0 for c > i (T = R1^{-1}): skip the zero blocks
  double* yout;             // GRAM: optional copy of the X tile (M x pmax, ld ldy, columns >= p are 0)
  int ldy;
  int u16;                  // (set by launch_ts) all Ucat blocks 16-byte aligned with even ld/offsets
  int o16;                  // (set by launch_ts) STORE rows 16-byte aligned (even ldo)
};
// mode 0 = GRAM (partial X^T X, X = Ucat T), 1 = STORE (out = Ucat T)
cudaError_t launch_ts(int mode, const TsArgs& a, int pmax, int grid, cudaStream_t s);
int ts_pmax_for(int p);          // padded width used by the instantiations
int ts_grid_for(int M, int reserved = 0);   // persistent grid size (SM count minus reserved SMs)
// G = sum_b partials[b] (fixed order), full symmetric pmax x pmax
cudaError_t launch_gram_reduce(const double* partials, int nblocks, int pmax, double* G,
                               cudaStream_t s);

// ------------------------------------------------------------------------------------------
// a2/a5: small dense kernels (single CTA)
// ------------------------------------------------------------------------------------------
struct VBlock {
  const double* ptr; int ld;
  int w_fixed; int w_idx; int w_mul;   // width = w_idx>=0 ? w_mul*rk[w_idx] : w_fixed ... (see kernel)
  double scale;                        // block multiplier
  int diag;                            // -1: none, else the row of the right-diagonal table (G x n)
  int use_omega;                       // 0: scale, 1: scale*omega, 2: scale*(1-omega)
};
struct VDesc { VBlock b[kMaxUBlocks]; int nb; int pad_even; };   // pad_even: as UDesc (zero pad columns)

struct State {          // device-resident per-solve state
  int* rk;              // rank array, rk[j] = rank of X_{j-1} (j = 0..N+1)
  int* p;               // current Gram width p = min(n, w)
  int* w;               // current concatenation width
  int* flags;           // error bits (1: Cholesky failed after escalations, 2: NaN)
  int* esc;             // shift escalations
  int* sweeps;          // Jacobi sweeps (summed over calls)
  int* prevp;           // p of the previous core SVD (warm-start validity)
  double* sigma;        // [N][kSigmaStride]
  double* scal;         // scalar slots: [0] ||B||^2, [1] ||R||^2 residual
};

struct SmallBufs {
  double* Vcat_unused;
  double* T1;     // w x pmax   (R_V^T)
  double* QV;     // n x pmax   (Q_V[:, :p])
  double* G;      // pmax x pmax reduced Gram
  double* R1;     // pmax x pmax
  double* R1i;    // pmax x pmax (R1^{-1}, upper)
  double* Wz;     // pmax x ldZ  (W_r Sigma_r^{-1})
  double* Wv;     // pmax x ldZ  (W_r Sigma_r)
  double* W0;     // pmax x pmax (warm-start basis Q_V^T B_prev), null: warm start off
  double* Wfull;  // pmax x pmax (full right basis W of the core)
  double* Bprev;  // n x pmax    (Q_V W of the previous iteration)
  int ldT;        // = pmax
  int ldZ;        // = capp
};

// vside: build Vcat (n x w) from the descriptor, Householder QR, write T1 = R_V^T and Q_V.
cudaError_t launch_vside(const VDesc& d, int n, const double* dtab,
                         const double* omega, int k, State st, SmallBufs b, int wmax,
                         cudaStream_t s);
// chol1: R1 = chol(G + s1 I) (escalating), R1^{-1}
cudaError_t launch_chol1(State st, SmallBufs b, int pmax, int wmax, cudaStream_t s);
// chol2 + SVD: R2 = chol(G + s2 I), R = R2 R1, Jacobi SVD, rank rule, W_r Sigma_r^{-1}, V'
cudaError_t launch_chol2_svd(State st, SmallBufs b, int pmax, int wmax, int n, double tol,
                             int cap, int rank_slot, int sigma_row, double* Vout, int ldv,
                             cudaStream_t s);
// C (m x ncols) = A (m x k) B (k x ncols), m/k device-resident (d_m/d_k) or fixed; m_max bounds the grid
cudaError_t launch_tiny_gemm(const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                             int ncols, const int* d_m, int m_fixed, int m_max, const int* d_k,
                             int k_fixed, cudaStream_t s, int transA = 0);
// scal[slot] = trace(G) over p (for ||X||_F^2)
cudaError_t launch_trace(State st, const double* G, int pmax, int slot, cudaStream_t s);

// misc
cudaError_t launch_fill_int(int* p, int v, int n, cudaStream_t s);
struct PvalArgs { const double* v[kMaxT]; double e[kMaxT]; };
cudaError_t launch_form_pvals(const PvalArgs& pa, int T, long long nnz, double* p, cudaStream_t s);
cudaError_t launch_cheb_inner(int nb, int rows, int ncols, int ld, long long bs, const double* R, const double* Y,
                              const double* Zc, const double* Zp, double* Zout, double w, double g, int first,
                              const int* d_r, int r_fixed, cudaStream_t s);
cudaError_t launch_s2_update(int rows, int ncols, int ld, const double* U, int ldu, double* W, double g,
                             cudaStream_t s);
cudaError_t launch_copy_out(const double* src, int ld_src, double* dst, int ld_dst, int rows, int cols,
                            const int* d_rank, const int* flags, cudaStream_t s);
cudaError_t launch_zero_cols(double* X, int rows, int ld, const int* d_r, int r_fixed, int cols,
                             cudaStream_t s);

}  // namespace lrc
