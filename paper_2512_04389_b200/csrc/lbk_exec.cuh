// lbk_exec.cuh — persistent tile-DAG executor for the dense GETRF and panel
// solves of one dependency level.
//
// A diagonal block's LU (factorize.py:38-78) and every dense panel solve
// (GESSM factorize.py:98-109, TSTRF :112-130) are expanded on the host into
// 64x64-tile tasks with explicit dependencies (per-tile update chains, so
// the floating-point order is fixed and results are deterministic).  One
// launch per level runs all of them: each CTA pulls the next task index
// (host order is topological), waits for its dependency counter to reach
// zero, executes it, and decrements its successors' counters.  A task is
// only ever waited on after an earlier index was taken by a running CTA, so
// progress is guaranteed without co-residency assumptions.
//
// Tile kernels stage 64x64 tiles in shared memory and run compact blocked
// routines (16-column panels: one warp with shuffles for the LU panel, row /
// column-owning threads for triangular panels, all 256 threads for the
// trailing updates; DMMA for tile GEMMs).  Critical-chain pairs are fused
// (last update + LU of a diagonal tile, update + solve of the next panel tile).
//
// Mutable tiles may have been written by other SMs during the launch: every
// global read of tile data uses ld.global.cg (L2, bypassing the
// non-coherent L1).
//
// GETRF speculates "no row swap" and verifies the reference's pivot rule
// exactly (see lbk_dense.cuh): in-tile and below-tile |d_qc| before scaling
// feed bmax[c]; FINAL compares them with |u_cc| and colmax[c].

#pragma once

#include "lbk_common.cuh"
#include "lbk_dense.cuh"

namespace lbk {

#ifndef LBK_SPIN_NS
#define LBK_SPIN_NS 32  // back-off of a CTA waiting on its task's dependency counter
#endif

constexpr int XT = 64;          // tile edge
constexpr int XTP = XT + 1;     // padded smem column stride
constexpr int XS = XT + 4;      // DMMA operand stride
constexpr int XREG = XT * XS;   // one smem tile region (fits either stride)
constexpr int EXEC_SMEM = (3 * XREG + 4 * XT) * 8;
#ifdef LBK_ABSORB_TILES
#define LBK_ABSORB_TILES_ENABLED LBK_ABSORB_TILES
#else
#define LBK_ABSORB_TILES_ENABLED 0
#endif
static_assert(!LBK_ABSORB_TILES_ENABLED || GEMM_SMEM <= EXEC_SMEM, "absorbed DMMA SSSSM tiles run in the executor's shared memory");
constexpr int COLMAX_ROWS = 128;  // rows per colmax task (GETRF's first tile waits for a whole column of them)

enum XType : int8_t {
  X_COLMAX = 0,  // colmax / bmax / perm reset of column tile c of diagonal block a
  X_GETRF = 1,   // factor diagonal tile (k,k) of block a
  X_TRSM_L = 2,  // tile (r,k) <- tile U_kk^{-1}
  X_TRSM_U = 3,  // tile (k,c) <- L_kk^{-1} tile
  X_GEMM = 4,    // tile (r,c) -= tile(r,k) tile(k,c)
  X_FINAL = 5,   // pivot verdict of block a
  X_PG_DIAG = 6, // GESSM panel a (rows R_X): tile (r,c) <- L[R_r,R_r]^{-1} tile
  X_PG_UPD = 7,  // tile (r,c) -= L[R_r, R_k] tile(k,c)
  X_PT_DIAG = 8, // TSTRF panel a (cols C_X): tile (r,c) <- tile U[C_c,C_c]^{-1}
  X_PT_UPD = 9,  // tile (r,c) -= tile(r,k) U[C_k, C_c]
  X_BAND = 10,   // LU of an independent segment [d, d + k) of a banded FULL diagonal block a (r, c = bandwidths)
  X_GETRF_UPD = 11,  // tile (r,r) -= tile(r,k) tile(k,r), then its LU (the diagonal chain, fused)
  X_PG_FUSED = 12,   // GESSM: X_PG_UPD from step k into tile (r,c), then X_PG_DIAG of (r,c)
  X_PT_FUSED = 13,   // TSTRF: X_PT_UPD from step k into tile (r,c), then X_PT_DIAG of (r,c)
  X_NOP = 14,        // dependency marker (tile column / row of a diagonal factor complete)
  X_SSSSM = 15,      // DMMA SSSSM output tile a (index into the GemmItems) of the previous level (absorbed)
};

struct XTask {
  int8_t type;
  int8_t chain;  // X_GETRF / X_GETRF_UPD: 1: then also solve L(r+1, r) and U(r, r+1) (the next step's update
                 // operands); 2: then also solve L(r+1, r), releasing the other successors first
  int16_t r, c, k;
  int16_t pad1;  // chain == 2: successor entries released early (after the diagonal tile's LU);
                 // X_GEMM / X_PG_UPD / X_PT_UPD: number of consecutive steps k.. aggregated (0 / 1: one)
  int32_t a;     // block the task writes
  int32_t d;     // diagonal block (panel tasks), = a for GETRF tasks
  int32_t step;  // elimination step (error records)
};

struct XLevel {
  const XTask* tasks;
  const int32_t* succ_ptr;
  const int32_t* succ;  // (successor << 1) | phase
  int* deps;   // working dependency counters, two per task (phase 1, phase 2), reset per run
  int* head;   // task counter of this level
  int ntasks;
  const GemmItem* gitems;     // X_SSSSM tasks: the DMMA SSSSM items and their tasks
  const GemmTask* gtasks;
  unsigned long long* trace;  // optional: per task [dequeue, ready, done, phase 0..3, operands complete] in ns (globaltimer)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }


// 1/x on the critical path: MUFU approximation + two Newton steps (<= 1 ulp
// from the rounded quotient; the 1e-10 factor tolerance is untouched), the
// IEEE division only outside the normal range (0, inf, NaN, denormals).
__device__ __forceinline__ double rcp_nr(double x) {
  const double ax = fabs(x);
  if (!(ax >= 1e-300 && ax <= 1e300)) return 1.0 / x;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Branch-free 1/x: MUFU + two Newton steps; 0 -> +-inf, inf -> 0 like the
// IEEE division (a zero pivot is then caught by the pivot verdict as usual).
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  r = fabs(x) < 1e-300 ? copysign(__longlong_as_double(0x7ff0000000000000LL), x) : r;
  return isinf(x) ? copysign(0.0, x) : r;
}

// First column of executor tile t of diagonal block A (subtree-aligned boundaries, or
// uniform 64-column tiles when the plan recorded none); tile t spans [xo(t), xo(t + 1)).
__device__ __forceinline__ int xo(const DevPools& P, const BlockDev& A, int t) {
  return A.xtb1 ? __ldg(P.xtb + (A.xtb1 - 1) + t) : min(t * XT, A.nrows);
}

// Panel blocks: first compressed row (GESSM) / column (TSTRF) of chain tile t (lim = nR / nC).
__device__ __forceinline__ int xop(const DevPools& P, const BlockDev& A, int t, int lim) {
  return A.xtb1 ? __ldg(P.xtb + (A.xtb1 - 1) + t) : min(t * XT, lim);
}

// acc_c -= sum_k l[k] * B(k, c) for the columns c = c0, c0 + 4, ... < ce, three
// independent accumulation chains at a time.  Col(c) = address of column c of
// the target (row offset applied), Bk(c) = address of B(0, c) (k contiguous).
template <class TA, class TB>
__device__ __forceinline__ void trail16(const double (&l)[16], int c0, int ce, TA col, TB bk) {
#pragma unroll 1
  for (int c = c0; c < ce; c += 12) {
    const bool v1 = c + 4 < ce, v2 = c + 8 < ce;
    const double* b0 = bk(c);
    const double* b1 = bk(v1 ? c + 4 : c);
    const double* b2 = bk(v2 ? c + 8 : c);
    double a0 = *col(c), a1 = v1 ? *col(c + 4) : 0.0, a2 = v2 ? *col(c + 8) : 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(-l[k], b0[k], a0);
      a1 = fma(-l[k], b1[k], a1);
      a2 = fma(-l[k], b2[k], a2);
    }
    *col(c) = a0;
    if (v1) *col(c + 4) = a1;
    if (v2) *col(c + 8) = a2;
  }
}


#ifndef LBK_LATE_FLUSH
#define LBK_LATE_FLUSH 1  // colmax flush of GETRF / TRSM_L tiles after their successors are released
#endif

#ifndef LBK_TILE_DMMA
#define LBK_TILE_DMMA 0  // 1: trailing updates inside the tile LU / TRSM routines on DMMA (measured slower)
#endif

// C[r0 + i, c0 + j] -= sum_{k < 16} A[r0 + i + k * lda] * B[k + (c0 + j) * ldb]  (i < nr, j < nc; all in
// shared memory, column-major).  The rank-16 trailing update of the blocked tile routines on DMMA
// (m8n8k4): 8x8 output tiles dealt over the 8 warps, up to 8 tiles per warp with independent
// accumulators; operands outside the range read as zero.  Replaces ~200 FMAs and ~240 shared loads per
// thread (shared-memory bound) by <= 32 DMMAs per warp.  Callers fence with __syncthreads on both sides.
__device__ __noinline__ void mma_sub_k16(double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                                         int r0, int nr, int c0, int nc) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int tr = (nr + 7) >> 3, ntile = tr * ((nc + 7) >> 3);
  if (warp >= ntile) return;
  // this warp's tiles warp, warp + 8, ...: fragment offsets computed once (-1: outside the range)
  int oa[8], ob[8];
  int ti = warp % tr, tj = warp / tr;  // tile coordinates, advanced by 8 tiles per slot
  const int step_j = 8 / tr, step_i = 8 % tr;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = ti * 8 + g, j = tj * 8 + g;
    const bool live = warp + 8 * q < ntile;
    oa[q] = live && i < nr ? r0 + i + t * lda : -1;
    ob[q] = live && j < nc ? t + (c0 + j) * ldb : -1;
    ti += step_i;
    tj += step_j;
    if (ti >= tr) {
      ti -= tr;
      ++tj;
    }
  }
  double acc[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  const int nq = (ntile - warp + 7) >> 3;  // tiles of this warp (warp-uniform)
#pragma unroll
  for (int k4 = 0; k4 < 16; k4 += 4) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < nq) {
        const double a = oa[q] >= 0 ? A[oa[q] + k4 * lda] : 0.0;
        const double b = ob[q] >= 0 ? B[ob[q] + k4] : 0.0;
        dmma(acc[q][0], acc[q][1], a, b);
      }
    }
  }
  ti = warp % tr;
  tj = warp / tr;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < nq) {
      const int i = ti * 8 + g, j = tj * 8 + 2 * t;
      if (i < nr) {
        if (j < nc) C[r0 + i + (c0 + j) * ldc] -= acc[q][0];
        if (j + 1 < nc) C[r0 + i + (c0 + j + 1) * ldc] -= acc[q][1];
      }
    }
    ti += step_i;
    tj += step_j;
    if (ti >= tr) {
      ti -= tr;
      ++tj;
    }
  }
}


#ifndef LBK_TRSM_PB
#define LBK_TRSM_PB 16  // panel width of the tile triangular solves
#endif
#ifndef LBK_TRSM_4X4
#define LBK_TRSM_4X4 1  // their trailing updates in 4 x 4 register tiles
#endif

// C[r, c] -= sum_{k < PB} A[r, k] B[k, c] for rows [r0, r0 + R) x columns [c0, c0 + Cn) of
// 64-tiles in shared memory (column-major, XTP): A(r, k) = A[k * XTP + r], B(k, c) =
// B[c * XTP + k], C(r, c) = C[c * XTP + r].  4 x 4 register tiles (rows rg + i * RG:
// consecutive threads read consecutive rows; columns 4 cg + j: B loads broadcast within a
// warp), 8 shared loads per 16 FMA.
template <int PB>
__device__ __forceinline__ void trail_4x4(double* C, const double* A, const double* B, int r0, int R, int c0,
                                          int Cn) {
  const int RG = (R + 3) >> 2, CG = (Cn + 3) >> 2;
  for (int u = threadIdx.x; u < RG * CG; u += blockDim.x) {
    const int rg = u % RG, cb = c0 + 4 * (u / RG);
    int rr[4];
    double a[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rr[i] = rg + i * RG < R ? r0 + rg + i * RG : -1;
#pragma unroll
      for (int j = 0; j < 4; ++j) a[i][j] = (rr[i] >= 0 && cb + j < c0 + Cn) ? C[(cb + j) * XTP + rr[i]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < PB; ++k) {
      double l[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) l[i] = A[k * XTP + (rr[i] >= 0 ? rr[i] : 0)];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = B[min(cb + j, XT - 1) * XTP + k];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) a[i][j] = fma(-l[i], w[j], a[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (rr[i] >= 0 && cb + j < c0 + Cn) C[(cb + j) * XTP + rr[i]] = a[i][j];
  }
}

// X (smem, XTP) <- X U^{-1} for columns [0, nc); U upper in smem (XTP), rinv[j] =
// 1/u_jj.  Blocked by 16 columns: the panel solve needs no communication
// between rows (threads 0..63 own one row each), the trailing update runs on
// all 256 threads.  kCheck stages |x_rj| before scaling in Dd[j*XTP + r].
// Compact (rolled panel loop): the executor's code stays i-cache resident.
template <bool kCheck>
__device__ void tile_right_solve_blk(double* X, const double* U, const double* rinv, double* Dd, int nc) {
  const int tid = threadIdx.x;
  constexpr int PB = LBK_TRSM_PB;
  static_assert(PB == 16 || !LBK_TILE_DMMA, "the DMMA update is 16 deep");
#pragma unroll 1
  for (int pb = 0; pb < nc; pb += PB) {
    if (tid < XT) {
      const int r = tid;
      double x[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) x[i] = X[(pb + i) * XTP + r];
#pragma unroll
      for (int jj = 0; jj < PB; ++jj) {
        const int j = pb + jj;
        if (j < nc) {
          if (kCheck) Dd[j * XTP + r] = fabs(x[jj]);
          x[jj] *= rinv[j];
#pragma unroll
          for (int i = jj + 1; i < PB; ++i) x[i] = fma(-x[jj], U[(pb + i) * XTP + j], x[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) X[(pb + i) * XTP + r] = x[i];
    }
    __syncthreads();
    const int pe = pb + PB;
    if (pe >= nc) break;
#if LBK_TILE_DMMA
    mma_sub_k16(X, XTP, X + pb * XTP, XTP, U + pb, XTP, 0, XT, pe, nc - pe);
#elif LBK_TRSM_4X4
    trail_4x4<PB>(X, X + pb * XTP, U + pb, 0, XT, pe, nc - pe);
#else
    {
      static_assert(PB == 16, "trail16 is 16 deep");
      const int r = tid & (XT - 1);
      double l[PB];
#pragma unroll
      for (int k = 0; k < PB; ++k) l[k] = X[(pb + k) * XTP + r];
      trail16(l, pe + (tid >> 6), nc, [&](int c) { return X + c * XTP + r; },
              [&](int c) { return U + c * XTP + pb; });
    }
#endif
    __syncthreads();
  }
}

// X (smem, XTP) <- L^{-1} X for rows [0, nr); L unit lower in smem (XTP).  Thread
// c < 64 owns column c of the 16-row panel; the trailing rows on all 256 threads.
__device__ void tile_left_solve_blk(double* X, const double* Lm, int nr) {
  const int tid = threadIdx.x;
  constexpr int PB = LBK_TRSM_PB;
  static_assert(PB == 16 || !LBK_TILE_DMMA, "the DMMA update is 16 deep");
#pragma unroll 1
  for (int pb = 0; pb < nr; pb += PB) {
    if (tid < XT) {
      const int c = tid;
      double x[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) x[i] = X[c * XTP + pb + i];
#pragma unroll
      for (int k = 0; k < PB; ++k)
#pragma unroll
        for (int i = k + 1; i < PB; ++i) x[i] = fma(-Lm[(pb + k) * XTP + pb + i], x[k], x[i]);
#pragma unroll
      for (int i = 0; i < PB; ++i) X[c * XTP + pb + i] = x[i];
    }
    __syncthreads();
    const int pe = pb + PB;
    if (pe >= nr) break;
#if LBK_TILE_DMMA
    mma_sub_k16(X, XTP, Lm + pb * XTP, XTP, X + pb, XTP, pe, nr - pe, 0, XT);
#elif LBK_TRSM_4X4
    trail_4x4<PB>(X, Lm + pb * XTP, X + pb, pe, nr - pe, 0, XT);
#else
    {
      // X[r, c] -= sum_k L[r, pb + k] X[pb + k, c] for the R = nr - pe rows below
      // the panel: work units (row, group of 4 columns) dealt over all 256
      // threads (4 independent chains per unit)
      const int R = nr - pe;
#pragma unroll 1
      for (int e = tid; e < R * (XT / 4); e += blockDim.x) {
        const int r = pe + e % R, c0 = 4 * (e / R);
        double a4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) a4[j] = X[(c0 + j) * XTP + r];
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          const double l = Lm[(pb + k) * XTP + r];
#pragma unroll
          for (int j = 0; j < 4; ++j) a4[j] = fma(-l, X[(c0 + j) * XTP + pb + k], a4[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) X[(c0 + j) * XTP + r] = a4[j];
      }
    }
#endif
    __syncthreads();
  }
}


#ifndef LBK_PANEL4
#define LBK_PANEL4 0  // 1: tile-LU panels on 4 warps, 2 threads per row (measured slower)
#endif

// Panel [pb, pb + 16) of the n x n tile T (smem, XTP) factored by threads 0..127:
// thread (row r = t / 2, half h = t % 2) keeps the row's 16 panel entries in
// registers and updates the 8 columns of its half, plus column jj + 1 (the next
// multiplier's operand, so both threads of a pair hold it); the pivot row is
// published through a double-buffered shared row (prow[2][16]) and one 128-thread
// named barrier per column.  Same arithmetic per entry as the one-warp panel
// (l = d * rcp_nr(u), fma updates in column order), a quarter of its issue per warp.
__device__ __forceinline__ void bar_panel() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __noinline__ void panel16_4w(double* T, int pb, int n, double* Dd, double* prow) {
  constexpr int PB = 16;
  const int tid = threadIdx.x, r = tid >> 1, h = tid & 1;
  double x[PB];
#pragma unroll
  for (int i = 0; i < PB; ++i) x[i] = T[(pb + i) * XTP + r];
#pragma unroll
  for (int jj = 0; jj < PB; ++jj) {
    const int j = pb + jj;
    if (j >= n) break;
    double* pr = prow + (jj & 1) * PB;
    if (r == j) {  // the pivot row's pair publishes its current entries (column jj from both)
#pragma unroll
      for (int i = jj; i < PB; ++i)
        if (i == jj || (i >> 3) == h) pr[i] = x[i];
    }
    bar_panel();
    const double rinv = rcp_nr(pr[jj]);
    if (r > j && r < n) {
      const double d = x[jj];
      if (h == 0) Dd[j * XTP + r] = fabs(d);
      const double l = d * rinv;
      x[jj] = l;
#pragma unroll
      for (int i = jj + 1; i < PB; ++i)
        if ((i >> 3) == h || i == jj + 1) x[i] = fma(-l, pr[i], x[i]);
    }
  }
  if (r >= pb && r < n) {
#pragma unroll
    for (int i = 0; i < PB; ++i)
      if ((i >> 3) == h) T[(pb + i) * XTP + r] = x[i];
  }
}

// LU (no exchange) of the n x n (n <= 64) tile in smem T (column-major, XTP
// stride), blocked by 16-column panels.  Per panel: (1) the 64 x 16 panel is
// factored by threads 0..63 (thread r holds row r's 16 panel entries in
// registers; the pivot row is published to smem, one 64-thread named barrier
// per column); (2) U12 <- L11^{-1} A12 by one thread per trailing column;
// (3) A22 -= L21 U12 by all 256 threads.  Every column is scaled only after
// all updates from the columns left of it, so |d_rj| staged in Dd (r > j) is
// the value the reference's pivot search sees.  Ends with a CTA barrier.
#ifndef LBK_LU_PB
#define LBK_LU_PB 8  // panel width of the 64x64 tile LU (8: C2 167.3 -> 161.6 ms vs 16, profiles/r2_lu_pb_ab.txt)
#endif
#ifndef LBK_A22_4X4
#define LBK_A22_4X4 1  // trailing update of the tile LU in 4 x 4 register tiles
#endif
__device__ void tile_lu64_blocked(double* T, int n, double* Dd, double* urow, long long* prof = nullptr) {
  const int tid = threadIdx.x;
  constexpr int PB = LBK_LU_PB;
  static_assert(PB == 16 || (!LBK_PANEL4 && !LBK_TILE_DMMA), "the 4-warp panel and the DMMA update are 16 wide");
  long long t0 = prof ? clock64() : 0;
#pragma unroll 1
  for (int pb = 0; pb < n; pb += PB) {
#if LBK_PANEL4
    if (tid < 128) panel16_4w(T, pb, n, Dd, urow);
#else
    if (tid < 32) {
      // warp 0 holds rows lane and lane + 32 of the panel; the pivot row is
      // broadcast with shuffles (no barrier), every lane forms 1/u_jj itself
      const int lane = tid, ra = lane, rb = lane + 32;
      double pa[PB], pc[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        pa[i] = T[(pb + i) * XTP + ra];
        pc[i] = T[(pb + i) * XTP + rb];
      }
#pragma unroll
      for (int jj = 0; jj < PB; ++jj) {
        const int j = pb + jj;
        if (j < n) {
          const int src = j & 31;
          const bool hi = j >= 32;
          double u[PB];
#pragma unroll
          for (int i = jj; i < PB; ++i) u[i] = __shfl_sync(0xffffffffu, hi ? pc[i] : pa[i], src);
          const double rinv = rcp_nr(u[jj]);
          if (ra > j && ra < n) {
            const double d = pa[jj];
            Dd[j * XTP + ra] = fabs(d);
            const double l = d * rinv;
            pa[jj] = l;
#pragma unroll
            for (int i = jj + 1; i < PB; ++i) pa[i] = fma(-l, u[i], pa[i]);
          }
          if (rb > j && rb < n) {
            const double d = pc[jj];
            Dd[j * XTP + rb] = fabs(d);
            const double l = d * rinv;
            pc[jj] = l;
#pragma unroll
            for (int i = jj + 1; i < PB; ++i) pc[i] = fma(-l, u[i], pc[i]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < PB; ++i) {
        if (ra >= pb) T[(pb + i) * XTP + ra] = pa[i];
        if (rb >= pb) T[(pb + i) * XTP + rb] = pc[i];
      }
    }
#endif
    if (prof) { __syncthreads(); const long long t1 = clock64(); if (tid == 0) prof[0] += t1 - t0; t0 = t1; }
    __syncthreads();
    const int pe = min(n, pb + PB);
    if (pe >= n) break;
    // (2) U12: rows pb..pe-1 of trailing columns c >= pe, L11 unit lower
    if (prof) { __syncthreads(); const long long t1 = clock64(); if (tid == 0) prof[3] += t1 - t0; t0 = t1; }
    if (tid >= pe && tid < n) {
      const int c = tid;
      double x[PB];
#pragma unroll
      for (int i = 0; i < PB; ++i) x[i] = T[c * XTP + pb + i];
#pragma unroll
      for (int k = 0; k < PB; ++k)
#pragma unroll
        for (int i = k + 1; i < PB; ++i) x[i] = fma(-T[(pb + k) * XTP + pb + i], x[k], x[i]);
#pragma unroll
      for (int i = 0; i < PB; ++i) T[c * XTP + pb + i] = x[i];
    }
    __syncthreads();
    if (prof) { const long long t1 = clock64(); if (tid == 0) prof[1] += t1 - t0; t0 = t1; }
    // (3) A22 -= L21 U12 (tensor cores, or work units (row, group of 4 columns) dealt over all 256 threads)
#if LBK_TILE_DMMA
    mma_sub_k16(T, XTP, T + pb * XTP, XTP, T + pb, XTP, pe, n - pe, pe, n - pe);
#elif LBK_A22_4X4
    {
      // 4 x 4 register tiles: rows pe + rg + i * RG (consecutive threads -> consecutive rows:
      // conflict-free L / C accesses), columns pe + 4 cg + j (U loads broadcast in a warp);
      // 8 shared loads per 16 FMA instead of 5 per 4
      const int R = n - pe, RG = (R + 3) / 4, CG = (R + 3) / 4;
      if (tid < RG * CG) {
        const int rg = tid % RG, c0 = pe + 4 * (tid / RG);
        int rr[4];
        double a[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          rr[i] = pe + rg + i * RG;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            a[i][j] = (rr[i] < n && c0 + j < n) ? T[(c0 + j) * XTP + rr[i]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          double l[4], u[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) l[i] = T[(pb + k) * XTP + min(rr[i], XT - 1)];
#pragma unroll
          for (int j = 0; j < 4; ++j) u[j] = T[min(c0 + j, XT - 1) * XTP + pb + k];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[i][j] = fma(-l[i], u[j], a[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (rr[i] < n && c0 + j < n) T[(c0 + j) * XTP + rr[i]] = a[i][j];
      }
    }
#else
    {
      const int R = n - pe, CG = (n - pe + 3) / 4;
#pragma unroll 1
      for (int e = tid; e < R * CG; e += blockDim.x) {
        const int r = pe + e % R, c0 = pe + 4 * (e / R);
        double a4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) a4[j] = c0 + j < n ? T[(c0 + j) * XTP + r] : 0.0;
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          const double l = T[(pb + k) * XTP + r];
#pragma unroll
          for (int j = 0; j < 4; ++j) a4[j] = fma(-l, T[min(c0 + j, XT - 1) * XTP + pb + k], a4[j]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c0 + j < n) T[(c0 + j) * XTP + r] = a4[j];
      }
    }
#endif
    __syncthreads();
    if (prof) { const long long t1 = clock64(); if (tid == 0) prof[2] += t1 - t0; t0 = t1; }
  }
  __syncthreads();
}

#ifndef LBK_LU_LA
#define LBK_LU_LA 0  // 1: tile LU with a one-panel lookahead (measured slower: C2 118.5 -> 122.2 ms, profiles/r2_lu_la_ab.txt)
#endif

// Panel [pb, pe) (pe - pb <= 8) of the n x n tile T factored by warp 0 (the one-warp
// shuffle panel of tile_lu64_blocked, PB = 8).
__device__ __noinline__ void panel8_w0(double* T, int pb, int n, double* Dd) {
  constexpr int PB = 8;
  const int lane = threadIdx.x & 31, ra = lane, rb = lane + 32;
  double pa[PB], pc[PB];
#pragma unroll
  for (int i = 0; i < PB; ++i) {
    pa[i] = T[(pb + i) * XTP + ra];
    pc[i] = T[(pb + i) * XTP + rb];
  }
#pragma unroll
  for (int jj = 0; jj < PB; ++jj) {
    const int j = pb + jj;
    if (j < n) {
      const int src = j & 31;
      const bool hi = j >= 32;
      double u[PB];
#pragma unroll
      for (int i = jj; i < PB; ++i) u[i] = __shfl_sync(0xffffffffu, hi ? pc[i] : pa[i], src);
      const double rinv = rcp_nr(u[jj]);
      if (ra > j && ra < n) {
        const double d = pa[jj];
        Dd[j * XTP + ra] = fabs(d);
        const double l = d * rinv;
        pa[jj] = l;
#pragma unroll
        for (int i = jj + 1; i < PB; ++i) pa[i] = fma(-l, u[i], pa[i]);
      }
      if (rb > j && rb < n) {
        const double d = pc[jj];
        Dd[j * XTP + rb] = fabs(d);
        const double l = d * rinv;
        pc[jj] = l;
#pragma unroll
        for (int i = jj + 1; i < PB; ++i) pc[i] = fma(-l, u[i], pc[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < PB; ++i) {
    if (ra >= pb) T[(pb + i) * XTP + ra] = pa[i];
    if (rb >= pb) T[(pb + i) * XTP + rb] = pc[i];
  }
}

// LU of the n x n tile with a one-panel lookahead: after panel p (8 columns) is factored,
// warp 0 alone brings the NEXT panel's columns up to date (U12 rows + rank-8 update) and
// factors it right away, while warps 1-7 update the rest of the trailing matrix - the
// trailing update leaves the panel chain (one barrier per panel instead of three).  Every
// entry sees the same operations in the same order as tile_lu64_blocked (same fma
// sequence over k, same U12 substitution): bitwise identical factors, staged |d| included.
__device__ void tile_lu64_la(double* T, int n, double* Dd) {
  constexpr int PB = 8;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) panel8_w0(T, 0, n, Dd);
  __syncthreads();
#pragma unroll 1
  for (int pb = 0;; pb += PB) {
    const int pe = min(n, pb + PB);
    if (pe >= n) break;
    const int pe2 = min(n, pe + PB);
    if (tid < 32) {
      // U12 of the next panel's columns c in [pe, pe2): lanes 0..7, one column each
      if (lane < pe2 - pe) {
        const int c = pe + lane;
        double x[PB];
#pragma unroll
        for (int i = 0; i < PB; ++i) x[i] = T[c * XTP + pb + i];
#pragma unroll
        for (int k = 0; k < PB; ++k)
#pragma unroll
          for (int i = k + 1; i < PB; ++i) x[i] = fma(-T[(pb + k) * XTP + pb + i], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < PB; ++i) T[c * XTP + pb + i] = x[i];
      }
      __syncwarp();
      // rank-8 update of those columns, rows >= pe: lane owns rows pe + lane and pe + lane + 32
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = pe + lane + 32 * h;
        if (r < n) {
          double l[PB];
#pragma unroll
          for (int k = 0; k < PB; ++k) l[k] = T[(pb + k) * XTP + r];
#pragma unroll
          for (int j = 0; j < PB; ++j) {
            const int c = pe + j;
            if (c < pe2) {
              double a = T[c * XTP + r];
#pragma unroll
              for (int k = 0; k < PB; ++k) a = fma(-l[k], T[c * XTP + pb + k], a);
              T[c * XTP + r] = a;
            }
          }
        }
      }
      __syncwarp();
      panel8_w0(T, pe, n, Dd);
    } else {
      const int t2 = tid - 32, nt2 = blockDim.x - 32;
      // U12 of the remaining columns [pe2, n)
      for (int c = pe2 + t2; c < n; c += nt2) {
        double x[PB];
#pragma unroll
        for (int i = 0; i < PB; ++i) x[i] = T[c * XTP + pb + i];
#pragma unroll
        for (int k = 0; k < PB; ++k)
#pragma unroll
          for (int i = k + 1; i < PB; ++i) x[i] = fma(-T[(pb + k) * XTP + pb + i], x[k], x[i]);
#pragma unroll
        for (int i = 0; i < PB; ++i) T[c * XTP + pb + i] = x[i];
      }
      asm volatile("bar.sync 2, %0;" ::"r"(nt2) : "memory");
      // rows >= pe, columns >= pe2 in 4 x 4 register tiles
      const int R = n - pe, C = n - pe2, RG = (R + 3) / 4, CG = (C + 3) / 4;
      for (int u = t2; u < RG * CG; u += nt2) {
        const int rg = u % RG, c0 = pe2 + 4 * (u / RG);
        int rr[4];
        double a[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          rr[i] = pe + rg + i * RG;
#pragma unroll
          for (int j = 0; j < 4; ++j) a[i][j] = (rr[i] < n && c0 + j < n) ? T[(c0 + j) * XTP + rr[i]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < PB; ++k) {
          double l[4], w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) l[i] = T[(pb + k) * XTP + min(rr[i], XT - 1)];
#pragma unroll
          for (int j = 0; j < 4; ++j) w[j] = T[min(c0 + j, XT - 1) * XTP + pb + k];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) a[i][j] = fma(-l[i], w[j], a[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (rr[i] < n && c0 + j < n) T[(c0 + j) * XTP + rr[i]] = a[i][j];
      }
    }
    __syncthreads();
  }
}

// bmax[j] (global, bits) = max over rows r > j (r < nr) of the staged |d_rj|;
// rows_all: the whole column is "below" (TRSM_L tiles).
// Thread (column c = tid & 63, row quarter tid >> 6) reduces 16 independent
// smem reads, the 4 quarter maxima meet in `part` (256 doubles of scratch),
// one atomic per column: ~0.2 us instead of 8 serial shuffle reductions per warp.
__device__ __forceinline__ void flush_colmax(const double* Dd, int nr, int nc, bool rows_all,
                                             unsigned long long* bmax, double* part) {
  const int c = threadIdx.x & (XT - 1), q = threadIdx.x >> 6;
  double mx = 0.0;
  if (c < nc) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int rr = q * 16 + i;
      const double v = Dd[c * XTP + rr];
      if (rr < nr && (rows_all || rr > c)) mx = fmax(mx, v);
    }
  }
  part[q * XT + c] = mx;
  __syncthreads();
  if (threadIdx.x < nc) {
    const double m = fmax(fmax(part[c], part[XT + c]), fmax(part[2 * XT + c], part[3 * XT + c]));
    if (m > 0.0) atomic_max_nonneg(&bmax[c], m);
  }
}

// ---- smem staging -------------------------------------------------------------
// 64x64 tiles, 256 threads: thread owns row r = tid & 63 and columns (tid >> 6) + 4i,
// i < 16.  All 16 loads are issued before the first smem store (one L2 round trip
// per tile instead of one per element).
constexpr int XTHREADS = 256;
constexpr int XPER = XT * XT / XTHREADS;  // 16

// not inlined: ~20 call sites would otherwise put ~60 KB of address arithmetic
// into the executor (i-cache), for a routine that runs a few times per task
template <int STRIDE>
__device__ __noinline__ void stage_tile(double* T, const double* G, int ld, int nr, int nc,
                                           const int32_t* rg, const int32_t* cg) {
  const int r = threadIdx.x & (XT - 1), c0 = threadIdx.x >> 6;
  const bool rok = r < nr;
  const size_t roff = rok ? static_cast<size_t>(rg ? rg[r] : r) : 0;
  int cix[XPER];
#pragma unroll
  for (int i = 0; i < XPER; ++i) {
    const int c = c0 + 4 * i;
    cix[i] = (c < nc) ? (cg ? cg[c] : c) : -1;
  }
  double v[XPER];
#pragma unroll
  for (int i = 0; i < XPER; ++i) v[i] = (rok && cix[i] >= 0) ? ldcg(G + static_cast<size_t>(cix[i]) * ld + roff) : 0.0;
#pragma unroll
  for (int i = 0; i < XPER; ++i) T[(c0 + 4 * i) * STRIDE + r] = v[i];
}

// (nr x nc) tile, column-major global (ld), optional row/column gathers -> smem T[c*XTP + r]
__device__ __forceinline__ void load_tile(double* T, const double* G, int ld, int nr, int nc,
                                          const int32_t* rg = nullptr, const int32_t* cg = nullptr) {
  stage_tile<XTP>(T, G, ld, nr, nc, rg, cg);
}

// DMMA A operand ([k][r], stride XS) / B operand ([c][k], stride XS)
__device__ __forceinline__ void load_opA(double* As, const double* G, int ld, int nr, int nk,
                                         const int32_t* rg = nullptr, const int32_t* kg = nullptr) {
  stage_tile<XS>(As, G, ld, nr, nk, rg, kg);
}

__device__ __forceinline__ void load_opB(double* Bs, const double* G, int ld, int nk, int nc,
                                         const int32_t* kg = nullptr, const int32_t* cg = nullptr) {
  stage_tile<XS>(Bs, G, ld, nk, nc, kg, cg);
}

// target tile (registers via smem T0) -= A * B on DMMA, 64x64x64, 8 warps of 32x16
__device__ void tile_mma_sub(double* Cs, const double* As, const double* Bs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < XT; k += 4) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[(k + t) * XS + wm + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 2; ++j) b[j] = Bs[(wn + j * 8 + g) * XS + k + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = wm + i * 8 + g, c = wn + j * 8 + 2 * t;
      Cs[c * XTP + r] -= acc[i][j][0];
      Cs[(c + 1) * XTP + r] -= acc[i][j][1];
    }
  __syncthreads();
}

// C (smem, XTP stride) -> global, masked
__device__ __noinline__ void store_tile(double* G, int ld, const double* T, int nr, int nc) {
  const int r = threadIdx.x & (XT - 1), c0 = threadIdx.x >> 6;
  if (r >= nr) return;
#pragma unroll
  for (int i = 0; i < XPER; ++i) {
    const int c = c0 + 4 * i;
    if (c < nc) G[static_cast<size_t>(c) * ld + r] = T[c * XTP + r];
  }
}

// instrumented replays: phase stamps inside a task (thread 0, after a barrier)
__device__ __forceinline__ void stamp(unsigned long long* ph, int k) {
  if (ph) {
    __syncthreads();
    if (threadIdx.x == 0) ph[k] = gtimer();
  }
}

// ---- banded diagonal blocks -------------------------------------------------------
// A FULL diagonal block whose filled pattern lies inside a narrow band (lower
// bandwidth bl, upper bu <= 15: e.g. the bodies of bordered-block-diagonal
// matrices) needs no tile DAG: its LU never leaves the band, so one CTA sweeps
// the columns with the band staged in shared memory (diagonal storage,
// CHUNK columns at a time + the bw-column overlap), one barrier per column:
// thread (i, j) updates entry (k+i, k+j) of step k.  Pivot rule exactly as
// the tile path (factorize.py:38-78): colmax at entry over the band, |d_ik|
// before scaling staged per column, the verdict per chunk.  Rows outside the
// band are structural zeros, so they can neither be a pivot nor change colmax.
constexpr int BAND_MAX = 15;
constexpr int BAND_CH = 128;

static_assert(((BAND_CH + BAND_MAX) * (2 * BAND_MAX + 1) + 2 * BAND_CH * 16) * 8 <= EXEC_SMEM, "band smem");

// Narrow symmetric bands (bl = bu = B <= 4), one thread: the whole 5x5 active window of the
// elimination lives in that thread's registers (entry (r, c) in w[r % 5][c % 5],
// so nothing moves when the window slides; the column loop is unrolled by 5).
// Per column: one reciprocal, bl multipliers, a 4x4 fma update, the final U
// row and L column out to shared memory and the entering row / column in.
// The chain between columns is reciprocal -> multiply -> fma (no barrier, no
// shuffle), and the rest of the column's work overlaps it.  Same arithmetic as
// the barrier-stepped sweep below (l = d * rcp_fast(u), fma updates in column
// order), so the factors are identical.  Chunks of the segment are staged
// through shared memory by the whole CTA; the thread keeps its window across
// chunks, so a chunk only needs its columns plus the 5 the window reaches past it.

template <int B, int Q>
__device__ __forceinline__ void band_reg_col(double (&w)[5][5], double* base, double* Sv, int Wm1) {
  // base = &Bs(kk, kk); (kk, kk + j) at base + j * Wm1; (kk + i, kk) at base + i
  const double u = w[Q][Q];
  const double rinv = rcp_fast(u);
  base[0] = u;
#pragma unroll
  for (int j = 1; j <= B; ++j) base[j * Wm1] = w[Q][(Q + j) % 5];
  double below = 0.0;
#pragma unroll
  for (int i = 1; i <= B; ++i) {
    const double d = w[(Q + i) % 5][Q];
    const double l = d * rinv;
    const double ad = fabs(d);
    below = ad > below ? ad : below;  // = fmax (a NaN |d| is skipped), fewer instructions
    base[i] = l;
#pragma unroll
    for (int j = 1; j <= B; ++j) w[(Q + i) % 5][(Q + j) % 5] = fma(-l, w[Q][(Q + j) % 5], w[(Q + i) % 5][(Q + j) % 5]);
  }
  *Sv = below;
  // entering row kk + 5 (columns kk + 1 .. kk + 5) and column kk + 5 (rows kk + 1 .. kk + 4);
  // unpredicated: rows >= m and the columns past the staged chunk hold zeros
#pragma unroll
  for (int j = 1; j < 5; ++j)
    if (5 - j <= B) w[Q][(Q + j) % 5] = base[j * Wm1 + 5];
  w[Q][Q] = base[5 * Wm1 + 5];
#pragma unroll
  for (int i = 1; i < 5; ++i)
    if (5 - i <= B) w[(Q + i) % 5][Q] = base[5 * Wm1 + i];
}

template <int B>
__device__ __noinline__ void band_getrf_reg(const BlockDev& A, const DevPools& P, double* sm, int s0, int m, int step,
                                            double pivot_tol) {
  constexpr int W = 2 * B + 1, Wm1 = W - 1;
  const int ld = A.nrows, tid = threadIdx.x;
  constexpr int SMEM_D = EXEC_SMEM / 8;
  constexpr int CH = ((SMEM_D - 5 * W) / (W + 1)) / 5 * 5 < 1000 ? ((SMEM_D - 5 * W) / (W + 1)) / 5 * 5 : 1000;
  double* G = P.vals + A.ent + static_cast<size_t>(s0) * ld + s0;
  double* Bs = sm;                // (CH + 5) x W band values, (r, c) at (c - c0) * W + r - c + B
  double* S = sm + (CH + 5) * W;  // CH staged max |d| below the diagonal
  double* colmax = P.colmax + A.dg + s0;
  double w[5][5];
  for (int c0 = 0; c0 < m; c0 += CH) {
    const int ce = min(m, c0 + CH + 5), kend = min(m, c0 + CH);
    const int total = (ce - c0) * W;
    __syncthreads();
    // all loads of a batch in flight at once; slots past the segment are zero-filled
    for (int b = tid; b < (CH + 5) * W; b += 8 * XTHREADS) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = b + u * XTHREADS, c = c0 + idx / W, r = c - B + idx % W;
        v[u] = (idx < total && r >= 0 && r < m) ? ldcg(G + static_cast<size_t>(c) * ld + r) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b + u * XTHREADS < (CH + 5) * W) Bs[b + u * XTHREADS] = v[u];
    }
    __syncthreads();
    // column maxima of the columns whose band is still pristine in this chunk
    // (the sweep stores final U rows into columns [kend, ce))
    for (int c = (c0 == 0 ? 0 : c0 + 5) + tid; c < ce; c += blockDim.x) {
      double mx = 0.0;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const int r = c - B + q;
        if (r >= 0 && r < m) mx = fmax(mx, fabs(Bs[(c - c0) * W + q]));
      }
      colmax[c] = mx;
    }
    __syncthreads();
    if (tid == 0) {
      if (c0 == 0) {
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
          for (int c = 0; c < 5; ++c)
            w[r][c] = (c - r <= B && r - c <= B && r < m && c < ce) ? Bs[c * W + r - c + B] : 0.0;
      }
#pragma unroll 1
      for (int k = c0; k < kend; k += 5) {
        double* base = Bs + (k - c0) * W + B;
        band_reg_col<B, 0>(w, base, S + k - c0, Wm1);
        if (k + 1 >= kend) break;
        band_reg_col<B, 1>(w, base + W, S + k + 1 - c0, Wm1);
        if (k + 2 >= kend) break;
        band_reg_col<B, 2>(w, base + 2 * W, S + k + 2 - c0, Wm1);
        if (k + 3 >= kend) break;
        band_reg_col<B, 3>(w, base + 3 * W, S + k + 3 - c0, Wm1);
        if (k + 4 >= kend) break;
        band_reg_col<B, 4>(w, base + 4 * W, S + k + 4 - c0, Wm1);
      }
    }
    __syncthreads();
    for (int k = c0 + tid; k < kend; k += blockDim.x) {
      const double uk = Bs[(k - c0) * W + B];
      const double below = S[k - c0];
      const double piv = fmax(fabs(uk), below);
      if (piv == 0.0 || piv < pivot_tol * colmax[k] || isnan(uk)) record(&P.err[0], step, s0 + k);
      else if (below > fabs(uk)) record(&P.err[1], step, s0 + k);
    }
    for (int idx = tid; idx < total; idx += blockDim.x) {
      const int c = c0 + idx / W, r = c - B + idx % W;
      if (r >= 0 && r < m) G[static_cast<size_t>(c) * ld + r] = Bs[idx];
    }
  }
}

// Segment [s0, s0 + m) of the block: independent of the rest of the block
// (no band entry crosses its ends), so it is factored on its own.
__device__ void band_getrf(const BlockDev& A, const DevPools& P, double* sm, int bl, int bu, int s0, int m, int step,
                           double pivot_tol) {
  const int ld = A.nrows, W = bl + bu + 1, bw = max(bl, bu), tid = threadIdx.x;
  double* G = P.vals + A.ent + static_cast<size_t>(s0) * ld + s0;
  double* Bs = sm;                                   // (BAND_CH + bw) x W band values
  double* S = sm + (BAND_CH + BAND_MAX) * (2 * BAND_MAX + 1);  // BAND_CH x 16 staged |d|
  double* Lc = S + BAND_CH * 16;                     // BAND_CH x 16 multipliers
  double* colmax = P.colmax + A.dg + s0;
  for (int c = tid; c < m; c += blockDim.x) {
    double mx = 0.0;
    const int r1 = min(m - 1, c + bl);
    for (int r = max(0, c - bu); r <= r1; ++r) mx = fmax(mx, fabs(ldcg(G + static_cast<size_t>(c) * ld + r)));
    colmax[c] = mx;
  }
  // band entry (r, c) -> Bs[(c - c0) * W + (r - c + bu)]
  const int i = tid >> 4, j = tid & 15;
  for (int c0 = 0; c0 < m; c0 += BAND_CH) {
    const int ce = min(m, c0 + BAND_CH + bw), kend = min(m, c0 + BAND_CH);
    __syncthreads();
    for (int idx = tid; idx < (ce - c0) * W; idx += blockDim.x) {
      const int c = c0 + idx / W, r = c - bu + idx % W;
      Bs[idx] = (r >= 0 && r < m) ? ldcg(G + static_cast<size_t>(c) * ld + r) : 0.0;
    }
    __syncthreads();
    if (bl * (bu + 1) <= 32) {
      // narrow band: the bl x (bu + 1) update pairs fit one warp (fixed lane ->
      // (i, j) map); steps only need a __syncwarp, the other warps wait
      if (tid < 32) {
        const int q = tid, ii = 1 + q / (bu + 1), jj = q % (bu + 1);
        const bool own = q < bl * (bu + 1);
#pragma unroll 1
        for (int k = c0; k < kend; ++k) {
          const double* colk = Bs + (k - c0) * W + bu;
          const double rinv = rcp_fast(colk[0]);
          if (own && k + ii < m) {
            const double d = colk[ii];
            const double l = d * rinv;
            if (jj == 0) {
              S[(k - c0) * 16 + ii] = fabs(d);
              Lc[(k - c0) * 16 + ii] = l;
            } else if (k + jj < m) {
              double* e = Bs + (k + jj - c0) * W + (ii - jj + bu);
              *e = fma(-l, Bs[(k + jj - c0) * W + (bu - jj)], *e);
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
    } else
    for (int k = c0; k < kend; ++k) {
      const double* colk = Bs + (k - c0) * W + bu;  // (k + i, k) = colk[i]
      const double u = colk[0];
      const bool act = i >= 1 && i <= bl && k + i < m;
      if (act) {
        const double d = colk[i];
        const double l = d * rcp_nr(u);
        if (j == 0) {
          S[(k - c0) * 16 + i] = fabs(d);
          Lc[(k - c0) * 16 + i] = l;
        } else if (j <= bu && k + j < m) {
          double* e = Bs + (k + j - c0) * W + (i - j + bu);  // (k + i, k + j)
          const double urow = Bs[(k + j - c0) * W + (bu - j)];  // (k, k + j)
          *e = fma(-l, urow, *e);
        }
      }
      __syncthreads();
    }
    // multipliers into the band, pivot verdict of the chunk's columns, write-back
    for (int idx = tid; idx < (kend - c0) * 16; idx += blockDim.x) {
      const int kk = idx >> 4, ii = idx & 15;
      if (ii >= 1 && ii <= bl && c0 + kk + ii < m) Bs[kk * W + bu + ii] = Lc[idx];
    }
    for (int k = c0 + tid; k < kend; k += blockDim.x) {
      const double uk = Bs[(k - c0) * W + bu];
      double below = 0.0;
      for (int ii = 1; ii <= bl && k + ii < m; ++ii) below = fmax(below, S[(k - c0) * 16 + ii]);
      const double piv = fmax(fabs(uk), below);
      if (piv == 0.0 || piv < pivot_tol * colmax[k] || isnan(uk)) record(&P.err[0], step, s0 + k);
      else if (below > fabs(uk)) record(&P.err[1], step, s0 + k);
    }
    __syncthreads();
    for (int idx = tid; idx < (ce - c0) * W; idx += blockDim.x) {
      const int c = c0 + idx / W, r = c - bu + idx % W;
      if (r >= 0 && r < m) G[static_cast<size_t>(c) * ld + r] = Bs[idx];
    }
  }
}

// Phase-2 dependencies: a task that loaded its target tile waits here for its operands.
// (trace: the time the operands were complete goes to slot 7 of the task's record)
__device__ __forceinline__ void wait_phase2(volatile int* d2, unsigned long long* ph = nullptr) {
  if (!d2) return;
  if (threadIdx.x == 0) {
    while (*d2 > 0) __nanosleep(LBK_SPIN_NS);
    __threadfence();
    if (ph) ph[4] = gtimer();
  }
  __syncthreads();
}

#ifndef LBK_ABSORB_TILES
#define LBK_ABSORB_TILES 0  // 1: executor runs absorbed DMMA SSSSM tiles (LBK_ABSORB=1 plans; measured slower)
#endif

// the DMMA SSSSM pipeline of an absorbed update tile (inlined: a call would spill)
__device__ __forceinline__ void run_ssssm(const GemmItem* gitems, const GemmTask* gtasks, int item, const DevPools& P,
                                       double* sm) {
  gemm_map_item(gitems[item], gtasks, P, sm);
}

// Early release of a chain-2 GETRF task (XTask::chain == 2: it also solves L(k+1, k)): its first
// XTask::pad1 successor entries need only the factored diagonal tile and are released right after
// it is stored; the rest after the fused solve (exec_body).
struct EarlyRelease {
  const XLevel* L;
  int t;
  __device__ void operator()() const {
    __threadfence();
    __syncthreads();
    const int e0 = L->succ_ptr[t], ne = L->tasks[t].pad1;
    for (int e = e0 + threadIdx.x; e < e0 + ne; e += blockDim.x) {
      const int sx = L->succ[e];
      atomicSub(L->deps + 2 * (sx >> 1) + (sx & 1), 1);
    }
  }
  __device__ explicit operator bool() const { return L != nullptr; }
};

template <bool kBandReg>
__device__ void run_task(const XTask& tk, const DevPools& P, double* sm, double pivot_tol,
                         unsigned long long* ph = nullptr, volatile int* d2 = nullptr,
                         const GemmItem* gitems = nullptr, const GemmTask* gtasks = nullptr,
                         EarlyRelease early = EarlyRelease{nullptr, 0}) {
  double* T0 = sm;                  // target tile (XTP stride)
  double* T1 = sm + XREG;           // operand tile (XTP stride) / DMMA A (XS stride)
  double* T2 = sm + 2 * XREG;       // DMMA B (XS stride)
  double* rinv = sm + 3 * XREG;     // XT doubles
#if LBK_ABSORB_TILES
  if (tk.type == X_SSSSM) {  // (tk.a indexes the SSSSM items, not the blocks)
    run_ssssm(gitems, gtasks, tk.a, P, sm);
    return;
  }
#endif
  const BlockDev A = P.blk[tk.a];
  switch (tk.type) {
    case X_COLMAX: {  // rows [r*COLMAX_ROWS, ...) of column tile c: atomic max into colmax
      const int m = A.nrows, c0 = xo(P, A, tk.c), nc = xo(P, A, tk.c + 1) - c0;
      const int rb = tk.r * COLMAX_ROWS, re = min(m, rb + COLMAX_ROWS);
      const double* G = P.vals + A.ent;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      unsigned long long* cmax = reinterpret_cast<unsigned long long*>(P.colmax) + A.dg;
      // four columns per round, 4 x 4 coalesced loads of a lane in flight at once
      // (latency-bound otherwise: the chain of a block starts after its first column's colmax)
      static_assert(COLMAX_ROWS == 4 * 32, "4 loads per lane and column");
      for (int cb = c0 + 4 * warp; cb < c0 + nc; cb += 4 * nw) {
        double v[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double* col = G + static_cast<size_t>(min(cb + q, c0 + nc - 1)) * m;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = rb + lane + 32 * j;
            v[q][j] = r < re ? ldcg(col + r) : 0.0;
          }
        }
        double mq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          mq[q] = fmax(fmax(fabs(v[q][0]), fabs(v[q][1])), fmax(fabs(v[q][2]), fabs(v[q][3])));
#pragma unroll
          for (int o = 16; o; o >>= 1) mq[q] = fmax(mq[q], __shfl_xor_sync(0xffffffffu, mq[q], o));
        }
        if (lane < 4 && cb + lane < c0 + nc) {
          const double mv = lane == 0 ? mq[0] : lane == 1 ? mq[1] : lane == 2 ? mq[2] : mq[3];
          if (mv > 0.0) atomic_max_nonneg(cmax + cb + lane, mv);
        }
      }
      break;
    }
    case X_GETRF:
    case X_GETRF_UPD: {
      const int m = A.nrows, k0 = xo(P, A, tk.r), n = xo(P, A, tk.r + 1) - k0;
      double* G = P.vals + A.ent + static_cast<size_t>(k0) * m + k0;
      load_tile(T0, G, m, n, n);
      wait_phase2(d2, ph);  // the operand tiles of the fused update
      if (tk.type == X_GETRF_UPD) {  // the last trailing update of this tile first
        const int u0 = xo(P, A, tk.k), nu = xo(P, A, tk.k + 1) - u0;
        const double* base = P.vals + A.ent;
        load_opA(T1, base + static_cast<size_t>(u0) * m + k0, m, n, nu);
        load_opB(T2, base + static_cast<size_t>(k0) * m + u0, m, nu, n);
        __syncthreads();
        tile_mma_sub(T0, T1, T2);
      }
      __syncthreads();
      stamp(ph, 0);
#if LBK_LU_LA
      tile_lu64_la(T0, n, T1);
#else
      tile_lu64_blocked(T0, n, T1, rinv);
#endif
      stamp(ph, 1);
      store_tile(G, m, T0, n, n);
      if (tk.chain == 2 && early) early();  // the tasks that need only this factored tile start now
      if (!LBK_LATE_FLUSH || tk.chain) flush_colmax(T1, n, n, false, P.bmax + A.dg + k0, T2);
      stamp(ph, 2);
      if (tk.chain) {
        // the critical chain of the diagonal block continues through L(k+1, k) and U(k, k+1):
        // solve them here with the factored tile still in shared memory (no handoff, no reload)
        const int r0 = k0 + n, nr = xo(P, A, tk.r + 2) - r0;
        __syncthreads();
        load_tile(T1, P.vals + A.ent + static_cast<size_t>(k0) * m + r0, m, nr, n);  // L tile (r0, k0)
        if (threadIdx.x < XT) rinv[threadIdx.x] = threadIdx.x < n ? 1.0 / T0[threadIdx.x * XTP + threadIdx.x] : 1.0;
        __syncthreads();
        tile_right_solve_blk<true>(T1, T0, rinv, T2, n);
        store_tile(P.vals + A.ent + static_cast<size_t>(k0) * m + r0, m, T1, nr, n);
        flush_colmax(T2, nr, n, true, P.bmax + A.dg + k0, T1);
        if (tk.chain == 1) {
          __syncthreads();
          load_tile(T1, P.vals + A.ent + static_cast<size_t>(r0) * m + k0, m, n, nr);  // U tile (k0, r0)
          __syncthreads();
          tile_left_solve_blk(T1, T0, n);
          store_tile(P.vals + A.ent + static_cast<size_t>(r0) * m + k0, m, T1, n, nr);
        }
        stamp(ph, 3);
      }
      break;
    }
    case X_TRSM_L: {  // rows of tile (r,k) in registers, U_kk in smem
      const int m = A.nrows, k0 = xo(P, A, tk.k), r0 = xo(P, A, tk.r), nk = xo(P, A, tk.k + 1) - k0,
                nr = xo(P, A, tk.r + 1) - r0;
      double* G = P.vals + A.ent + static_cast<size_t>(k0) * m + r0;
      load_tile(T0, G, m, nr, nk);  // the target first: its last update is done (phase 1)
      wait_phase2(d2, ph);              // the factored diagonal tile
      load_tile(T1, P.vals + A.ent + static_cast<size_t>(k0) * m + k0, m, nk, nk);
      __syncthreads();
      stamp(ph, 0);
      if (threadIdx.x < XT) rinv[threadIdx.x] = threadIdx.x < nk ? 1.0 / T1[threadIdx.x * XTP + threadIdx.x] : 1.0;
      __syncthreads();
      tile_right_solve_blk<true>(T0, T1, rinv, T2, nk);
      stamp(ph, 1);
      store_tile(G, m, T0, nr, nk);
      stamp(ph, 2);
      if (!LBK_LATE_FLUSH) flush_colmax(T2, nr, nk, true, P.bmax + A.dg + k0, T1);
      stamp(ph, 3);
      break;
    }
    case X_TRSM_U: {  // columns of tile (k,c) in registers, L_kk in smem
      const int m = A.nrows, k0 = xo(P, A, tk.k), c0 = xo(P, A, tk.c), nk = xo(P, A, tk.k + 1) - k0,
                nc = xo(P, A, tk.c + 1) - c0;
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * m + k0;
      load_tile(T0, G, m, nk, nc);  // the target first (phase 1)
      wait_phase2(d2, ph);              // the factored diagonal tile
      load_tile(T1, P.vals + A.ent + static_cast<size_t>(k0) * m + k0, m, nk, nk);
      __syncthreads();
      tile_left_solve_blk(T0, T1, nk);
      store_tile(G, m, T0, nk, nc);
      break;
    }
    case X_GEMM: {  // tk.pad1 > 1: the updates from steps k .. k + pad1 - 1, in k order (one target load / store)
      const int m = A.nrows, r0 = xo(P, A, tk.r), c0 = xo(P, A, tk.c);
      const int nr = xo(P, A, tk.r + 1) - r0, nc = xo(P, A, tk.c + 1) - c0;
      const double* base = P.vals + A.ent;
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * m + r0;
      load_tile(T0, G, m, nr, nc);
      for (int q = 0, nq = max(1, static_cast<int>(tk.pad1)); q < nq; ++q) {
        const int k0 = xo(P, A, tk.k + q), nk = xo(P, A, tk.k + q + 1) - k0;
        load_opA(T1, base + static_cast<size_t>(k0) * m + r0, m, nr, nk);
        load_opB(T2, base + static_cast<size_t>(c0) * m + k0, m, nk, nc);
        __syncthreads();
        tile_mma_sub(T0, T1, T2);
      }
      store_tile(G, m, T0, nr, nc);
      break;
    }
    case X_FINAL: {
      const int m = A.nrows;
      const double* G = P.vals + A.ent;
      for (int c = threadIdx.x; c < m; c += blockDim.x) {
        const double u = fabs(ldcg(G + static_cast<size_t>(c) * m + c));
        const double below = __longlong_as_double(static_cast<long long>(
            __ldcg(reinterpret_cast<const unsigned long long*>(P.bmax + A.dg + c))));
        const double piv = fmax(u, below);
        if (piv == 0.0 || piv < pivot_tol * __ldcg(P.colmax + A.dg + c) || isnan(u)) record(&P.err[0], tk.step, c);
        else if (below > u) record(&P.err[1], tk.step, c);
      }
      break;
    }
    case X_PG_DIAG:
    case X_PG_UPD:
    case X_PG_FUSED: {
      // GESSM on panel X (rows R_X): L = unit lower of diagonal block D restricted to R_X
      const BlockDev D = P.blk[tk.d];
      const int m = D.nrows, ld = A.nR;
      const int32_t* Rl = A.store == STORE_RECT ? P.rlist + A.roff : nullptr;
      const int r0 = xop(P, A, tk.r, A.nR), c0 = tk.c * XT, nr = xop(P, A, tk.r + 1, A.nR) - r0,
                nc = min(XT, A.nC - c0);
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * ld + r0;
      const double* Dv = P.vals + D.ent;
      if (tk.type == X_PG_DIAG || tk.type == X_PG_FUSED) {
        load_tile(T0, G, ld, nr, nc);
        if (tk.type == X_PG_FUSED) {  // the update from the previous row step first
          const int k0 = xop(P, A, tk.k, A.nR), nk = xop(P, A, tk.k + 1, A.nR) - k0;
          if (Rl) load_opA(T1, Dv, m, nr, nk, Rl + r0, Rl + k0);
          else load_opA(T1, Dv + static_cast<size_t>(k0) * m + r0, m, nr, nk);
          load_opB(T2, P.vals + A.ent + static_cast<size_t>(c0) * ld + k0, ld, nk, nc);
          __syncthreads();
          tile_mma_sub(T0, T1, T2);
        }
        if (Rl) load_tile(T1, Dv, m, nr, nr, Rl + r0, Rl + r0);
        else load_tile(T1, Dv + static_cast<size_t>(r0) * m + r0, m, nr, nr);
        __syncthreads();
        tile_left_solve_blk(T0, T1, nr);
        store_tile(G, ld, T0, nr, nc);
      } else {  // tk.pad1 > 1: the updates from steps k .. k + pad1 - 1, in k order (one target load / store)
        load_tile(T0, G, ld, nr, nc);
        for (int q = 0, nq = max(1, static_cast<int>(tk.pad1)); q < nq; ++q) {
          const int k0 = xop(P, A, tk.k + q, A.nR), nk = xop(P, A, tk.k + q + 1, A.nR) - k0;
          if (Rl) load_opA(T1, Dv, m, nr, nk, Rl + r0, Rl + k0);
          else load_opA(T1, Dv + static_cast<size_t>(k0) * m + r0, m, nr, nk);
          load_opB(T2, P.vals + A.ent + static_cast<size_t>(c0) * ld + k0, ld, nk, nc);
          __syncthreads();
          tile_mma_sub(T0, T1, T2);  // (ends with a barrier: T1 / T2 free for the next step)
        }
        store_tile(G, ld, T0, nr, nc);
      }
      break;
    }
    case X_PT_DIAG:
    case X_PT_UPD:
    case X_PT_FUSED: {
      // TSTRF on panel X (cols C_X): U = upper of diagonal block D restricted to C_X
      const BlockDev D = P.blk[tk.d];
      const int m = D.nrows, ld = A.nR;
      const int32_t* Cl = A.store == STORE_RECT ? P.clist + A.coff : nullptr;
      const int r0 = tk.r * XT, c0 = xop(P, A, tk.c, A.nC), nr = min(XT, A.nR - r0),
                nc = xop(P, A, tk.c + 1, A.nC) - c0;
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * ld + r0;
      const double* Dv = P.vals + D.ent;
      if (tk.type == X_PT_DIAG || tk.type == X_PT_FUSED) {
        load_tile(T0, G, ld, nr, nc);
        if (tk.type == X_PT_FUSED) {  // the update from the previous column step first
          const int k0 = xop(P, A, tk.k, A.nC), nk = xop(P, A, tk.k + 1, A.nC) - k0;
          load_opA(T1, P.vals + A.ent + static_cast<size_t>(k0) * ld + r0, ld, nr, nk);
          if (Cl) load_opB(T2, Dv, m, nk, nc, Cl + k0, Cl + c0);
          else load_opB(T2, Dv + static_cast<size_t>(c0) * m + k0, m, nk, nc);
          __syncthreads();
          tile_mma_sub(T0, T1, T2);
        }
        if (Cl) load_tile(T1, Dv, m, nc, nc, Cl + c0, Cl + c0);
        else load_tile(T1, Dv + static_cast<size_t>(c0) * m + c0, m, nc, nc);
        __syncthreads();
        if (threadIdx.x < XT) rinv[threadIdx.x] = threadIdx.x < nc ? 1.0 / T1[threadIdx.x * XTP + threadIdx.x] : 1.0;
        __syncthreads();
        tile_right_solve_blk<false>(T0, T1, rinv, nullptr, nc);
        store_tile(G, ld, T0, nr, nc);
      } else {  // tk.pad1 > 1: the updates from steps k .. k + pad1 - 1, in k order (one target load / store)
        load_tile(T0, G, ld, nr, nc);
        for (int q = 0, nq = max(1, static_cast<int>(tk.pad1)); q < nq; ++q) {
          const int k0 = xop(P, A, tk.k + q, A.nC), nk = xop(P, A, tk.k + q + 1, A.nC) - k0;
          load_opA(T1, P.vals + A.ent + static_cast<size_t>(k0) * ld + r0, ld, nr, nk);
          if (Cl) load_opB(T2, Dv, m, nk, nc, Cl + k0, Cl + c0);
          else load_opB(T2, Dv + static_cast<size_t>(c0) * m + k0, m, nk, nc);
          __syncthreads();
          tile_mma_sub(T0, T1, T2);
        }
        store_tile(G, ld, T0, nr, nc);
      }
      break;
    }
    case X_BAND:
      // (one instance only: more instances push the executor past 255 registers)
      if (kBandReg && tk.r == 4 && tk.c == 4) band_getrf_reg<4>(A, P, sm, tk.d, tk.k, tk.step, pivot_tol);
      else band_getrf(A, P, sm, tk.r, tk.c, tk.d, tk.k, tk.step, pivot_tol);
      break;
    default:
      break;
  }
}

// kBandReg: the launch holds band sweeps of half-bandwidth 4 (BBD bodies),
// run by the register-window sweep; its registers (> 128) allow one CTA per SM,
// so levels without such sweeps use the plain instance at two CTAs per SM.
// Late colmax flush: a GETRF tile and a TRSM_L tile release their successors as soon
// as their tile is stored; the staged |d| maxima (still in shared memory) are folded
// into bmax afterwards.  Only the pivot verdict (X_FINAL) reads bmax, so it alone is
// released after the flush.  Takes the flush (~1-1.5 us) off the critical tile chain.
__device__ __forceinline__ bool late_flush(const XTask& tk) {
  return LBK_LATE_FLUSH && (((tk.type == X_GETRF || tk.type == X_GETRF_UPD) && !tk.chain) || tk.type == X_TRSM_L);
}

__device__ void run_late_flush(const XTask& tk, const DevPools& P, double* sm) {
  double* T1 = sm + XREG;
  double* T2 = sm + 2 * XREG;
  const BlockDev A = P.blk[tk.a];
  if (tk.type == X_TRSM_L) {
    const int k0 = xo(P, A, tk.k), r0 = xo(P, A, tk.r), nk = xo(P, A, tk.k + 1) - k0, nr = xo(P, A, tk.r + 1) - r0;
    flush_colmax(T2, nr, nk, true, P.bmax + A.dg + k0, T1);
  } else {
    const int k0 = xo(P, A, tk.r), n = xo(P, A, tk.r + 1) - k0;
    flush_colmax(T1, n, n, false, P.bmax + A.dg + k0, T2);
  }
}

template <bool kBandReg>
__device__ __forceinline__ void exec_body(const XLevel& L, const DevPools& P, double pivot_tol) {
  extern __shared__ double sm[];
  __shared__ int s_t;
  for (;;) {
    if (threadIdx.x == 0) {
      const int t = atomicAdd(L.head, 1);
      if (t < L.ntasks) {
        if (L.trace) L.trace[8 * t] = gtimer();
        volatile int* dp = L.deps + 2 * t;  // phase-1 dependencies
        while (*dp > 0) __nanosleep(LBK_SPIN_NS);
        __threadfence();
        if (L.trace) L.trace[8 * t + 1] = gtimer();
      }
      s_t = t;
    }
    __syncthreads();
    const int t = s_t;
    if (t >= L.ntasks) break;
    const XTask tk = L.tasks[t];
    run_task<kBandReg>(tk, P, sm, pivot_tol, L.trace ? L.trace + 8 * t + 3 : nullptr, L.deps + 2 * t + 1, L.gitems,
                       L.gtasks, EarlyRelease{&L, t});
    // every thread fences its own tile writes before the barrier, so the
    // successor releases after it are ordered behind all of them; the
    // releases are spread over the CTA (a GETRF tile has ~2x(tiles per
    // column) successors: one thread walking them costs an L2 round trip each)
    __threadfence();
    __syncthreads();
    const bool late = late_flush(tk);
    {
      // (a chain-2 GETRF task released its first tk.pad1 entries inside run_task)
      const int e0 = L.succ_ptr[t] + (tk.chain == 2 ? tk.pad1 : 0), e1 = L.succ_ptr[t + 1];
      for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int sx = L.succ[e];
        if (!late || L.tasks[sx >> 1].type != X_FINAL) atomicSub(L.deps + 2 * (sx >> 1) + (sx & 1), 1);
      }
    }
    if (threadIdx.x == 0 && L.trace) L.trace[8 * t + 2] = gtimer();
    if (late) {
      run_late_flush(tk, P, sm);  // (flush_colmax ends with its atomics; fence + barrier below)
      __threadfence();
      __syncthreads();
      const int e0 = L.succ_ptr[t], e1 = L.succ_ptr[t + 1];
      for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int sx = L.succ[e];
        if (L.tasks[sx >> 1].type == X_FINAL) atomicSub(L.deps + 2 * (sx >> 1) + (sx & 1), 1);
      }
    }
  }
}

__global__ void __launch_bounds__(256, 2) exec_kernel(XLevel L, DevPools P, double pivot_tol) {
  exec_body<false>(L, P, pivot_tol);
}

__global__ void __launch_bounds__(256) exec_band_kernel(XLevel L, DevPools P, double pivot_tol) {
  exec_body<true>(L, P, pivot_tol);
}

}  // namespace lbk
