// lbk_solve.cuh — device triangular solve on the resident factors.
//
// Replaces the host solve of the reference,
//   x = U^-1 L^-1 b[perm_global]      factorize.py:451-457 (spsolve_triangular
//                                     on the assembled CSR, _assemble :218-239)
// with a blocked substitution over the factor blocks exactly as the device
// holds them after lbk_factorize (working layout: FULL / RECT tiles, CSC):
// L = unit lower (diagonal blocks' strict lower part + I, blocks bi > bj),
// U = upper (diagonal blocks' upper part incl. the diagonal, blocks bi < bj),
// the same blocks LUFactors exports (factorize.py:370-384), so the quirk of
// unpermuted L blocks left of a pivoting diagonal block is reproduced too.
//
// Column-oriented: step i solves the diagonal block of block row i in one
// CTA (64-row chunks: the 64x64 triangle by one warp out of shared memory,
// the rest of the chunk's column panel as a GEMV on all threads), then one
// launch updates every target block row k with the stored blocks of block
// column i: r_k -= B_ki y_i — distinct targets per block, row chunks per
// item, so no atomics and a fixed summation order.  2p + 2p launches per
// solve, captured once into a CUDA graph.

#pragma once

#include "lbk_common.cuh"

namespace lbk {

constexpr int SOLVE_CHUNK = 64;     // rows per diagonal-solve chunk
constexpr int UPD_ROWS = 256;       // block rows per update item

struct SolveStep {
  int32_t diag;   // diagonal block id
  int32_t off;    // global offset of the block row
  int32_t span;
  int32_t nupd;   // update items of this step
  int64_t upd_off;
};

struct SolveUpd {
  int32_t blk;      // factor block B_ki
  int32_t tgt_off;  // global offset of block row k
  int32_t src_off;  // global offset of block row i (solved segment)
  int32_t r0;       // first stored row (FULL/SPARSE: local row; RECT: row-list index)
};

// v[g] = b[blockstart[g] + perm[dgrow[g]]]  (b[perm_global])
__global__ void solve_perm_kernel(const double* __restrict__ b, double* __restrict__ v,
                                  const int32_t* __restrict__ perm, const int32_t* __restrict__ bstart,
                                  const int64_t* __restrict__ dgrow, int64_t n) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[g] = b[bstart[g] + perm[dgrow[g]]];
}

// Diagonal block of one step, one CTA (256 threads).  Dynamic smem: the
// segment y[span] and one 64x64 triangle (column-major, stride 65).
// FULL storage: blocked; SPARSE storage (all-CSC plans): column sweep.
__global__ void __launch_bounds__(256) solve_diag_kernel(DevPools P, const SolveStep* __restrict__ steps, int s,
                                                        double* __restrict__ v, int upper) {
  extern __shared__ double sm[];
  const SolveStep S = steps[s];
  const BlockDev D = P.blk[S.diag];
  const int m = S.span, tid = threadIdx.x, lane = tid & 31;
  double* y = sm;
  double* Tr = sm + ((m + 1) & ~1);
  for (int r = tid; r < m; r += blockDim.x) y[r] = v[S.off + r];
  __syncthreads();
  const double* G = P.vals + D.ent;
  if (D.store == STORE_SPARSE) {
    // column sweep on the CSC pattern (rows sorted): forward k ascending, the
    // entries below the diagonal update later rows; backward k descending
    const int32_t* cp = P.colptr + D.cp;
    const int32_t* rw = P.rows + D.ent;
    for (int q = 0; q < m; ++q) {
      const int k = upper ? m - 1 - q : q;
      const int e0 = cp[k], e1 = cp[k + 1];
      double yk = y[k];
      if (upper) {
        double ukk = 1.0;
        for (int e = e0; e < e1; ++e)
          if (rw[e] == k) ukk = G[e];
        yk = yk / ukk;
      }
      __syncthreads();
      if (tid == 0) y[k] = yk;
      for (int e = e0 + tid; e < e1; e += blockDim.x) {
        const int r = rw[e];
        if (upper ? r < k : r > k) y[r] = fma(-G[e], yk, y[r]);
      }
      __syncthreads();
    }
  } else {
    const int ld = D.nR;  // FULL: m x m column-major
    const int nchunks = (m + SOLVE_CHUNK - 1) / SOLVE_CHUNK;
    for (int q = 0; q < nchunks; ++q) {
      const int cb = upper ? nchunks - 1 - q : q;
      const int c0 = cb * SOLVE_CHUNK, cn = min(SOLVE_CHUNK, m - c0);
      // stage the chunk's triangle
      for (int e = tid; e < SOLVE_CHUNK * SOLVE_CHUNK; e += blockDim.x) {
        const int r = e & (SOLVE_CHUNK - 1), c = e >> 6;
        Tr[c * 65 + r] = (r < cn && c < cn) ? G[static_cast<size_t>(c0 + c) * ld + c0 + r] : 0.0;
      }
      __syncthreads();
      if (tid < 32) {
        double ya = lane < cn ? y[c0 + lane] : 0.0, yb = lane + 32 < cn ? y[c0 + 32 + lane] : 0.0;
        for (int kk = 0; kk < cn; ++kk) {
          const int k = upper ? cn - 1 - kk : kk;
          double yk = __shfl_sync(0xffffffffu, k < 32 ? ya : yb, k & 31);
          if (upper) yk = yk / Tr[k * 65 + k];
          if (lane == (k & 31)) {
            if (k < 32) ya = yk;
            else yb = yk;
          }
          const int ra = lane, rb = lane + 32;
          if (upper ? ra < k : (ra > k && ra < cn)) ya = fma(-Tr[k * 65 + ra], yk, ya);
          if (upper ? rb < k : (rb > k && rb < cn)) yb = fma(-Tr[k * 65 + rb], yk, yb);
        }
        if (lane < cn) y[c0 + lane] = ya;
        if (lane + 32 < cn) y[c0 + 32 + lane] = yb;
      }
      __syncthreads();
      // the rest of the chunk's columns: rows below (forward) / above (backward)
      const int rb0 = upper ? 0 : c0 + cn, rb1 = upper ? c0 : m;
      for (int r = rb0 + tid; r < rb1; r += blockDim.x) {
        double acc = y[r];
        const double* col = G + static_cast<size_t>(c0) * ld + r;
#pragma unroll 8
        for (int k = 0; k < cn; ++k) acc = fma(-col[static_cast<size_t>(k) * ld], y[c0 + k], acc);
        y[r] = acc;
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < m; r += blockDim.x) v[S.off + r] = y[r];
}

// r_k -= B_ki y_i for one row chunk of one stored block (256 threads, one row each).
// Dynamic smem: the source segment (block column span).
__global__ void __launch_bounds__(256) solve_upd_kernel(DevPools P, const SolveUpd* __restrict__ items,
                                                       double* __restrict__ v) {
  extern __shared__ double ys[];
  const SolveUpd it = items[blockIdx.x];
  const BlockDev B = P.blk[it.blk];
  const int tid = threadIdx.x;
  for (int c = tid; c < B.ncols; c += blockDim.x) ys[c] = v[it.src_off + c];
  __syncthreads();
  const double* G = P.vals + B.ent;
  const int a = it.r0 + tid;
  if (B.store == STORE_SPARSE) {
    if (a >= B.nrows) return;
    const int32_t* rp = P.csr_ptr + B.rp;
    const int32_t* cc = P.csr_col + B.csr;
    const int32_t* ps = P.csr_pos + B.csr;
    double acc = 0.0;
    for (int g = rp[a]; g < rp[a + 1]; ++g) acc = fma(G[ps[g]], ys[cc[g]], acc);
    v[it.tgt_off + a] -= acc;
  } else {
    if (a >= B.nR) return;
    const int32_t* cl = B.store == STORE_RECT ? P.clist + B.coff : nullptr;
    const int row = B.store == STORE_RECT ? P.rlist[B.roff + a] : a;
    double acc = 0.0;
    const double* col = G + a;
#pragma unroll 4
    for (int c = 0; c < B.nC; ++c) acc = fma(col[static_cast<size_t>(c) * B.nR], ys[cl ? cl[c] : c], acc);
    v[it.tgt_off + row] -= acc;
  }
}

}  // namespace lbk
