#pragma once
#include "../paper_2512_04389_b200/csrc/lbk_exec.cuh"
namespace lbk {
// ---- compact rotated-line solvers (the executor's critical-path tiles) -----------
// Threads 0..63 each own one line (a row for right solves and the LU, a column
// for left solves) of a 64x64 tile in x[64].  The loop over elimination steps
// is rolled; every step rotates the line down by one, so the live entry is
// always x[0] and all register indexing stays static.  A step is one
// broadcast smem read + one FMA per remaining entry, and the code of one
// solver is ~2 KB of SASS: the executor's task mix no longer thrashes the
// instruction cache (the fully unrolled 32x32 routines above are ~60 KB each).
// Entries rotated in past column 63 are dummies: they may pick up garbage
// from neighbouring smem but are never stored and never reach x[0].

constexpr int RS = 66;  // published-row stride (16-byte aligned rows)

// X <- X U^{-1} (TSTRF / below-diagonal tiles of GETRF).  U upper, column-major
// smem (XTP stride); rinv[j] = 1/u_jj.  Thread r stores x_rj to G as soon as it
// is final; kCheck stages |x_rj| before scaling in Dd[j*XTP + r].
template <bool kCheck>
__device__ __forceinline__ void rot_right_upper(double (&x)[XT], int nc, const double* U, const double* rinv,
                                                double* Dd, double* G, int ld, bool live) {
  const int r = threadIdx.x;
#pragma unroll 1
  for (int j = 0; j < nc; ++j) {
    const double d = x[0];
    if (kCheck) Dd[j * XTP + r] = live ? fabs(d) : 0.0;
    const double xj = d * rinv[j];
    if (live) G[static_cast<size_t>(j) * ld + r] = xj;
    const double* Uj = U + j * XTP + j;  // U(j, j + c) = Uj[c * XTP]
#pragma unroll
    for (int c = 1; c < XT; ++c) x[c - 1] = fma(-xj, Uj[c * XTP], x[c]);
  }
}

// X <- L^{-1} X, L unit lower column-major smem (XTP stride).  Thread c owns
// column c; row k of it is written to Out[c*XTP + k] when final.
__device__ __forceinline__ void rot_left_unit_lower(double (&x)[XT], int nr, const double* Lm, double* Out) {
  const int c = threadIdx.x;
#pragma unroll 1
  for (int k = 0; k < nr; ++k) {
    const double xk = x[0];
    Out[c * XTP + k] = xk;
    const double* Lk = Lm + k * XTP + k;  // L(k + r, k) = Lk[r]
#pragma unroll
    for (int r = 1; r < XT; ++r) x[r - 1] = fma(-Lk[r], xk, x[r]);
  }
}

__device__ __forceinline__ void bar_rows() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

// LU without row exchange of an n x n tile, thread r owns row r.  Step j: the
// owner of row j publishes it (rotated: R[j*RS + c] = a_{j, j+c}) and 1/u_jj,
// one 64-thread named barrier, every row r > j forms l_rj = d_rj * (1/u_jj)
// (stored to G at once, |d_rj| staged in Dd) and updates its entries.  Rows
// are published exactly once (R keeps all of them: no WAR hazard), so the
// U part is written out of R afterwards by the whole CTA.
__device__ __forceinline__ void rot_lu(double (&x)[XT], int n, double* R, double* rinv_s, double* Dd, double* G,
                                       int ld) {
  const int r = threadIdx.x;
#pragma unroll 1
  for (int j = 0; j < n; ++j) {
    if (r == j) {
      double* Rj = R + j * RS;
#pragma unroll
      for (int c = 0; c < XT; c += 2) *reinterpret_cast<double2*>(Rj + c) = make_double2(x[c], x[c + 1]);
      rinv_s[j] = 1.0 / x[0];
    }
    bar_rows();
    if (r > j) {
      const double d = x[0];
      const bool live = r < n;
      Dd[j * XTP + r] = live ? fabs(d) : 0.0;
      const double l = d * rinv_s[j];
      if (live) G[static_cast<size_t>(j) * ld + r] = l;
      const double* Rj = R + j * RS;  // a_{j, j+c} = Rj[c]; x_new[c-1] = x[c] - l * Rj[c]
      x[0] = fma(-l, Rj[1], x[1]);
#pragma unroll
      for (int c = 2; c < XT; c += 2) {
        const double2 u = *reinterpret_cast<const double2*>(Rj + c);
        x[c - 1] = fma(-l, u.x, x[c]);
        x[c] = fma(-l, u.y, x[c + 1]);
      }
    }
  }
}

// U part (columns >= row) of the rows published by rot_lu -> G, coalesced.
__device__ __forceinline__ void store_lu_rows(double* G, int ld, const double* R, int n) {
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int j = e & (XT - 1), col = e >> 6;
    if (j < n && col < n && col >= j) G[static_cast<size_t>(col) * ld + j] = R[j * RS + (col - j)];
  }
}

// X (smem tile, XTP) <- L^{-1} X: thread c < 64 owns column c (conflict-free smem column reads).
__device__ __forceinline__ void left_solve_rot(double* X, const double* Lm, int nr) {
  if (threadIdx.x < XT) {
    double x[XT];
#pragma unroll
    for (int r = 0; r < XT; ++r) x[r] = X[threadIdx.x * XTP + r];
    rot_left_unit_lower(x, nr, Lm, X);
  }
  __syncthreads();
}

// Row r of a column-major tile into x[64] (coalesced across threads), zero padded.
__device__ __forceinline__ void load_row64(double (&x)[XT], const double* G, int ld, int nr, int nc) {
  const int r = threadIdx.x;
#pragma unroll
  for (int c = 0; c < XT; ++c) x[c] = (r < nr && c < nc) ? ldcg(G + static_cast<size_t>(c) * ld + r) : 0.0;
}


}  // namespace lbk
