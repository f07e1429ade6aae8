// lbk_dense.cuh — FP64 tensor-core (DMMA) kernels for density-tagged blocks.
//
// Blocks whose density reaches the tag threshold (reference: nnz*2 >=
// nrows*ncols, factorize.py:271-275) are stored as their full rectangle,
// column-major with ld = nrows (a "full CSC" block), so the four kernels
// run as dense tiles on the FP64 tensor pipe:
//   SSSSM  dgemm_tile_kernel: C -= L*U, 128x64 CTA tiles, 8 warps of 32x32,
//          3-stage cp.async pipeline, mma.sync m8n8k4 f64 (SASS DMMA.8x8x4);
//   GETRF  dense_getrf_kernel: blocked right-looking LU, block-local partial
//          pivoting with the reference's rules (factorize.py:38-78), DMMA
//          trailing updates;
//   GESSM  dense_gessm_kernel: blocked forward substitution per 64-column strip;
//   TSTRF  dense_tstrf_kernel: blocked back substitution per 64-row strip.
// tcgen05 has no f64 kind; warp-level mma.sync is the FP64 tensor path on
// sm_100a.  Results equal the sparse kernels' within rounding (the blocked
// order changes the summation order, never the operands).

#pragma once

namespace lbk_dense {

constexpr int GBM = 128, GBN = 64, GBK = 16, GSTAGES = 3;
constexpr int SA = GBM + 4;  // padded k-column stride of the A tile (bank-conflict free frags)
constexpr int SB = GBK + 4;  // padded n-column stride of the B tile
constexpr int GEMM_SMEM = GSTAGES * (GBK * SA + GBN * SB) * 8;
constexpr int NB = 32;       // panel width of the blocked LU / TRSM
constexpr int STRIP = 64;    // columns (GESSM) / rows (TSTRF) per CTA

struct GemmItem {
  int32_t a, b, c;  // L, U, C block ids
  int32_t m0, n0;   // tile origin in C
  int32_t pad;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* src, bool valid) {
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// C[M x N] -= A[M x K] * B[K x N] for one 128x64 tile of C; all operands
// column-major dense blocks of the pool.
__global__ void __launch_bounds__(256) dgemm_tile_kernel(const GemmItem* __restrict__ items, DevPools P) {
  extern __shared__ double sm[];
  const GemmItem it = items[blockIdx.x];
  const BlockDev Lb = P.blk[it.a], Ub = P.blk[it.b], Cb = P.blk[it.c];
  const double* __restrict__ A = P.vals + Lb.ent;
  const double* __restrict__ B = P.vals + Ub.ent;
  double* C = P.vals + Cb.ent;
  const int lda = Lb.nrows, ldb = Ub.nrows, ldc = Cb.nrows;
  const int M = Cb.nrows, N = Cb.ncols, K = Lb.ncols;
  const int m0 = it.m0, n0 = it.n0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int nk = (K + GBK - 1) / GBK;
  auto stageA = [&](int s) { return sm + s * (GBK * SA + GBN * SB); };
  auto stageB = [&](int s) { return sm + s * (GBK * SA + GBN * SB) + GBK * SA; };
  auto load = [&](int s, int kt) {
    const int k0 = kt * GBK;
    double* As = stageA(s);
    double* Bs = stageB(s);
#pragma unroll
    for (int i = 0; i < (GBK * GBM) / 256; ++i) {
      const int idx = tid + i * 256;
      const int kk = idx / GBM, mm = idx % GBM;
      const int gr = m0 + mm, gk = k0 + kk;
      const bool v = gr < M && gk < K;
      cp_async8(As + kk * SA + mm, v ? A + static_cast<size_t>(gk) * lda + gr : A, v);
    }
#pragma unroll
    for (int i = 0; i < (GBK * GBN) / 256; ++i) {
      const int idx = tid + i * 256;
      const int nn = idx / GBK, kk = idx % GBK;
      const int gc = n0 + nn, gk = k0 + kk;
      const bool v = gc < N && gk < K;
      cp_async8(Bs + nn * SB + kk, v ? B + static_cast<size_t>(gc) * ldb + gk : B, v);
    }
  };
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    const int pf = kt + GSTAGES - 1;
    if (pf < nk) load(pf % GSTAGES, pf);
    cp_async_commit();
    const double* As = stageA(kt % GSTAGES);
    const double* Bs = stageB(kt % GSTAGES);
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[(kk + t) * SA + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + g) * SB + kk + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + wn + j * 8 + 2 * t;
      if (c < N) C[static_cast<size_t>(c) * ldc + r] -= acc[i][j][0];
      if (c + 1 < N) C[static_cast<size_t>(c + 1) * ldc + r] -= acc[i][j][1];
    }
  }
}

// CTA-cooperative C -= A*B with fragments read straight from global (L1/L2
// resident panels); warps own 32x32 tiles of C.
__device__ void cta_gemm_sub(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int M,
                             int N, int K) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int tm = (M + 31) / 32, tn = (N + 31) / 32;
  for (int tile = warp; tile < tm * tn; tile += nw) {
    const int m0 = (tile % tm) * 32, n0 = (tile / tm) * 32;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int k = 0; k < K; k += 4) {
      const int kk = k + t;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = m0 + i * 8 + g;
        a[i] = (r < M && kk < K) ? A[static_cast<size_t>(kk) * lda + r] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = n0 + j * 8 + g;
        b[j] = (c < N && kk < K) ? B[static_cast<size_t>(c) * ldb + kk] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + i * 8 + g;
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = n0 + j * 8 + 2 * t;
        if (c < N) C[static_cast<size_t>(c) * ldc + r] -= acc[i][j][0];
        if (c + 1 < N) C[static_cast<size_t>(c + 1) * ldc + r] -= acc[i][j][1];
      }
    }
  }
}

struct DenseItem {
  int32_t kind;
  int32_t a, b;   // GETRF: diag block, step; GESSM/TSTRF: diag block, panel block
  int32_t c;      // GETRF: swaps allowed; GESSM: apply perm
  int32_t begin;  // strip origin (GESSM column / TSTRF row)
  int32_t step;
};

// Blocked right-looking LU of one dense diagonal block (one CTA).
__device__ void dense_getrf(const DenseItem& it, const DevPools& P, double* sh, double pivot_tol,
                            double static_eps) {
  const BlockDev D = P.blk[it.a];
  const int m = D.nrows, step = it.b;
  const bool can_swap = it.c != 0;
  double* A = P.vals + D.ent;
  int32_t* perm = P.perm + D.dg;
  double* colmax = sh;             // m
  double* red_v = sh + m;          // 32
  int* red_r = reinterpret_cast<int*>(sh + m + 32);  // 32
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const bool use_static = !isnan(static_eps);
  for (int c = tid; c < m; c += nt) {
    double mx = 0.0;
    const double* col = A + static_cast<size_t>(c) * m;
    for (int r = 0; r < m; ++r) mx = fmax(mx, fabs(col[r]));
    colmax[c] = mx;
    perm[c] = c;
  }
  __syncthreads();
  for (int kb = 0; kb < m; kb += NB) {
    const int nb = min(NB, m - kb);
    for (int j = 0; j < nb; ++j) {
      const int c = kb + j;
      double* colc = A + static_cast<size_t>(c) * m;
      // first-max pivot search over rows c..m-1
      double best = -1.0;
      int brow = m;
      for (int r = c + tid; r < m; r += nt) {
        const double a = fabs(colc[r]);
        if (a > best) { best = a; brow = r; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
        if (ob > best || (ob == best && orow < brow)) { best = ob; brow = orow; }
      }
      if (lane == 0) { red_v[warp] = best; red_r[warp] = brow; }
      __syncthreads();
      if (tid == 0) {
        double b = red_v[0];
        int br = red_r[0];
        for (int w = 1; w < nw; ++w)
          if (red_v[w] > b || (red_v[w] == b && red_r[w] < br)) { b = red_v[w]; br = red_r[w]; }
        int action = 0;  // 0 none, 1 swap
        if (b == 0.0 || b < pivot_tol * colmax[c]) {
          if (use_static) {
            const double cur = colc[c];
            colc[c] = (cur == 0.0) ? static_eps : copysign(static_eps, cur);
          } else {
            record(&P.err[0], step, c);
          }
        } else if (br != c) {
          if (can_swap) {
            action = 1;
            const int pt = perm[c];
            perm[c] = perm[br];
            perm[br] = pt;
          } else {
            record(&P.err[1], step, c);
          }
        }
        red_r[0] = action ? br : -1;
      }
      __syncthreads();
      const int sw = red_r[0];
      if (sw >= 0) {
        for (int q = tid; q < m; q += nt) {  // whole-row swap inside the block
          double* col = A + static_cast<size_t>(q) * m;
          const double tv = col[c];
          col[c] = col[sw];
          col[sw] = tv;
        }
        __syncthreads();
      }
      const double piv = colc[c];
      for (int r = c + 1 + tid; r < m; r += nt) colc[r] = __ddiv_rn(colc[r], piv);
      __syncthreads();
      // rank-1 update restricted to the panel columns c+1 .. kb+nb-1
      const int pc = kb + nb - c - 1;
      const int rows = m - c - 1;
      for (int idx = tid; idx < pc * rows; idx += nt) {
        const int q = c + 1 + idx % rows;
        const int jj = c + 1 + idx / rows;
        double* colj = A + static_cast<size_t>(jj) * m;
        colj[q] = __dsub_rn(colj[q], __dmul_rn(colc[q], colj[c]));
      }
      __syncthreads();
    }
    const int rest = m - kb - nb;
    if (rest <= 0) break;
    // U12 = L11^{-1} A12 (unit lower), one thread per column
    for (int jc = kb + nb + tid; jc < m; jc += nt) {
      double* col = A + static_cast<size_t>(jc) * m;
      for (int k = 0; k < nb; ++k) {
        const double xk = col[kb + k];
        const double* lk = A + static_cast<size_t>(kb + k) * m;
        for (int r = k + 1; r < nb; ++r) col[kb + r] = __dsub_rn(col[kb + r], __dmul_rn(lk[kb + r], xk));
      }
    }
    __syncthreads();
    // A22 -= L21 * U12
    cta_gemm_sub(A + static_cast<size_t>(kb + nb) * m + kb + nb, m, A + static_cast<size_t>(kb) * m + kb + nb, m,
                 A + static_cast<size_t>(kb + nb) * m + kb, m, rest, rest, nb);
    __syncthreads();
  }
}

// X(i,j)[:, strip] <- L_ii^{-1} P_i X(i,j)[:, strip]
__device__ void dense_gessm(const DenseItem& it, const DevPools& P, double* sh) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int m = D.nrows, ncol = X.ncols;
  const double* L = P.vals + D.ent;
  double* Xv = P.vals + X.ent;
  const int c0 = it.begin, nc = min(STRIP, ncol - c0);
  const int tid = threadIdx.x, nt = blockDim.x;
  double* Xs = Xv + static_cast<size_t>(c0) * m;
  if (it.c) {  // apply the block row permutation (full panel), column by column through smem
    const int32_t* perm = P.perm + D.dg;
    for (int j = 0; j < nc; ++j) {
      double* col = Xs + static_cast<size_t>(j) * m;
      for (int r = tid; r < m; r += nt) sh[r] = col[perm[r]];
      __syncthreads();
      for (int r = tid; r < m; r += nt) col[r] = sh[r];
      __syncthreads();
    }
  }
  for (int kb = 0; kb < m; kb += NB) {
    const int nb = min(NB, m - kb);
    for (int j = tid; j < nc; j += nt) {
      double* col = Xs + static_cast<size_t>(j) * m;
      for (int k = 0; k < nb; ++k) {
        const double xk = col[kb + k];
        const double* lk = L + static_cast<size_t>(kb + k) * m;
        for (int r = k + 1; r < nb; ++r) col[kb + r] = __dsub_rn(col[kb + r], __dmul_rn(lk[kb + r], xk));
      }
    }
    __syncthreads();
    const int rest = m - kb - nb;
    if (rest > 0)
      cta_gemm_sub(Xs + kb + nb, m, L + static_cast<size_t>(kb) * m + kb + nb, m, Xs + kb, m, rest, nc, nb);
    __syncthreads();
  }
}

// X(k,i)[strip, :] <- X(k,i)[strip, :] U_ii^{-1}
__device__ void dense_tstrf(const DenseItem& it, const DevPools& P) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int m = D.nrows, ldx = X.nrows;
  const double* U = P.vals + D.ent;
  double* Xv = P.vals + X.ent;
  const int r0 = it.begin, nr = min(STRIP, ldx - r0);
  const int tid = threadIdx.x, nt = blockDim.x;
  double* Xs = Xv + r0;
  for (int kb = 0; kb < m; kb += NB) {
    const int nb = min(NB, m - kb);
    for (int q = tid; q < nr; q += nt) {
      for (int k = 0; k < nb; ++k) {
        const double* uk = U + static_cast<size_t>(kb + k) * m;  // column kb+k of U
        double* xk = Xs + static_cast<size_t>(kb + k) * ldx + q;
        // x[:,k] -= sum over previous in-block columns was applied eagerly below
        const double v = __ddiv_rn(*xk, uk[kb + k]);
        *xk = v;
        for (int jj = k + 1; jj < nb; ++jj) {
          const double u = U[static_cast<size_t>(kb + jj) * m + kb + k];
          double* xj = Xs + static_cast<size_t>(kb + jj) * ldx + q;
          *xj = __dsub_rn(*xj, __dmul_rn(v, u));
        }
      }
    }
    __syncthreads();
    const int rest = m - kb - nb;
    if (rest > 0)
      cta_gemm_sub(Xs + static_cast<size_t>(kb + nb) * ldx, ldx, Xs + static_cast<size_t>(kb) * ldx, ldx,
                   U + static_cast<size_t>(kb + nb) * m + kb, m, nr, rest, nb);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) dense_kernel(const DenseItem* __restrict__ items, DevPools P,
                                                    double pivot_tol, double static_eps) {
  extern __shared__ double sh[];
  const DenseItem it = items[blockIdx.x];
  if (it.kind == 0) dense_getrf(it, P, sh, pivot_tol, static_eps);
  else if (it.kind == 1) dense_gessm(it, P, sh);
  else dense_tstrf(it, P);
}

}  // namespace lbk_dense
