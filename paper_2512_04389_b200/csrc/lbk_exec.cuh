// lbk_exec.cuh — persistent tile-DAG executor for the dense GETRF and panel
// solves of one dependency level.
//
// A diagonal block's LU (factorize.py:38-78) and every dense panel solve
// (GESSM factorize.py:98-109, TSTRF :112-130) are expanded on the host into
// 64x64-tile tasks with explicit dependencies (per-tile update chains, so
// the floating-point order is fixed and results are deterministic).  One
// launch per level runs all of them: each CTA pulls the next task index
// (host order is topological), waits for its dependency counter to reach
// zero, executes it, and decrements its successors' counters.  Tasks are
// only ever waited on after an earlier index was taken by a running CTA, so
// progress is guaranteed without co-residency assumptions.
//
// Mutable tiles may have been written by other SMs during the launch: all
// global reads of tile data use ld.global.cg (L2, bypassing the
// non-coherent L1).
//
// GETRF speculates "no row swap" and verifies the reference's pivot rule
// exactly (see lbk_dense.cuh): in-tile and below-tile |d_qc| before scaling
// feed bmax[c]; FINALIZE compares them with |u_cc| and colmax[c].

#pragma once

#include "lbk_common.cuh"
#include "lbk_dense.cuh"

namespace lbk {

constexpr int XT = 64;          // tile edge
constexpr int XTP = XT + 1;     // padded smem column stride (64 doubles + 1)
constexpr int XS = XT + 4;      // DMMA operand stride
constexpr int XREG = XT * XS;   // one smem tile region (fits either stride)
constexpr int EXEC_SMEM = (3 * XREG + XT) * 8;

enum XType : int8_t {
  X_COLMAX = 0,  // colmax / bmax / perm reset of diagonal block a
  X_GETRF = 1,   // factor diagonal tile (k,k) of block a
  X_TRSM_L = 2,  // tile (r,k) <- tile U_kk^{-1}
  X_TRSM_U = 3,  // tile (k,c) <- L_kk^{-1} tile
  X_GEMM = 4,    // tile (r,c) -= tile(r,k) tile(k,c)
  X_FINAL = 5,   // pivot verdict of block a
  X_PG_DIAG = 6, // GESSM panel a (rows R_X): tile (r,c) <- L[R_r,R_r]^{-1} tile
  X_PG_UPD = 7,  // tile (r,c) -= L[R_r, R_k] tile(k,c)
  X_PT_DIAG = 8, // TSTRF panel a (cols C_X): tile (r,c) <- tile U[C_c,C_c]^{-1}
  X_PT_UPD = 9,  // tile (r,c) -= tile(r,k) U[C_k, C_c]
};

struct XTask {
  int8_t type;
  int8_t pad0;
  int16_t r, c, k;
  int16_t pad1;
  int32_t a;     // block the task writes
  int32_t d;     // diagonal block (panel tasks), = a for GETRF tasks
  int32_t step;  // elimination step (error records)
};

struct XLevel {
  const XTask* tasks;
  const int32_t* succ_ptr;
  const int32_t* succ;
  int* deps;   // working dependency counters (reset from a pristine copy per run)
  int* head;   // task counter of this level
  int ntasks;
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// load a (nr x nc) tile from column-major global memory (leading dim ld) into
// smem T[c*XTP + r]; zero padding outside; optional row/column gathers.
__device__ __forceinline__ void load_tile(double* T, const double* G, int ld, int nr, int nc,
                                          const int32_t* rg = nullptr, const int32_t* cg = nullptr) {
  for (int idx = threadIdx.x; idx < XT * XT; idx += blockDim.x) {
    const int r = idx % XT, c = idx / XT;
    double v = 0.0;
    if (r < nr && c < nc) {
      const int gr = rg ? rg[r] : r, gc = cg ? cg[c] : c;
      v = ldcg(G + static_cast<size_t>(gc) * ld + gr);
    }
    T[c * XTP + r] = v;
  }
}

__device__ __forceinline__ void store_tile(double* G, int ld, const double* T, int nr, int nc) {
  for (int idx = threadIdx.x; idx < XT * XT; idx += blockDim.x) {
    const int r = idx % XT, c = idx / XT;
    if (r < nr && c < nc) G[static_cast<size_t>(c) * ld + r] = T[c * XTP + r];
  }
}

// Right-looking LU without row exchange of the tile in smem (n x n), 256
// threads; records max |d_qc| over in-tile rows below the diagonal before
// scaling into bmax (global, bits) for the block's columns c0 + j.
__device__ void tile_lu(double* T, int n, unsigned long long* bmax) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int j = 0; j < n; ++j) {
    const double u = T[j * XTP + j];
    double mx = 0.0;
    if (tid < 64) {
      const int r = tid;
      if (r > j && r < n) {
        const double v = T[j * XTP + r];
        mx = fabs(v);
        T[j * XTP + r] = __ddiv_rn(v, u);
      }
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0 && mx > 0.0) atomic_max_nonneg(&bmax[j], mx);
    }
    __syncthreads();
    const int rows = n - j - 1;
    for (int idx = tid; idx < rows * rows; idx += blockDim.x) {
      const int r = j + 1 + idx % rows, c = j + 1 + idx / rows;
      T[c * XTP + r] = dsub_mul(T[c * XTP + r], T[j * XTP + r], T[c * XTP + j]);
    }
    __syncthreads();
  }
}

// X (nr x nc, smem) <- X U^{-1}, U upper (nc x nc, smem, diag included).
// If bmax != nullptr: record max |x_qj| before the division per column j.
// Rows are independent: thread q owns row q (<= 64 rows); the column loop is
// sequential, operands in smem.
__device__ void tile_right_upper(double* X, int nr, int nc, const double* U, unsigned long long* bmax,
                                 double* cmx) {
  const int tid = threadIdx.x;
  if (bmax)
    for (int c = tid; c < XT; c += blockDim.x) cmx[c] = 0.0;
  __syncthreads();
  if (tid < nr) {
    for (int j = 0; j < nc; ++j) {
      const double d = X[j * XTP + tid];
      if (bmax && d != 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(&cmx[j]),
                  static_cast<unsigned long long>(__double_as_longlong(fabs(d))));
      const double x = __ddiv_rn(d, U[j * XTP + j]);
      X[j * XTP + tid] = x;
      for (int jj = j + 1; jj < nc; ++jj) X[jj * XTP + tid] = dsub_mul(X[jj * XTP + tid], x, U[jj * XTP + j]);
    }
  }
  __syncthreads();
  if (bmax)
    for (int c = tid; c < nc; c += blockDim.x)
      if (cmx[c] != 0.0) atomic_max_nonneg(&bmax[c], cmx[c]);
}

// X (nr x nc, smem) <- L^{-1} X, L unit lower (nr x nr, smem).  Thread c owns column c.
__device__ void tile_left_unit_lower(double* X, int nr, int nc, const double* L) {
  const int tid = threadIdx.x;
  if (tid < nc) {
    double* x = X + tid * XTP;
    for (int k = 0; k < nr; ++k) {
      const double xk = x[k];
      for (int r = k + 1; r < nr; ++r) x[r] = dsub_mul(x[r], L[k * XTP + r], xk);
    }
  }
  __syncthreads();
}

// C (smem, XTP stride) -= A (XS stride, [k][r]) * B (XS stride, [c][k]), 64x64x64, 8 warps of 32x16.
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
  __syncthreads();
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

// stage a tile as DMMA A operand ([k][r], stride XS) or B operand ([c][k], stride XS)
__device__ __forceinline__ void load_opA(double* As, const double* G, int ld, int nr, int nk,
                                         const int32_t* rg = nullptr, const int32_t* kg = nullptr) {
  for (int idx = threadIdx.x; idx < XT * XT; idx += blockDim.x) {
    const int r = idx % XT, k = idx / XT;
    double v = 0.0;
    if (r < nr && k < nk) v = ldcg(G + static_cast<size_t>(kg ? kg[k] : k) * ld + (rg ? rg[r] : r));
    As[k * XS + r] = v;
  }
}

__device__ __forceinline__ void load_opB(double* Bs, const double* G, int ld, int nk, int nc,
                                         const int32_t* kg = nullptr, const int32_t* cg = nullptr) {
  for (int idx = threadIdx.x; idx < XT * XT; idx += blockDim.x) {
    const int k = idx % XT, c = idx / XT;
    double v = 0.0;
    if (k < nk && c < nc) v = ldcg(G + static_cast<size_t>(cg ? cg[c] : c) * ld + (kg ? kg[k] : k));
    Bs[c * XS + k] = v;
  }
}

__device__ void run_task(const XTask& tk, const DevPools& P, double* sm, double pivot_tol) {
  double* T0 = sm;             // target tile (XTP stride)
  double* T1 = sm + XREG;      // operand tile (XTP stride) / DMMA A (XS stride)
  double* T2 = sm + 2 * XREG;  // DMMA B (XS stride)
  double* cmx = sm + 3 * XREG; // per-column scratch
  const BlockDev A = P.blk[tk.a];
  switch (tk.type) {
    case X_COLMAX: {
      const int m = A.nrows;
      const double* G = P.vals + A.ent;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int c = warp; c < m; c += nw) {
        double mx = 0.0;
        for (int r = lane; r < m; r += 32) mx = fmax(mx, fabs(ldcg(G + static_cast<size_t>(c) * m + r)));
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) {
          P.colmax[A.dg + c] = mx;
          P.bmax[A.dg + c] = 0ull;
          P.perm[A.dg + c] = c;
        }
      }
      break;
    }
    case X_GETRF: {
      const int m = A.nrows, k0 = tk.k * XT, n = min(XT, m - k0);
      double* G = P.vals + A.ent + static_cast<size_t>(k0) * m + k0;
      load_tile(T0, G, m, n, n);
      __syncthreads();
      tile_lu(T0, n, P.bmax + A.dg + k0);
      store_tile(G, m, T0, n, n);
      break;
    }
    case X_TRSM_L: {
      const int m = A.nrows, k0 = tk.k * XT, r0 = tk.r * XT, nk = min(XT, m - k0), nr = min(XT, m - r0);
      const double* Gd = P.vals + A.ent + static_cast<size_t>(k0) * m + k0;
      double* G = P.vals + A.ent + static_cast<size_t>(k0) * m + r0;
      load_tile(T1, Gd, m, nk, nk);
      load_tile(T0, G, m, nr, nk);
      __syncthreads();
      tile_right_upper(T0, nr, nk, T1, P.bmax + A.dg + k0, cmx);
      store_tile(G, m, T0, nr, nk);
      break;
    }
    case X_TRSM_U: {
      const int m = A.nrows, k0 = tk.k * XT, c0 = tk.c * XT, nk = min(XT, m - k0), nc = min(XT, m - c0);
      const double* Gd = P.vals + A.ent + static_cast<size_t>(k0) * m + k0;
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * m + k0;
      load_tile(T1, Gd, m, nk, nk);
      load_tile(T0, G, m, nk, nc);
      __syncthreads();
      tile_left_unit_lower(T0, nk, nc, T1);
      store_tile(G, m, T0, nk, nc);
      break;
    }
    case X_GEMM: {
      const int m = A.nrows, k0 = tk.k * XT, r0 = tk.r * XT, c0 = tk.c * XT;
      const int nk = min(XT, m - k0), nr = min(XT, m - r0), nc = min(XT, m - c0);
      const double* base = P.vals + A.ent;
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * m + r0;
      load_tile(T0, G, m, nr, nc);
      load_opA(T1, base + static_cast<size_t>(k0) * m + r0, m, nr, nk);
      load_opB(T2, base + static_cast<size_t>(c0) * m + k0, m, nk, nc);
      __syncthreads();
      tile_mma_sub(T0, T1, T2);
      store_tile(G, m, T0, nr, nc);
      break;
    }
    case X_FINAL: {
      const int m = A.nrows;
      const double* G = P.vals + A.ent;
      for (int c = threadIdx.x; c < m; c += blockDim.x) {
        const double u = fabs(ldcg(G + static_cast<size_t>(c) * m + c));
        const double below = __longlong_as_double(static_cast<long long>(__ldcg(
            reinterpret_cast<const unsigned long long*>(P.bmax + A.dg + c))));
        const double piv = fmax(u, below);
        if (piv == 0.0 || piv < pivot_tol * __ldcg(P.colmax + A.dg + c) || isnan(u)) record(&P.err[0], tk.step, c);
        else if (below > u) record(&P.err[1], tk.step, c);
      }
      break;
    }
    case X_PG_DIAG:
    case X_PG_UPD: {
      // GESSM on panel X (rows R_X): L = unit lower of diagonal block D restricted to R_X
      const BlockDev D = P.blk[tk.d];
      const int m = D.nrows, ld = A.nR;
      const int32_t* R = A.store == STORE_RECT ? P.rlist + A.roff : nullptr;
      const int r0 = tk.r * XT, c0 = tk.c * XT, nr = min(XT, A.nR - r0), nc = min(XT, A.nC - c0);
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * ld + r0;
      const double* Dv = P.vals + D.ent;
      if (tk.type == X_PG_DIAG) {
        // gathered L_sub = D[R[r0+a], R[r0+b]]
        if (R) load_tile(T1, Dv, m, nr, nr, R + r0, R + r0);
        else load_tile(T1, Dv + static_cast<size_t>(r0) * m + r0, m, nr, nr);
        load_tile(T0, G, ld, nr, nc);
        __syncthreads();
        tile_left_unit_lower(T0, nr, nc, T1);
      } else {
        const int k0 = tk.k * XT, nk = min(XT, A.nR - k0);
        load_tile(T0, G, ld, nr, nc);
        if (R) load_opA(T1, Dv, m, nr, nk, R + r0, R + k0);
        else load_opA(T1, Dv + static_cast<size_t>(k0) * m + r0, m, nr, nk);
        load_opB(T2, P.vals + A.ent + static_cast<size_t>(c0) * ld + k0, ld, nk, nc);
        __syncthreads();
        tile_mma_sub(T0, T1, T2);
      }
      store_tile(G, ld, T0, nr, nc);
      break;
    }
    case X_PT_DIAG:
    case X_PT_UPD: {
      // TSTRF on panel X (cols C_X): U = upper of diagonal block D restricted to C_X
      const BlockDev D = P.blk[tk.d];
      const int m = D.nrows, ld = A.nR;
      const int32_t* Cl = A.store == STORE_RECT ? P.clist + A.coff : nullptr;
      const int r0 = tk.r * XT, c0 = tk.c * XT, nr = min(XT, A.nR - r0), nc = min(XT, A.nC - c0);
      double* G = P.vals + A.ent + static_cast<size_t>(c0) * ld + r0;
      const double* Dv = P.vals + D.ent;
      if (tk.type == X_PT_DIAG) {
        if (Cl) load_tile(T1, Dv, m, nc, nc, Cl + c0, Cl + c0);
        else load_tile(T1, Dv + static_cast<size_t>(c0) * m + c0, m, nc, nc);
        load_tile(T0, G, ld, nr, nc);
        __syncthreads();
        tile_right_upper(T0, nr, nc, T1, nullptr, cmx);
      } else {
        const int k0 = tk.k * XT, nk = min(XT, A.nC - k0);
        load_tile(T0, G, ld, nr, nc);
        load_opA(T1, P.vals + A.ent + static_cast<size_t>(k0) * ld + r0, ld, nr, nk);
        if (Cl) load_opB(T2, Dv, m, nk, nc, Cl + k0, Cl + c0);
        else load_opB(T2, Dv + static_cast<size_t>(c0) * m + k0, m, nk, nc);
        __syncthreads();
        tile_mma_sub(T0, T1, T2);
      }
      store_tile(G, ld, T0, nr, nc);
      break;
    }
    default:
      break;
  }
}

__global__ void __launch_bounds__(256) exec_kernel(XLevel L, DevPools P, double pivot_tol) {
  extern __shared__ double sm[];
  __shared__ int s_t;
  for (;;) {
    if (threadIdx.x == 0) {
      int t = atomicAdd(L.head, 1);
      if (t < L.ntasks) {
        volatile int* dp = L.deps + t;
        while (*dp > 0) __nanosleep(64);
        __threadfence();
      }
      s_t = t;
    }
    __syncthreads();
    const int t = s_t;
    if (t >= L.ntasks) break;
    const XTask tk = L.tasks[t];
    run_task(tk, P, sm, pivot_tol);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int e = L.succ_ptr[t]; e < L.succ_ptr[t + 1]; ++e) atomicSub(L.deps + L.succ[e], 1);
    }
    __syncthreads();
  }
}

}  // namespace lbk
