// lbk_dense.cuh — FP64 tensor-core (DMMA) kernels for RECT / FULL tiles.
//
// tcgen05 has no f64 kind: warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4)
// is the FP64 tensor path on sm_100a.  Kernels:
//   gemm_map_kernel      SSSSM C -= L*U on tiles, 128x64 CTA tiles, 8 warps of
//                        32x32, 3-stage cp.async pipeline; operand gathers
//                        (inner index intersection) and output scatters (row /
//                        column position maps) for RECT tiles (factorize.py:307-325)
//   panel_kernel         GESSM / TSTRF of a RECT/FULL panel against a FULL
//                        diagonal tile, 64-wide strips, blocked (nb = 32) with
//                        DMMA updates (factorize.py:98-130)
//   exact_getrf (panel_kernel kind 0)  single-CTA LU with true block-local
//                        partial pivoting (dense-scratch mode / static pivot)
//   tiled GETRF          colmax -> [tile_getrf -> tile_trsm -> tile_gemm] x
//                        ceil(m/64) -> finalize: a multi-CTA LU of a FULL
//                        diagonal block that speculates "no row swap" and
//                        verifies it against the reference's pivot rule
//                        exactly: per column c, piv = max(|u_cc|, max_{q>c}
//                        |d_qc|) from the values before scaling; ZeroPivot
//                        iff piv == 0 or piv < tol*colmax_at_entry; a swap
//                        iff some |d_qc| > |u_cc| (first-max keeps ties on the
//                        diagonal) -> LBK_ERR_PIVOT_SWAP and the host re-runs
//                        in dense-scratch mode (factorize.py:38-78).

#pragma once

#include "lbk_common.cuh"

namespace lbk {

#ifndef LBK_GBK
#define LBK_GBK 16
#endif
#ifndef LBK_GSTAGES
#define LBK_GSTAGES 3
#endif
constexpr int GBM = 128, GBN = 64, GBK = LBK_GBK, GSTAGES = LBK_GSTAGES;
constexpr int SA = GBM + 4;  // padded k-column stride of the A tile (conflict-free fragment loads)
constexpr int SB = GBK + 4;  // padded n-column stride of the B tile
constexpr int GEMM_SMEM = GSTAGES * (GBK * SA + GBN * SB) * 8;
constexpr int NB = 32;     // blocking of the panel solves / exact LU
constexpr int STRIP = 64;  // panel columns (GESSM) / rows (TSTRF) per CTA
constexpr int TS = 64;     // tile of the tiled GETRF
constexpr int TSP = TS + 1;

struct GemmTask {
  int32_t a, b, c;                  // L, U, C block ids
  int32_t K;                        // inner length (|C_L cap R_U|)
  int64_t kL, kU, rmap, cmap;       // offsets into P.maps, -1 = identity
};

struct GemmItem {
  int32_t task;
  int32_t m0, n0;
  int32_t nkc;     // < 0: every GBK-chunk of the inner dimension; else the number of listed chunks
  int64_t kc_off;  // offset of the chunk list in P.kchunks (chunks whose L rows x U columns hold entries)
  int32_t ks, ke;  // split-K: this item's range of the tile's chunk sequence ([0, all) unsplit)
  int32_t wslot;   // split-K: workspace slot of its partial product (-1: C -= product directly)
  int32_t nsplit;  // reduce items: partial products of the tile, in slots wslot .. wslot + nsplit - 1
};

constexpr int GEMM_PART = GBM * GBN;  // doubles per split-K partial (thread-fragment order)

struct DenseItem {
  int32_t kind;   // 0 exact GETRF, 1 GESSM strip, 2 TSTRF strip
  int32_t a, b;   // GETRF: diag block, step; GESSM/TSTRF: diag block, panel block
  int32_t c;      // GETRF: swaps allowed; GESSM: apply perm (FULL panel)
  int32_t begin;  // strip origin (GESSM tile column / TSTRF tile row)
  int32_t step;
};

struct TileItem {  // tiled GETRF work
  int32_t blk, step;
  int32_t kb;      // tile column origin of this sub-step
  int32_t r0, c0;  // tile origins (trsm: type in c0 < 0 ? ...) see kernels
  int32_t type;
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

// ------------------------------------------------------------- SSSSM ----
__device__ __forceinline__ void gemm_epilogue(const double (&acc)[4][4][2], const GemmTask& tk, const DevPools& P,
                                              int m0, int n0);
__device__ __forceinline__ void gemm_map_item(const GemmItem it, const GemmTask* __restrict__ tasks, const DevPools& P,
                                              double* sm) {
  const GemmTask tk = tasks[it.task];
  const BlockDev Lb = P.blk[tk.a], Ub = P.blk[tk.b];
  const double* __restrict__ A = P.vals + Lb.ent;
  const double* __restrict__ B = P.vals + Ub.ent;
  const int lda = Lb.nR, ldb = Ub.nR;
  const int M = Lb.nR, N = Ub.nC, K = tk.K;
  const int32_t* kL = tk.kL >= 0 ? P.maps + tk.kL : nullptr;
  const int32_t* kU = tk.kU >= 0 ? P.maps + tk.kU : nullptr;
  const int m0 = it.m0, n0 = it.n0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // inner-dimension chunks: all of them, or (k-chunk skipping) only those in which the
  // tile's L rows and U columns both hold pattern entries - the others multiply exact zeros
  const int nk = it.ke - it.ks;
  const int32_t* kcl = (it.nkc < 0 ? nullptr : P.kchunks + it.kc_off);
  const int kbase = it.ks;
  auto stageA = [&](int s) { return sm + s * (GBK * SA + GBN * SB); };
  auto stageB = [&](int s) { return sm + s * (GBK * SA + GBN * SB) + GBK * SA; };
  // The gathered inner indices of a chunk (the chunk list entry, then kL / kU) are two
  // dependent global loads: they are fetched one chunk ahead into registers, so the
  // cp.async issue of chunk kt + 2 never waits on them (they were the top stall)
  constexpr int NA = (GBK * GBM) / 256, NBL = (GBK * GBN) / 256;
  struct ChunkIdx {
    int k0;
    int colA[NA];
    int rowB;
  };
  auto fetch = [&](int kt, ChunkIdx& ci) {
    ci.k0 = (kcl ? __ldg(kcl + kbase + kt) : kbase + kt) * GBK;
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int kk = (tid + i * 256) / GBM, gk = ci.k0 + kk;
      ci.colA[i] = gk < K ? (kL ? __ldg(kL + gk) : gk) : -1;
    }
    const int gk = ci.k0 + (tid % GBK);
    ci.rowB = gk < K ? (kU ? __ldg(kU + gk) : gk) : -1;
  };
  auto issue = [&](int s, const ChunkIdx& ci) {
    double* As = stageA(s);
    double* Bs = stageB(s);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      const int idx = tid + i * 256;
      const int kk = idx / GBM, mm = idx % GBM;
      const int gr = m0 + mm;
      const bool v = gr < M && ci.colA[i] >= 0;
      cp_async8(As + kk * SA + mm, v ? A + static_cast<size_t>(ci.colA[i]) * lda + gr : A, v);
    }
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
      const int idx = tid + i * 256;
      const int nn = idx / GBK, kk = idx % GBK;
      const int gc = n0 + nn;
      const bool v = gc < N && ci.rowB >= 0;
      cp_async8(Bs + nn * SB + kk, v ? B + static_cast<size_t>(gc) * ldb + ci.rowB : B, v);
    }
  };
  ChunkIdx nxt;
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nk) {
      fetch(s, nxt);
      issue(s, nxt);
    }
    cp_async_commit();
  }
  if (GSTAGES - 1 < nk) fetch(GSTAGES - 1, nxt);
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    const int pf = kt + GSTAGES - 1;
    if (pf < nk) issue(pf % GSTAGES, nxt);
    cp_async_commit();
    if (pf + 1 < nk) fetch(pf + 1, nxt);  // consumed next iteration: its latency hides behind this chunk
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
  if (it.wslot >= 0) {  // split-K: the partial product goes to the workspace (thread-fragment order)
    double* W = P.gemm_ws + static_cast<size_t>(it.wslot) * GEMM_PART + tid * 32;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        W[(i * 4 + j) * 2] = acc[i][j][0];
        W[(i * 4 + j) * 2 + 1] = acc[i][j][1];
      }
    return;
  }
  gemm_epilogue(acc, tk, P, m0, n0);
}

// C(rows of L, cols of U) -= acc through the row / column scatter maps (a product row or
// column outside the target's support only carries exact zeros and is skipped)
__device__ __forceinline__ void gemm_epilogue(const double (&acc)[4][4][2], const GemmTask& tk, const DevPools& P,
                                              int m0, int n0) {
  const BlockDev Lb = P.blk[tk.a], Ub = P.blk[tk.b], Cb = P.blk[tk.c];
  double* Cv = P.vals + Cb.ent;
  const int ldc = Cb.nR, M = Lb.nR, N = Ub.nC;
  const int32_t* rmap = tk.rmap >= 0 ? P.maps + tk.rmap : nullptr;
  const int32_t* cmap = tk.cmap >= 0 ? P.maps + tk.cmap : nullptr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
  // per row group, its 8 target entries are all loaded before the first store (the maps
  // are injective, so no entry is read after another one is written; one dependent
  // read-modify-write per entry serialised 32 L2 round trips per thread)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + g;
    const int rr = r < M ? (rmap ? rmap[r] : r) : -1;  // < 0: row outside the product's support (exact zeros)
    int cc[4][2];
    double cv[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + 2 * t + h;
        cc[j][h] = (rr >= 0 && c < N) ? (cmap ? cmap[c] : c) : -1;
        cv[j][h] = cc[j][h] >= 0 ? Cv[static_cast<size_t>(cc[j][h]) * ldc + rr] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (cc[j][h] >= 0) Cv[static_cast<size_t>(cc[j][h]) * ldc + rr] = cv[j][h] - acc[i][j][h];
  }
}

__global__ void __launch_bounds__(256, 2) gemm_map_kernel(const GemmItem* __restrict__ items,
                                                       const GemmTask* __restrict__ tasks, DevPools P) {
  extern __shared__ double sm[];
  gemm_map_item(items[blockIdx.x], tasks, P, sm);
}

// Split-K reduction: one CTA per tile sums its partial products in slot order (a fixed
// order: deterministic) and applies the usual scatter epilogue.
__global__ void __launch_bounds__(256, 2) gemm_reduce_kernel(const GemmItem* __restrict__ items,
                                                          const GemmTask* __restrict__ tasks, DevPools P) {
  const GemmItem it = items[blockIdx.x];
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int sp = 0; sp < it.nsplit; ++sp) {
    const double* W = P.gemm_ws + static_cast<size_t>(it.wslot + sp) * GEMM_PART + threadIdx.x * 32;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j][0] += W[(i * 4 + j) * 2];
        acc[i][j][1] += W[(i * 4 + j) * 2 + 1];
      }
  }
  gemm_epilogue(acc, tasks[it.task], P, it.m0, it.n0);
}

// Throttled variant for the deferred (off-critical-path) SSSSM updates: a
// fixed number of CTAs loop over the items, so the deferred work never holds
// more than gridDim.x CTA slots while the next level's critical work runs.
__global__ void __launch_bounds__(256, 2) gemm_map_loop_kernel(const GemmItem* __restrict__ items, int n,
                                                            const GemmTask* __restrict__ tasks, DevPools P) {
  extern __shared__ double sm[];
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    gemm_map_item(items[i], tasks, P, sm);
    __syncthreads();  // the next item's prologue overwrites the pipeline stages
  }
}

// CTA-cooperative C -= A*B, operands read straight from global (L1/L2
// resident) with optional row/column gathers; warps own 32x32 tiles of C.
// A(r,k) = A[(acol ? acol[k] : k) * lda + (arow ? arow[r] : r)]
// B(k,c) = B[(bcol ? bcol[c] : c) * ldb + (brow ? brow[k] : k)]
__device__ void cta_gemm_sub(double* C, int ldc, const double* A, int lda, const int32_t* arow,
                             const int32_t* acol, const double* B, int ldb, const int32_t* brow,
                             const int32_t* bcol, int M, int N, int K) {
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
    int ar[4], bc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + i * 8 + g;
      ar[i] = r < M ? (arow ? arow[r] : r) : -1;
      const int c = n0 + i * 8 + g;
      bc[i] = c < N ? (bcol ? bcol[c] : c) : -1;
    }
    for (int k = 0; k < K; k += 4) {
      const int kk = k + t;
      const bool kv = kk < K;
      const int ak = kv ? (acol ? acol[kk] : kk) : 0;
      const int bk = kv ? (brow ? brow[kk] : kk) : 0;
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (kv && ar[i] >= 0) ? A[static_cast<size_t>(ak) * lda + ar[i]] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = (kv && bc[j] >= 0) ? B[static_cast<size_t>(bc[j]) * ldb + bk] : 0.0;
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

// ------------------------------------------- exact single-CTA GETRF ----
// Blocked right-looking LU with true partial pivoting confined to the block;
// used in dense-scratch mode (swaps) and with static pivoting.
__device__ void exact_getrf(const DenseItem& it, const DevPools& P, double* sh, double pivot_tol,
                            double static_eps) {
  const BlockDev D = P.blk[it.a];
  const int m = D.nrows, step = it.b;
  const bool can_swap = it.c != 0;
  double* A = P.vals + D.ent;
  int32_t* perm = P.perm + D.dg;
  double* colmax = sh;
  double* red_v = sh + m;
  int* red_r = reinterpret_cast<int*>(sh + m + 32);
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const bool use_static = !isnan(static_eps);
  for (int c = warp; c < m; c += nw) {
    const double* col = A + static_cast<size_t>(c) * m;
    double mx = 0.0;
    for (int r = lane; r < m; r += 32) mx = fmax(mx, fabs(col[r]));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) colmax[c] = mx;
  }
  for (int c = tid; c < m; c += nt) perm[c] = c;
  __syncthreads();
  for (int kb = 0; kb < m; kb += NB) {
    const int nb = min(NB, m - kb);
    for (int j = 0; j < nb; ++j) {
      const int c = kb + j;
      double* colc = A + static_cast<size_t>(c) * m;
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
        int action = -1;
        if (b == 0.0 || b < pivot_tol * colmax[c]) {
          if (use_static) {
            const double cur = colc[c];
            colc[c] = (cur == 0.0) ? static_eps : copysign(static_eps, cur);
          } else {
            record(&P.err[0], step, c);
          }
        } else if (br != c) {
          if (can_swap) {
            action = br;
            const int pt = perm[c];
            perm[c] = perm[br];
            perm[br] = pt;
          } else {
            record(&P.err[1], step, c);
          }
        }
        red_r[0] = action;
      }
      __syncthreads();
      const int sw = red_r[0];
      if (sw >= 0) {
        for (int q = tid; q < m; q += nt) {  // whole-row swap inside the block (factorize.py:57-61)
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
      const int pc = kb + nb - c - 1;
      const int rows = m - c - 1;
      for (int idx = tid; idx < pc * rows; idx += nt) {
        const int q = c + 1 + idx % rows;
        double* colj = A + static_cast<size_t>(c + 1 + idx / rows) * m;
        colj[q] = dsub_mul(colj[q], colc[q], colj[c]);
      }
      __syncthreads();
    }
    const int rest = m - kb - nb;
    if (rest <= 0) break;
    for (int jc = kb + nb + tid; jc < m; jc += nt) {
      double* col = A + static_cast<size_t>(jc) * m;
      for (int k = 0; k < nb; ++k) {
        const double xk = col[kb + k];
        const double* lk = A + static_cast<size_t>(kb + k) * m;
        for (int r = k + 1; r < nb; ++r) col[kb + r] = dsub_mul(col[kb + r], lk[kb + r], xk);
      }
    }
    __syncthreads();
    cta_gemm_sub(A + static_cast<size_t>(kb + nb) * m + kb + nb, m, A + static_cast<size_t>(kb) * m + kb + nb, m,
                 nullptr, nullptr, A + static_cast<size_t>(kb + nb) * m + kb, m, nullptr, nullptr, rest, rest, nb);
    __syncthreads();
  }
}

// ------------------------------------------------ panel solves (GESSM / TSTRF) ----
// GESSM: X tile (nR x nC, ld nR) rows = R_X (or all), L = unit lower of the FULL
// diagonal tile restricted to R_X.  One CTA per strip of STRIP tile columns.
__device__ void dense_gessm(const DenseItem& it, const DevPools& P, double* sh) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int m = D.nrows, nr = X.nR;
  const int32_t* R = X.store == STORE_RECT ? P.rlist + X.roff : nullptr;
  const double* L = P.vals + D.ent;
  double* Xs = P.vals + X.ent + static_cast<size_t>(it.begin) * nr;
  const int nc = min(STRIP, X.nC - it.begin);
  const int tid = threadIdx.x, nt = blockDim.x;
  if (it.c) {  // FULL panel in dense-scratch mode: apply the block row permutation
    const int32_t* perm = P.perm + D.dg;
    for (int j = 0; j < nc; ++j) {
      double* col = Xs + static_cast<size_t>(j) * nr;
      for (int r = tid; r < nr; r += nt) sh[r] = col[perm[r]];
      __syncthreads();
      for (int r = tid; r < nr; r += nt) col[r] = sh[r];
      __syncthreads();
    }
  }
  for (int kb = 0; kb < nr; kb += NB) {
    const int nb = min(NB, nr - kb);
    for (int j = tid; j < nc; j += nt) {
      double* col = Xs + static_cast<size_t>(j) * nr;
      for (int k = 0; k < nb; ++k) {
        const double xk = col[kb + k];
        const int gk = R ? R[kb + k] : kb + k;
        const double* lk = L + static_cast<size_t>(gk) * m;
        for (int r = k + 1; r < nb; ++r) {
          const int gr = R ? R[kb + r] : kb + r;
          col[kb + r] = dsub_mul(col[kb + r], lk[gr], xk);
        }
      }
    }
    __syncthreads();
    const int rest = nr - kb - nb;
    if (rest > 0) {
      if (R)
        cta_gemm_sub(Xs + kb + nb, nr, L, m, R + kb + nb, R + kb, Xs + kb, nr, nullptr, nullptr, rest, nc, nb);
      else
        cta_gemm_sub(Xs + kb + nb, nr, L + static_cast<size_t>(kb) * m + kb + nb, m, nullptr, nullptr, Xs + kb, nr,
                     nullptr, nullptr, rest, nc, nb);
    }
    __syncthreads();
  }
}

// TSTRF: X tile (nR x nC), columns = C_X (or all), U = upper of the FULL
// diagonal tile restricted to C_X.  One CTA per strip of STRIP tile rows.
__device__ void dense_tstrf(const DenseItem& it, const DevPools& P) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int m = D.nrows, ld = X.nR, ncx = X.nC;
  const int32_t* Cl = X.store == STORE_RECT ? P.clist + X.coff : nullptr;
  const double* U = P.vals + D.ent;
  double* Xs = P.vals + X.ent + it.begin;
  const int nr = min(STRIP, ld - it.begin);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int kb = 0; kb < ncx; kb += NB) {
    const int nb = min(NB, ncx - kb);
    for (int q = tid; q < nr; q += nt) {
      for (int k = 0; k < nb; ++k) {
        const int gk = Cl ? Cl[kb + k] : kb + k;
        double* xk = Xs + static_cast<size_t>(kb + k) * ld + q;
        const double v = __ddiv_rn(*xk, U[static_cast<size_t>(gk) * m + gk]);
        *xk = v;
        for (int jj = k + 1; jj < nb; ++jj) {
          const int gj = Cl ? Cl[kb + jj] : kb + jj;
          double* xj = Xs + static_cast<size_t>(kb + jj) * ld + q;
          *xj = dsub_mul(*xj, v, U[static_cast<size_t>(gj) * m + gk]);
        }
      }
    }
    __syncthreads();
    const int rest = ncx - kb - nb;
    if (rest > 0) {
      if (Cl)
        cta_gemm_sub(Xs + static_cast<size_t>(kb + nb) * ld, ld, Xs + static_cast<size_t>(kb) * ld, ld, nullptr,
                     nullptr, U, m, Cl + kb, Cl + kb + nb, nr, rest, nb);
      else
        cta_gemm_sub(Xs + static_cast<size_t>(kb + nb) * ld, ld, Xs + static_cast<size_t>(kb) * ld, ld, nullptr,
                     nullptr, U + static_cast<size_t>(kb + nb) * m + kb, m, nullptr, nullptr, nr, rest, nb);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) panel_kernel(const DenseItem* __restrict__ items, DevPools P,
                                                    double pivot_tol, double static_eps) {
  extern __shared__ double sh[];
  const DenseItem it = items[blockIdx.x];
  if (it.kind == 0) exact_getrf(it, P, sh, pivot_tol, static_eps);
  else if (it.kind == 1) dense_gessm(it, P, sh);
  else dense_tstrf(it, P);
}

// ---------------------------------------------------------- tiled GETRF ----
// colmax / reset: item.blk, item.c0 = first column of a 64-column chunk.
__global__ void __launch_bounds__(256) getrf_colmax_kernel(const TileItem* __restrict__ items, DevPools P) {
  const TileItem it = items[blockIdx.x];
  const BlockDev D = P.blk[it.blk];
  const int m = D.nrows;
  const double* A = P.vals + D.ent;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = it.c0 + warp; c < min(m, it.c0 + TS); c += 8) {
    const double* col = A + static_cast<size_t>(c) * m;
    double mx = 0.0;
    for (int r = lane; r < m; r += 32) mx = fmax(mx, fabs(col[r]));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      P.colmax[D.dg + c] = mx;
      P.bmax[D.dg + c] = 0ull;
      P.perm[D.dg + c] = c;
    }
  }
}

// factor the diagonal tile (kb,kb) in shared memory, no row exchange;
// records max |d_qc| of in-tile rows below the diagonal (before scaling).
__global__ void __launch_bounds__(256) tile_getrf_kernel(const TileItem* __restrict__ items, DevPools P) {
  __shared__ double T[TS * TSP];
  const TileItem it = items[blockIdx.x];
  const BlockDev D = P.blk[it.blk];
  const int m = D.nrows, kb = it.kb, nb = min(TS, m - kb);
  double* A = P.vals + D.ent + static_cast<size_t>(kb) * m + kb;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const int r = idx % nb, c = idx / nb;
    T[c * TSP + r] = A[static_cast<size_t>(c) * m + r];
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double u = T[j * TSP + j];
    double mx = 0.0;
    for (int r = j + 1 + tid; r < nb; r += 256) {
      const double v = T[j * TSP + r];
      mx = fmax(mx, fabs(v));
      T[j * TSP + r] = __ddiv_rn(v, u);
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.0) atomic_max_nonneg(&P.bmax[D.dg + kb + j], mx);
    __syncthreads();
    const int rows = nb - j - 1;
    for (int idx = tid; idx < rows * rows; idx += 256) {
      const int r = j + 1 + idx % rows, c = j + 1 + idx / rows;
      T[c * TSP + r] = dsub_mul(T[c * TSP + r], T[j * TSP + r], T[c * TSP + j]);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nb * nb; idx += 256) {
    const int r = idx % nb, c = idx / nb;
    A[static_cast<size_t>(c) * m + r] = T[c * TSP + r];
  }
}

// type 0: L tile (rows r0.., cols kb..) <- X U_kk^{-1}, records max |d_qc| before division.
// type 1: U tile (rows kb.., cols c0..) <- L_kk^{-1} X.
constexpr int TRSM_SMEM = (2 * TS * TSP + TS) * 8;
constexpr int TGEMM_SMEM = 2 * TS * (TS + 4) * 8;

__global__ void __launch_bounds__(128) tile_trsm_kernel(const TileItem* __restrict__ items, DevPools P) {
  extern __shared__ double tsm[];
  double* Dk = tsm;
  double* X = tsm + TS * TSP;
  unsigned long long* cm = reinterpret_cast<unsigned long long*>(tsm + 2 * TS * TSP);
  const TileItem it = items[blockIdx.x];
  const BlockDev D = P.blk[it.blk];
  const int m = D.nrows, kb = it.kb, nb = min(TS, m - kb);
  const double* A = P.vals + D.ent;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < nb * nb; idx += 128) {
    const int r = idx % nb, c = idx / nb;
    Dk[c * TSP + r] = A[static_cast<size_t>(kb + c) * m + kb + r];
  }
  if (it.type == 0) {
    const int r0 = it.r0, nr = min(TS, m - r0);
    double* G = P.vals + D.ent + static_cast<size_t>(kb) * m + r0;
    for (int idx = tid; idx < nr * nb; idx += 128) {
      const int r = idx % nr, c = idx / nr;
      X[c * TSP + r] = G[static_cast<size_t>(c) * m + r];
    }
    for (int c = tid; c < TS; c += 128) cm[c] = 0ull;
    __syncthreads();
    if (tid < nr) {
      for (int j = 0; j < nb; ++j) {
        const double d = X[j * TSP + tid];
        if (d != 0.0) atomicMax(&cm[j], static_cast<unsigned long long>(__double_as_longlong(fabs(d))));
        const double x = __ddiv_rn(d, Dk[j * TSP + j]);
        X[j * TSP + tid] = x;
        for (int jj = j + 1; jj < nb; ++jj) X[jj * TSP + tid] = dsub_mul(X[jj * TSP + tid], x, Dk[jj * TSP + j]);
      }
    }
    __syncthreads();
    for (int c = tid; c < nb; c += 128)
      if (cm[c]) atomicMax(&P.bmax[D.dg + kb + c], cm[c]);
    for (int idx = tid; idx < nr * nb; idx += 128) {
      const int r = idx % nr, c = idx / nr;
      G[static_cast<size_t>(c) * m + r] = X[c * TSP + r];
    }
  } else {
    const int c0 = it.c0, nc = min(TS, m - c0);
    double* G = P.vals + D.ent + static_cast<size_t>(c0) * m + kb;
    for (int idx = tid; idx < nb * nc; idx += 128) {
      const int r = idx % nb, c = idx / nb;
      X[c * TSP + r] = G[static_cast<size_t>(c) * m + r];
    }
    __syncthreads();
    if (tid < nc) {
      for (int k = 0; k < nb; ++k) {
        const double xk = X[tid * TSP + k];
        for (int r = k + 1; r < nb; ++r) X[tid * TSP + r] = dsub_mul(X[tid * TSP + r], Dk[k * TSP + r], xk);
      }
    }
    __syncthreads();
    for (int idx = tid; idx < nb * nc; idx += 128) {
      const int r = idx % nb, c = idx / nb;
      G[static_cast<size_t>(c) * m + r] = X[c * TSP + r];
    }
  }
}

// trailing update of tile (r0, c0) -= L(r0, kb) * U(kb, c0): 64x64x64 on DMMA, 4 warps of 32x32.
__global__ void __launch_bounds__(128) tile_gemm_kernel(const TileItem* __restrict__ items, DevPools P) {
  extern __shared__ double gsm[];
  double* As = gsm;                // [k][r]
  double* Bs = gsm + TS * (TS + 4);  // [c][k]
  const TileItem it = items[blockIdx.x];
  const BlockDev D = P.blk[it.blk];
  const int m = D.nrows, kb = it.kb, nb = min(TS, m - kb);
  const int r0 = it.r0, c0 = it.c0, nr = min(TS, m - r0), nc = min(TS, m - c0);
  double* A = P.vals + D.ent;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  constexpr int S = TS + 4;
  for (int idx = tid; idx < TS * TS; idx += 128) {
    const int r = idx % TS, k = idx / TS;
    const bool v = r < nr && k < nb;
    cp_async8(As + k * S + r, v ? A + static_cast<size_t>(kb + k) * m + r0 + r : A, v);
    const int kk = idx % TS, c = idx / TS;
    const bool w = kk < nb && c < nc;
    cp_async8(Bs + c * S + kk, w ? A + static_cast<size_t>(c0 + c) * m + kb + kk : A, w);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k = 0; k < TS; k += 4) {
    double a[4], b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = As[(k + t) * S + wm + i * 8 + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + g) * S + k + t];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm + i * 8 + g;
    if (r >= nr) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn + j * 8 + 2 * t + h;
        if (c < nc) A[static_cast<size_t>(c0 + c) * m + r0 + r] -= acc[i][j][h];
      }
    }
  }
}

// pivot verdict per column: piv = max(|u_cc|, below max); ZeroPivot / swap.
__global__ void __launch_bounds__(256) getrf_finalize_kernel(const TileItem* __restrict__ items, DevPools P,
                                                             double pivot_tol) {
  const TileItem it = items[blockIdx.x];
  const BlockDev D = P.blk[it.blk];
  const int m = D.nrows;
  const double* A = P.vals + D.ent;
  for (int c = it.c0 + threadIdx.x; c < min(m, it.c0 + 256); c += blockDim.x) {
    const double u = fabs(A[static_cast<size_t>(c) * m + c]);
    const double below = __longlong_as_double(static_cast<long long>(P.bmax[D.dg + c]));
    const double piv = fmax(u, below);
    if (piv == 0.0 || piv < pivot_tol * P.colmax[D.dg + c] || isnan(u)) record(&P.err[0], it.step, c);
    else if (below > u) record(&P.err[1], it.step, c);
  }
}

}  // namespace lbk
