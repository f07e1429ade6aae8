// lbk_device.cu — sm_100a block-LU engine behind the C-ABI of include/lbk.h.
//
// Replaces the numerical factorization of the reference,
//   lublock.factorize.factorize(grid, tree, ...)   pkg/src/lublock/factorize.py:245-384
// with a level-by-level device scheduler: every dependency level of the
// task DAG (grid.py:223-378) becomes ONE kernel launch over a work list of
// (task, column/row range) items; all levels are captured once into a CUDA
// graph and replayed.
//
// Block storage (uploaded once; the filled pattern is elimination-closed so
// it never changes, grid.py:3-5): every stored block is local-index CSC
// (int32 col_ptr, int32 rows, f64 values) in pooled arrays, plus a CSR
// transpose index (row_ptr, col, pos) used by the row-oriented TSTRF.
//
// Kernels (one warp per column / row, dense accumulator of the block's
// span in shared memory — the scatter/gather scheme of SPEC factorize
// DESIGN DECISIONS):
//   GETRF  left-looking on the diagonal block, columns grouped by their
//          intra-block dependency level, block-local partial pivoting with
//          the reference's first-argmax / tolerance / static-pivot rules
//          (factorize.py:38-78);
//   GESSM  column forward substitution with the unit-lower L_ii
//          (factorize.py:98-109, 326-337);
//   TSTRF  row back substitution with U_ii (factorize.py:112-130, 338-345);
//   SSSSM  Gustavson column SpGEMM into the fixed target pattern
//          (factorize.py:307-325).
// GETRF/GESSM/TSTRF use separately rounded multiply and subtract / true
// division, in the reference's order, so they reproduce its bits; SSSSM
// accumulates with FMA (the reference's dgemm order is unpinned anyway).

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <new>
#include <string>
#include <vector>

#include "../../include/lbk.h"

namespace {

constexpr int KIND_GETRF = 0, KIND_GESSM = 1, KIND_TSTRF = 2, KIND_SSSSM = 3;
constexpr int64_t NO_ERR = std::numeric_limits<int64_t>::max();
constexpr int MAX_SMEM = 227 * 1024;

struct BlockDev {
  int32_t nrows, ncols;
  int32_t full;    // 1 if the stored pattern is the full nrows x ncols rectangle
  int32_t nlev;    // GETRF: number of intra-block column levels
  int64_t cp;      // offset into colptr pool (ncols+1 entries)
  int64_t ent;     // offset into rows / vals pools
  int64_t rp;      // offset into csr rowptr pool (nrows+1 entries)
  int64_t dg;      // diagonal blocks: offset into diag_csc / diag_csr / perm pools
  int64_t lvc;     // diagonal blocks: offset into level-column pool
  int64_t lvp;     // diagonal blocks: offset into level-pointer pool (nlev+1 entries)
};

struct Item {
  int32_t kind;
  int32_t a, b, c;  // block ids (see make_items)
  int32_t begin, end;
};

struct DevPools {
  const BlockDev* blk;
  const int32_t* colptr;
  const int32_t* rows;
  double* vals;
  const int32_t* csr_ptr;
  const int32_t* csr_col;
  const int32_t* csr_pos;
  const int32_t* diag_csc;  // per diagonal-block column: local CSC index of (c,c)
  const int32_t* diag_csr;  // per diagonal-block row: local CSR index of (r,r)
  const int32_t* lv_cols;
  const int32_t* lv_ptr;
  int32_t* perm;            // per diagonal-block row: local permutation
  unsigned long long* err;  // [0] zero-pivot key, [1] swap key (block<<32 | col), min wins
};

__device__ __forceinline__ double dsub_mul(double x, double l, double u) {
  // x - (l*u) with both operations separately rounded, like numpy's x -= outer(l, u)
  return __dsub_rn(x, __dmul_rn(l, u));
}

__device__ __forceinline__ void record(unsigned long long* w, int block, int col) {
  unsigned long long key = (static_cast<unsigned long long>(block) << 32) | static_cast<unsigned>(col);
  atomicMin(w, key);
}

// ---------------------------------------------------------------- SSSSM ----
// C(k,j) -= L(k,i) U(i,j); one warp per target column.
__device__ void ssssm_item(const Item& it, const DevPools& P, double* acc) {
  const BlockDev L = P.blk[it.a], U = P.blk[it.b], C = P.blk[it.c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* Lcp = P.colptr + L.cp;
  const int32_t* Lr = P.rows + L.ent;
  const double* Lv = P.vals + L.ent;
  const int32_t* Ucp = P.colptr + U.cp;
  const int32_t* Ur = P.rows + U.ent;
  const double* Uv = P.vals + U.ent;
  const int32_t* Ccp = P.colptr + C.cp;
  const int32_t* Cr = P.rows + C.ent;
  double* Cv = P.vals + C.ent;
  for (int c = it.begin + warp; c < it.end; c += nw) {
    const int u0 = Ucp[c], u1 = Ucp[c + 1];
    if (u0 == u1) continue;
    const int c0 = Ccp[c], c1 = Ccp[c + 1];
    for (int e = c0 + lane; e < c1; e += 32) acc[Cr[e]] = 0.0;
    __syncwarp();
    for (int e = u0; e < u1; ++e) {
      const int r = Ur[e];
      const double u = Uv[e];
      const int l0 = Lcp[r], l1 = Lcp[r + 1];
      for (int f = l0 + lane; f < l1; f += 32) acc[Lr[f]] = fma(Lv[f], u, acc[Lr[f]]);
      __syncwarp();
    }
    for (int e = c0 + lane; e < c1; e += 32) Cv[e] -= acc[Cr[e]];
    __syncwarp();
  }
}

// ---------------------------------------------------------------- GESSM ----
// X(i,j) <- L_ii^{-1} P_i X(i,j); one warp per column of X.
__device__ void gessm_item(const Item& it, const DevPools& P, double* acc) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* Dcp = P.colptr + D.cp;
  const int32_t* Dr = P.rows + D.ent;
  const double* Dv = P.vals + D.ent;
  const int32_t* dpos = P.diag_csc + D.dg;
  const int32_t* perm = P.perm + D.dg;
  const int32_t* Xcp = P.colptr + X.cp;
  const int32_t* Xr = P.rows + X.ent;
  double* Xv = P.vals + X.ent;
  const bool permute = (it.c != 0);  // host sets c=1 when X is full and perms may be non-identity
  for (int c = it.begin + warp; c < it.end; c += nw) {
    const int x0 = Xcp[c], x1 = Xcp[c + 1];
    if (x0 == x1) continue;
    if (permute) {
      // full column: new[r] = old[perm[r]]
      for (int e = x0 + lane; e < x1; e += 32) acc[Xr[e]] = Xv[x0 + perm[Xr[e]]];
    } else {
      for (int e = x0 + lane; e < x1; e += 32) acc[Xr[e]] = Xv[e];
    }
    __syncwarp();
    for (int e = x0; e < x1; ++e) {
      const int k = Xr[e];
      const double xk = acc[k];
      const int f1 = Dcp[k + 1];
      for (int f = dpos[k] + 1 + lane; f < f1; f += 32) {
        const int q = Dr[f];
        acc[q] = dsub_mul(acc[q], Dv[f], xk);
      }
      __syncwarp();
    }
    for (int e = x0 + lane; e < x1; e += 32) Xv[e] = acc[Xr[e]];
    __syncwarp();
  }
}

// ---------------------------------------------------------------- TSTRF ----
// X(k,i) <- X(k,i) U_ii^{-1}; one warp per row of X (CSR transpose index).
__device__ void tstrf_item(const Item& it, const DevPools& P, double* acc) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Dv = P.vals + D.ent;
  const int32_t* Dcsc = P.diag_csc + D.dg;
  const int32_t* Drow = P.diag_csr + D.dg;
  const int32_t* Drp = P.csr_ptr + D.rp;
  const int32_t* Dcc = P.csr_col + D.ent;
  const int32_t* Dcpos = P.csr_pos + D.ent;
  const int32_t* Xrp = P.csr_ptr + X.rp;
  const int32_t* Xcc = P.csr_col + X.ent;
  const int32_t* Xcpos = P.csr_pos + X.ent;
  double* Xv = P.vals + X.ent;
  for (int q = it.begin + warp; q < it.end; q += nw) {
    const int r0 = Xrp[q], r1 = Xrp[q + 1];
    if (r0 == r1) continue;
    for (int e = r0 + lane; e < r1; e += 32) acc[Xcc[e]] = Xv[Xcpos[e]];
    __syncwarp();
    for (int e = r0; e < r1; ++e) {
      const int k = Xcc[e];
      const double xk = __ddiv_rn(acc[k], Dv[Dcsc[k]]);
      __syncwarp();
      if (lane == 0) acc[k] = xk;
      const int g1 = Drp[k + 1];
      for (int g = Drow[k] + 1 + lane; g < g1; g += 32) {
        const int j = Dcc[g];
        acc[j] = dsub_mul(acc[j], xk, Dv[Dcpos[g]]);
      }
      __syncwarp();
    }
    for (int e = r0 + lane; e < r1; e += 32) Xv[Xcpos[e]] = acc[Xcc[e]];
    __syncwarp();
  }
}

// ---------------------------------------------------------------- GETRF ----
// Left-looking LU of the diagonal block; the whole CTA works on one block,
// warps take the columns of one intra-block dependency level at a time.
__device__ void getrf_item(const Item& it, const DevPools& P, double* acc, double pivot_tol,
                           double static_eps) {
  const BlockDev D = P.blk[it.a];
  const int step = it.b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* Dcp = P.colptr + D.cp;
  const int32_t* Dr = P.rows + D.ent;
  double* Dv = P.vals + D.ent;
  const int32_t* dpos = P.diag_csc + D.dg;
  int32_t* perm = P.perm + D.dg;
  const int32_t* lvc = P.lv_cols + D.lvc;
  const int32_t* lvp = P.lv_ptr + D.lvp;
  const bool use_static = !isnan(static_eps);
  const int m = D.nrows;
  for (int r = threadIdx.x; r < m; r += blockDim.x) perm[r] = r;
  __syncthreads();
  for (int lv = 0; lv < D.nlev; ++lv) {
    for (int idx = lvp[lv] + warp; idx < lvp[lv + 1]; idx += nw) {
      const int c = lvc[idx];
      const int d0 = Dcp[c], d1 = Dcp[c + 1], dp = dpos[c];
      double cmax = 0.0;
      for (int e = d0 + lane; e < d1; e += 32) {
        const double v = Dv[e];
        acc[Dr[e]] = v;
        cmax = fmax(cmax, fabs(v));
      }
      for (int o = 16; o; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
      __syncwarp();
      // left-looking updates from the finished columns k < c in U(:,c)
      for (int e = d0; e < dp; ++e) {
        const int k = Dr[e];
        const double xk = acc[k];
        const int f1 = Dcp[k + 1];
        for (int f = dpos[k] + 1 + lane; f < f1; f += 32) {
          const int q = Dr[f];
          acc[q] = dsub_mul(acc[q], Dv[f], xk);
        }
        __syncwarp();
      }
      // pivot search on rows >= c: first maximum in row order
      double best = -1.0;
      int brow = m;
      for (int e = dp + lane; e < d1; e += 32) {
        const int q = Dr[e];
        const double a = fabs(acc[q]);
        if (a > best || (a == best && q < brow)) { best = a; brow = q; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
        if (ob > best || (ob == best && orow < brow)) { best = ob; brow = orow; }
      }
      if (best == 0.0 || best < pivot_tol * cmax) {
        if (use_static) {
          if (lane == 0) {
            const double cur = acc[c];
            acc[c] = (cur == 0.0) ? static_eps : copysign(static_eps, cur);
          }
        } else if (lane == 0) {
          record(&P.err[0], step, c);
        }
      } else if (brow != c) {
        if (it.c) {
          // swap rows c and brow across the whole block (factorize.py:57-61):
          // finished L columns and not-yet-processed columns alike
          const int ncol = D.ncols;
          for (int j = lane; j < ncol; j += 32) {
            if (j == c) continue;
            double* col = Dv + Dcp[j];
            const double t = col[c];
            col[c] = col[brow];
            col[brow] = t;
          }
          if (lane == 0) {
            const double t = acc[c];
            acc[c] = acc[brow];
            acc[brow] = t;
            const int pt = perm[c];
            perm[c] = perm[brow];
            perm[brow] = pt;
          }
        } else if (lane == 0) {
          record(&P.err[1], step, c);
        }
      }
      __syncwarp();
      const double piv = acc[c];
      for (int e = dp + 1 + lane; e < d1; e += 32) {
        const int q = Dr[e];
        acc[q] = __ddiv_rn(acc[q], piv);
      }
      __syncwarp();
      for (int e = d0 + lane; e < d1; e += 32) Dv[e] = acc[Dr[e]];
      __syncwarp();
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) level_kernel(const Item* __restrict__ items, DevPools P,
                                                    int acc_len, double pivot_tol, double static_eps) {
  extern __shared__ double smem[];
  const Item it = items[blockIdx.x];
  double* acc = smem + static_cast<size_t>(threadIdx.x >> 5) * acc_len;
  switch (it.kind) {
    case KIND_SSSSM: ssssm_item(it, P, acc); break;
    case KIND_GESSM: gessm_item(it, P, acc); break;
    case KIND_TSTRF: tstrf_item(it, P, acc); break;
    default: getrf_item(it, P, acc, pivot_tol, static_eps); break;
  }
}

}  // namespace

#include "lbk_dense.cuh"

namespace {

// ------------------------------------------------------------------ host ----

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t count) {
    n = count;
    return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  }
  cudaError_t upload(const std::vector<T>& v) {
    cudaError_t e = alloc(v.size());
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
  }
};

struct Level {
  int64_t item_off;   // generic (sparse) items
  int32_t nitems;
  int32_t warps;
  int32_t acc_len;
  int64_t gemm_off;   // dense SSSSM tiles
  int32_t ngemm;
  int64_t dense_off;  // dense GETRF / GESSM / TSTRF items
  int32_t ndense;
  int32_t dense_smem; // bytes
  int32_t dense_threads;
};

}  // namespace

struct lbk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // plan
  int64_t n = 0, p = 0, nblocks = 0, nnz = 0;
  std::vector<int64_t> diag_block;  // per step i: block id of (i,i)
  std::vector<int64_t> diag_dg;     // per step i: dg offset
  std::vector<int32_t> span;        // per step i
  std::vector<BlockDev> hblk;
  std::vector<Level> levels;
  int64_t total_items = 0;
  double plan_pivot_tol = NAN, plan_static_eps = NAN;
  // device
  DevBuf<BlockDev> blk;
  DevBuf<int32_t> colptr, rows, csr_ptr, csr_col, csr_pos, diag_csc, diag_csr, lv_cols, lv_ptr, perm;
  DevBuf<double> vals, vals0;
  DevBuf<Item> items;
  DevBuf<lbk_dense::GemmItem> gitems;
  DevBuf<lbk_dense::DenseItem> ditems;
  DevBuf<unsigned long long> err;
  int64_t ndiag_rows = 0;
  int64_t total_gemm = 0, total_dense = 0;
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
};

namespace {

int fail(lbk_status* st, int code, const char* msg) {
  if (st) {
    st->code = code;
    st->block = -1;
    st->col = -1;
    std::snprintf(st->msg, sizeof(st->msg), "%s", msg);
  }
  return code;
}

int cuda_fail(lbk_status* st, cudaError_t e, const char* where) {
  char buf[256];
  std::snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  return fail(st, e == cudaErrorMemoryAllocation ? LBK_ERR_OOM : LBK_ERR_CUDA, buf);
}

#define LBK_CUDA(call, st)                                   \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail((st), e_, #call); \
  } while (0)

void ok(lbk_status* st) {
  if (st) {
    st->code = LBK_OK;
    st->block = -1;
    st->col = -1;
    st->msg[0] = 0;
  }
}

DevPools pools(lbk_ctx* c) {
  DevPools P;
  P.blk = c->blk.p;
  P.colptr = c->colptr.p;
  P.rows = c->rows.p;
  P.vals = c->vals.p;
  P.csr_ptr = c->csr_ptr.p;
  P.csr_col = c->csr_col.p;
  P.csr_pos = c->csr_pos.p;
  P.diag_csc = c->diag_csc.p;
  P.diag_csr = c->diag_csr.p;
  P.lv_cols = c->lv_cols.p;
  P.lv_ptr = c->lv_ptr.p;
  P.perm = c->perm.p;
  P.err = c->err.p;
  return P;
}

int choose_warps(int acc_len) {
  int w = MAX_SMEM / (acc_len * 8);
  return std::max(1, std::min(4, w));
}

}  // namespace

extern "C" {

int lbk_create(lbk_ctx** out, int device, lbk_status* st) {
  auto* c = new (std::nothrow) lbk_ctx();
  if (!c) return fail(st, LBK_ERR_OOM, "ctx alloc");
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lbk_dense::dgemm_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             lbk_dense::GEMM_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(lbk_dense::dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
    e = cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join[k], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(st, e, "lbk_create");
  }
  *out = c;
  ok(st);
  return 0;
}

void lbk_destroy(lbk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  for (int k = 0; k < 2; ++k) {
    if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
    if (c->join[k]) cudaEventDestroy(c->join[k]);
  }
  if (c->fork) cudaEventDestroy(c->fork);
  delete c;
}

// Build the device plan: block pools, transpose indices, intra-block column
// levels of the diagonal blocks, and the per-level work lists.
int lbk_plan(lbk_ctx* c, int64_t n, int64_t p, const int64_t* positions, int64_t nblocks,
             const int64_t* table, const int64_t* colptr, const int64_t* rowidx, int64_t ntasks,
             const int8_t* kinds, const int32_t* steps, const int32_t* trows, const int32_t* tcols,
             const int32_t* tlevels, const int64_t* costs, int32_t chunk, int32_t flags,
             lbk_status* st) {
  if (!c) return fail(st, LBK_ERR_BAD_ARG, "null ctx");
  LBK_CUDA(cudaSetDevice(c->device), st);
  const int64_t nb = nblocks;
  const int64_t* T_bi = table;
  const int64_t* T_bj = table + nb;
  const int64_t* T_nr = table + 2 * nb;
  const int64_t* T_nc = table + 3 * nb;
  const int64_t* T_nz = table + 4 * nb;
  const int64_t* T_cp = table + 5 * nb;
  const int64_t* T_ent = table + 6 * nb;
  c->n = n;
  c->p = p;
  c->nblocks = nb;
  int64_t nnz = 0, ncp = 0, nrp = 0;
  for (int64_t b = 0; b < nb; ++b) {
    nnz += T_nz[b];
    ncp += T_nc[b] + 1;
    nrp += T_nr[b] + 1;
  }
  c->nnz = nnz;
  std::vector<int64_t> bid(static_cast<size_t>(p * p), -1);
  for (int64_t b = 0; b < nb; ++b) bid[T_bi[b] * p + T_bj[b]] = b;
  for (int64_t i = 0; i < p; ++i)
    if (bid[i * p + i] < 0) return fail(st, LBK_ERR_DIM_MISMATCH, "missing diagonal block");
  try {
    std::vector<BlockDev> hb(nb);
    std::vector<int32_t> hcp(ncp), hrows(nnz), hrp(nrp), hcc(nnz), hcpos(nnz);
    std::vector<int32_t> hdcsc, hdcsr, hlvc, hlvp;
    c->diag_block.assign(p, -1);
    c->diag_dg.assign(p, 0);
    c->span.assign(p, 0);
    int64_t cpo = 0, ento = 0, rpo = 0;
    for (int64_t b = 0; b < nb; ++b) {
      BlockDev& d = hb[b];
      d.nrows = static_cast<int32_t>(T_nr[b]);
      d.ncols = static_cast<int32_t>(T_nc[b]);
      d.full = (T_nz[b] == T_nr[b] * T_nc[b]) ? 1 : 0;
      d.nlev = 0;
      d.cp = cpo;
      d.ent = ento;
      d.rp = rpo;
      d.dg = d.lvc = d.lvp = 0;
      const int64_t* scp = colptr + T_cp[b];
      const int64_t* sri = rowidx + T_ent[b];
      const int64_t nzb = T_nz[b];
      for (int64_t k = 0; k <= d.ncols; ++k) hcp[cpo + k] = static_cast<int32_t>(scp[k]);
      for (int64_t e = 0; e < nzb; ++e) hrows[ento + e] = static_cast<int32_t>(sri[e]);
      // CSR transpose: rows ascending, columns ascending within a row
      int32_t* rp = &hrp[rpo];
      std::fill(rp, rp + d.nrows + 1, 0);
      for (int64_t e = 0; e < nzb; ++e) rp[sri[e] + 1]++;
      for (int r = 0; r < d.nrows; ++r) rp[r + 1] += rp[r];
      std::vector<int32_t> w(rp, rp + d.nrows);
      for (int col = 0; col < d.ncols; ++col)
        for (int64_t e = scp[col]; e < scp[col + 1]; ++e) {
          const int32_t g = w[sri[e]]++;
          hcc[ento + g] = col;
          hcpos[ento + g] = static_cast<int32_t>(e);
        }
      if (T_bi[b] == T_bj[b]) {
        const int64_t i = T_bi[b];
        c->diag_block[i] = b;
        c->span[i] = d.nrows;
        d.dg = static_cast<int64_t>(hdcsc.size());
        c->diag_dg[i] = d.dg;
        hdcsc.resize(hdcsc.size() + d.ncols, -1);
        hdcsr.resize(hdcsr.size() + d.nrows, -1);
        for (int col = 0; col < d.ncols; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
            if (sri[e] == col) hdcsc[d.dg + col] = static_cast<int32_t>(e);
        for (int r = 0; r < d.nrows; ++r)
          for (int32_t g = rp[r]; g < rp[r + 1]; ++g)
            if (hcc[ento + g] == r) hdcsr[d.dg + r] = g;
        for (int col = 0; col < d.ncols; ++col)
          if (hdcsc[d.dg + col] < 0 || hdcsr[d.dg + col] < 0)
            return fail(st, LBK_ERR_DIM_MISMATCH, "diagonal block without full diagonal");
        // intra-block column levels: lev[c] = 1 + max lev[k] over k<c in U(:,c)
        std::vector<int32_t> lev(d.ncols, 0);
        int32_t nlev = 0;
        for (int col = 0; col < d.ncols; ++col) {
          int32_t lv = 0;
          if (d.full) {
            lv = col;  // dense mode: strictly sequential (row swaps touch every column)
          } else {
            for (int64_t e = scp[col]; e < scp[col + 1] && sri[e] < col; ++e)
              lv = std::max(lv, lev[sri[e]] + 1);
          }
          lev[col] = lv;
          nlev = std::max(nlev, lv + 1);
        }
        d.nlev = nlev;
        d.lvp = static_cast<int64_t>(hlvp.size());
        d.lvc = static_cast<int64_t>(hlvc.size());
        std::vector<int32_t> cnt(nlev + 1, 0);
        for (int col = 0; col < d.ncols; ++col) cnt[lev[col] + 1]++;
        for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
        hlvp.insert(hlvp.end(), cnt.begin(), cnt.end());
        std::vector<int32_t> order(d.ncols);
        std::vector<int32_t> wp(cnt.begin(), cnt.end() - 1);
        for (int col = 0; col < d.ncols; ++col) order[wp[lev[col]]++] = col;
        hlvc.insert(hlvc.end(), order.begin(), order.end());
      }
      cpo += d.ncols + 1;
      ento += nzb;
      rpo += d.nrows + 1;
    }
    c->ndiag_rows = static_cast<int64_t>(hdcsc.size());
    // per-level work lists
    int32_t nlevels = 0;
    for (int64_t t = 0; t < ntasks; ++t) nlevels = std::max(nlevels, tlevels[t] + 1);
    std::vector<std::vector<Item>> per(nlevels);
    std::vector<int32_t> lvl_acc(nlevels, 1);
    if (chunk < 1) chunk = 8;
    auto add_range = [&](int32_t lv, Item base, int32_t count) {
      for (int32_t s = 0; s < count; s += chunk) {
        Item it = base;
        it.begin = s;
        it.end = std::min(count, s + chunk);
        per[lv].push_back(it);
      }
    };
    using lbk_dense::DenseItem;
    using lbk_dense::GemmItem;
    const bool dense_on = (flags & 1) != 0;
    std::vector<std::vector<GemmItem>> gper(nlevels);
    std::vector<std::vector<DenseItem>> dper(nlevels);
    std::vector<int32_t> dsmem(nlevels, 0);
    for (int64_t t = 0; t < ntasks; ++t) {
      const int kind = kinds[t];
      const int64_t i = steps[t], r = trows[t], cc = tcols[t];
      const int32_t lv = tlevels[t];
      Item it{};
      it.kind = kind;
      if (kind == KIND_GETRF) {
        it.a = static_cast<int32_t>(bid[i * p + i]);
        it.b = static_cast<int32_t>(i);
        // row swaps are representable only when every block stores its full
        // rectangle (flags bit 1, the dense-scratch mode): a swapped U panel
        // feeds products that may leave any sparse target's pattern
        it.c = (flags & 2) ? 1 : 0;
        it.begin = 0;
        it.end = 1;
        if (dense_on && hb[it.a].full) {
          DenseItem d{0, it.a, it.b, it.c, 0, static_cast<int32_t>(i)};
          dper[lv].push_back(d);
          dsmem[lv] = std::max(dsmem[lv], (hb[it.a].nrows + 64) * 8);
          continue;
        }
        per[lv].push_back(it);
        lvl_acc[lv] = std::max(lvl_acc[lv], hb[it.a].nrows);
      } else if (kind == KIND_GESSM) {
        it.a = static_cast<int32_t>(bid[i * p + i]);
        it.b = static_cast<int32_t>(bid[i * p + cc]);
        it.c = hb[it.b].full;  // permute on the fly only for full panels
        if (dense_on && hb[it.a].full && hb[it.b].full) {
          for (int32_t s = 0; s < hb[it.b].ncols; s += lbk_dense::STRIP) {
            DenseItem d{1, it.a, it.b, 1, s, static_cast<int32_t>(i)};
            dper[lv].push_back(d);
          }
          dsmem[lv] = std::max(dsmem[lv], (hb[it.a].nrows + 64) * 8);
          continue;
        }
        lvl_acc[lv] = std::max(lvl_acc[lv], hb[it.b].nrows);
        add_range(lv, it, hb[it.b].ncols);
      } else if (kind == KIND_TSTRF) {
        it.a = static_cast<int32_t>(bid[i * p + i]);
        it.b = static_cast<int32_t>(bid[r * p + i]);
        if (dense_on && hb[it.a].full && hb[it.b].full) {
          for (int32_t s = 0; s < hb[it.b].nrows; s += lbk_dense::STRIP) {
            DenseItem d{2, it.a, it.b, 0, s, static_cast<int32_t>(i)};
            dper[lv].push_back(d);
          }
          dsmem[lv] = std::max(dsmem[lv], 64 * 8);
          continue;
        }
        lvl_acc[lv] = std::max(lvl_acc[lv], hb[it.b].ncols);
        add_range(lv, it, hb[it.b].nrows);
      } else {
        const int64_t tgt = bid[r * p + cc];
        if (tgt < 0) {
          if (costs[t] > 0) return fail(st, LBK_ERR_SUPPORT, "update hits an empty block");
          continue;  // zero-work update into an absent block (grid.py:332-362)
        }
        if (costs[t] == 0) continue;  // structurally empty product
        it.a = static_cast<int32_t>(bid[r * p + i]);
        it.b = static_cast<int32_t>(bid[i * p + cc]);
        it.c = static_cast<int32_t>(tgt);
        if (dense_on && hb[it.a].full && hb[it.b].full && hb[tgt].full) {
          for (int32_t n0 = 0; n0 < hb[tgt].ncols; n0 += lbk_dense::GBN)
            for (int32_t m0 = 0; m0 < hb[tgt].nrows; m0 += lbk_dense::GBM)
              gper[lv].push_back(GemmItem{it.a, it.b, it.c, m0, n0, 0});
          continue;
        }
        lvl_acc[lv] = std::max(lvl_acc[lv], hb[tgt].nrows);
        add_range(lv, it, hb[tgt].ncols);
      }
    }
    std::vector<Item> all;
    std::vector<GemmItem> gall;
    std::vector<DenseItem> dall;
    c->levels.clear();
    for (int32_t lv = 0; lv < nlevels; ++lv) {
      if (per[lv].empty() && gper[lv].empty() && dper[lv].empty()) continue;
      if (static_cast<int64_t>(lvl_acc[lv]) * 8 > MAX_SMEM || dsmem[lv] > MAX_SMEM)
        return fail(st, LBK_ERR_BAD_ARG, "block span too large for the shared-memory accumulator");
      Level L{};
      L.item_off = static_cast<int64_t>(all.size());
      L.nitems = static_cast<int32_t>(per[lv].size());
      L.acc_len = lvl_acc[lv];
      L.warps = choose_warps(L.acc_len);
      all.insert(all.end(), per[lv].begin(), per[lv].end());
      L.gemm_off = static_cast<int64_t>(gall.size());
      L.ngemm = static_cast<int32_t>(gper[lv].size());
      gall.insert(gall.end(), gper[lv].begin(), gper[lv].end());
      L.dense_off = static_cast<int64_t>(dall.size());
      L.ndense = static_cast<int32_t>(dper[lv].size());
      L.dense_smem = dsmem[lv];
      L.dense_threads = 256;
      for (const DenseItem& d : dper[lv])
        if (d.kind == 0) L.dense_threads = 512;
      dall.insert(dall.end(), dper[lv].begin(), dper[lv].end());
      c->levels.push_back(L);
    }
    c->total_items = static_cast<int64_t>(all.size());
    c->total_gemm = static_cast<int64_t>(gall.size());
    c->total_dense = static_cast<int64_t>(dall.size());
    c->hblk = hb;
    LBK_CUDA(c->blk.upload(hb), st);
    LBK_CUDA(c->colptr.upload(hcp), st);
    LBK_CUDA(c->rows.upload(hrows), st);
    LBK_CUDA(c->csr_ptr.upload(hrp), st);
    LBK_CUDA(c->csr_col.upload(hcc), st);
    LBK_CUDA(c->csr_pos.upload(hcpos), st);
    LBK_CUDA(c->diag_csc.upload(hdcsc), st);
    LBK_CUDA(c->diag_csr.upload(hdcsr), st);
    LBK_CUDA(c->lv_cols.upload(hlvc), st);
    LBK_CUDA(c->lv_ptr.upload(hlvp), st);
    LBK_CUDA(c->items.upload(all), st);
    LBK_CUDA(c->gitems.upload(gall), st);
    LBK_CUDA(c->ditems.upload(dall), st);
    LBK_CUDA(c->perm.alloc(hdcsc.size()), st);
    LBK_CUDA(c->vals.alloc(nnz), st);
    LBK_CUDA(c->vals0.alloc(nnz), st);
    LBK_CUDA(c->err.alloc(2), st);
  } catch (const std::bad_alloc&) {
    return fail(st, LBK_ERR_OOM, "host allocation in lbk_plan");
  }
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  ok(st);
  return 0;
}

// Pristine A values in pool order (host -> device, kept on device).
int lbk_upload_values(lbk_ctx* c, const double* values, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  LBK_CUDA(cudaMemcpyAsync(c->vals0.p, values, c->nnz * sizeof(double), cudaMemcpyHostToDevice,
                           c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

namespace {

// Capture every level into the current capture of c->stream: the generic
// (sparse) items on the main stream, dense GEMM tiles and dense
// GETRF/GESSM/TSTRF items on two forked branches, joined before the next
// level.  With `evs`, an external (timing-capable) event record node closes
// each level.
void capture_levels(lbk_ctx* c, double pivot_tol, double static_eps, std::vector<cudaEvent_t>* evs) {
  DevPools P = pools(c);
  cudaMemsetAsync(c->err.p, 0xff, 2 * sizeof(unsigned long long), c->stream);
  if (evs) cudaEventRecordWithFlags((*evs)[0], c->stream, cudaEventRecordExternal);
  for (size_t l = 0; l < c->levels.size(); ++l) {
    const Level& L = c->levels[l];
    const bool g = L.ngemm > 0, d = L.ndense > 0;
    if (g || d) cudaEventRecord(c->fork, c->stream);
    if (g) {
      cudaStreamWaitEvent(c->aux[0], c->fork, 0);
      lbk_dense::dgemm_tile_kernel<<<L.ngemm, 256, lbk_dense::GEMM_SMEM, c->aux[0]>>>(
          c->gitems.p + L.gemm_off, P);
      cudaEventRecord(c->join[0], c->aux[0]);
    }
    if (d) {
      cudaStreamWaitEvent(c->aux[1], c->fork, 0);
      lbk_dense::dense_kernel<<<L.ndense, L.dense_threads, L.dense_smem, c->aux[1]>>>(
          c->ditems.p + L.dense_off, P, pivot_tol, static_eps);
      cudaEventRecord(c->join[1], c->aux[1]);
    }
    if (L.nitems) {
      const size_t smem = static_cast<size_t>(L.warps) * L.acc_len * sizeof(double);
      level_kernel<<<L.nitems, L.warps * 32, smem, c->stream>>>(c->items.p + L.item_off, P, L.acc_len,
                                                                pivot_tol, static_eps);
    }
    if (g) cudaStreamWaitEvent(c->stream, c->join[0], 0);
    if (d) cudaStreamWaitEvent(c->stream, c->join[1], 0);
    if (evs) cudaEventRecordWithFlags((*evs)[l + 1], c->stream, cudaEventRecordExternal);
  }
}

int build_graph(lbk_ctx* c, double pivot_tol, double static_eps, lbk_status* st) {
  if (c->graph && ((c->plan_pivot_tol == pivot_tol) ||
                   (std::isnan(c->plan_pivot_tol) && std::isnan(pivot_tol))) &&
      ((c->plan_static_eps == static_eps) || (std::isnan(c->plan_static_eps) && std::isnan(static_eps))))
    return 0;
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t g;
  LBK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), st);
  capture_levels(c, pivot_tol, static_eps, nullptr);
  cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  if (e != cudaSuccess) return cuda_fail(st, e, "graph capture");
  e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(st, e, "graph instantiate");
  c->plan_pivot_tol = pivot_tol;
  c->plan_static_eps = static_eps;
  return 0;
}

int finish(lbk_ctx* c, lbk_status* st) {
  unsigned long long h[2];
  LBK_CUDA(cudaMemcpyAsync(h, c->err.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  const unsigned long long none = ~0ull;
  ok(st);
  if (h[0] != none && (h[1] == none || h[0] < h[1])) {
    st->code = LBK_ERR_ZERO_PIVOT;
    st->block = static_cast<int32_t>(h[0] >> 32);
    st->col = static_cast<int32_t>(h[0] & 0xffffffffu);
    std::snprintf(st->msg, sizeof(st->msg), "zero pivot in diagonal block %d, local column %d",
                  st->block, st->col);
    return st->code;
  }
  if (h[1] != none) {
    st->code = LBK_ERR_PIVOT_SWAP;
    st->block = static_cast<int32_t>(h[1] >> 32);
    st->col = static_cast<int32_t>(h[1] & 0xffffffffu);
    std::snprintf(st->msg, sizeof(st->msg), "row swap needed in sparse diagonal block %d, column %d",
                  st->block, st->col);
    return st->code;
  }
  return 0;
}

}  // namespace

// Device-resident factorization: vals <- vals0, run every level, report
// status.  *ms receives the device time of the level graph (events on the
// launching stream; the D2D reset is outside the timed pair).
int lbk_factorize(lbk_ctx* c, double pivot_tol, double static_eps, float* ms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (build_graph(c, pivot_tol, static_eps, st)) return st->code;
  LBK_CUDA(cudaMemcpyAsync(c->vals.p, c->vals0.p, c->nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->stream), st);
  LBK_CUDA(cudaEventRecord(c->ev0, c->stream), st);
  LBK_CUDA(cudaGraphLaunch(c->graph, c->stream), st);
  LBK_CUDA(cudaEventRecord(c->ev1, c->stream), st);
  int rc = finish(c, st);
  if (rc == LBK_ERR_CUDA || rc == LBK_ERR_OOM) return rc;
  if (ms) {
    float t = 0;
    cudaEventElapsedTime(&t, c->ev0, c->ev1);
    *ms = t;
  }
  return rc;
}

// End-to-end call through host buffers: H2D of A's values, factorization,
// D2H of the factor values (the reference-facing path).
int lbk_factorize_host(lbk_ctx* c, const double* a_values, double* lu_values, int32_t* perms,
                       double pivot_tol, double static_eps, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (build_graph(c, pivot_tol, static_eps, st)) return st->code;
  LBK_CUDA(cudaMemcpyAsync(c->vals.p, a_values, c->nnz * sizeof(double), cudaMemcpyHostToDevice,
                           c->stream), st);
  LBK_CUDA(cudaGraphLaunch(c->graph, c->stream), st);
  LBK_CUDA(cudaMemcpyAsync(lu_values, c->vals.p, c->nnz * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), st);
  if (perms && c->ndiag_rows)
    LBK_CUDA(cudaMemcpyAsync(perms, c->perm.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             c->stream), st);
  return finish(c, st);
}

int lbk_download(lbk_ctx* c, double* lu_values, int32_t* perms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  LBK_CUDA(cudaMemcpyAsync(lu_values, c->vals.p, c->nnz * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), st);
  if (perms && c->ndiag_rows)
    LBK_CUDA(cudaMemcpyAsync(perms, c->perm.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToHost,
                             c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

int lbk_set_perms(lbk_ctx* c, const int32_t* perms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (c->ndiag_rows)
    LBK_CUDA(cudaMemcpy(c->perm.p, perms, c->ndiag_rows * sizeof(int32_t), cudaMemcpyHostToDevice), st);
  ok(st);
  return 0;
}

// Page-locked host buffers for the end-to-end path (H2D/D2H at full PCIe rate).
int lbk_host_alloc(void** ptr, int64_t bytes) {
  return cudaHostAlloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 1)), cudaHostAllocDefault) ==
                 cudaSuccess
             ? 0
             : LBK_ERR_OOM;
}

void lbk_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

// Per-level device times: one instrumented replay (event record nodes between
// the level launches) of the resident values; out_ms[nlevels].
int lbk_level_times(lbk_ctx* c, double pivot_tol, double static_eps, float* out_ms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  const size_t nl = c->levels.size();
  std::vector<cudaEvent_t> ev(nl + 1);
  for (auto& e : ev) LBK_CUDA(cudaEventCreate(&e), st);
  cudaGraph_t g;
  cudaGraphExec_t ge = nullptr;
  LBK_CUDA(cudaMemcpyAsync(c->vals.p, c->vals0.p, c->nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->stream), st);
  LBK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), st);
  capture_levels(c, pivot_tol, static_eps, &ev);
  LBK_CUDA(cudaStreamEndCapture(c->stream, &g), st);
  cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(st, e, "instrumented graph");
  e = cudaGraphLaunch(ge, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess)
    for (size_t l = 0; l < nl; ++l) cudaEventElapsedTime(&out_ms[l], ev[l], ev[l + 1]);
  cudaGraphExecDestroy(ge);
  for (auto& x : ev) cudaEventDestroy(x);
  if (e != cudaSuccess) return cuda_fail(st, e, "instrumented replay");
  return finish(c, st);
}

// Level table for host-side accounting: per launched level its first item,
// item count, warps per CTA and accumulator length; items[6 x total] as
// kind, a, b, c, begin, end.
int lbk_plan_levels(lbk_ctx* c, int64_t* levels /* 4 x nlevels */, int32_t* items /* 6 x total */) {
  const size_t nl = c->levels.size();
  for (size_t l = 0; l < nl; ++l) {
    levels[l] = c->levels[l].item_off;
    levels[nl + l] = c->levels[l].nitems;
    levels[2 * nl + l] = c->levels[l].warps;
    levels[3 * nl + l] = c->levels[l].acc_len;
  }
  if (items) {
    std::vector<Item> h(c->total_items);
    if (c->total_items)
      cudaMemcpy(h.data(), c->items.p, h.size() * sizeof(Item), cudaMemcpyDeviceToHost);
    const size_t T = h.size();
    for (size_t k = 0; k < T; ++k) {
      items[k] = h[k].kind;
      items[T + k] = h[k].a;
      items[2 * T + k] = h[k].b;
      items[3 * T + k] = h[k].c;
      items[4 * T + k] = h[k].begin;
      items[5 * T + k] = h[k].end;
    }
  }
  return 0;
}

// Plan statistics: levels launched, work items, diagonal rows.
int lbk_plan_info(lbk_ctx* c, int64_t* info /* [8] */) {
  info[0] = static_cast<int64_t>(c->levels.size());
  info[1] = c->total_items;
  info[2] = c->ndiag_rows;
  info[3] = c->nnz;
  info[4] = c->total_gemm;
  info[5] = c->total_dense;
  int64_t launches = 0;
  for (const Level& L : c->levels) launches += (L.nitems > 0) + (L.ngemm > 0) + (L.ndense > 0);
  info[6] = launches;
  info[7] = 0;
  return 0;
}

}  // extern "C"
