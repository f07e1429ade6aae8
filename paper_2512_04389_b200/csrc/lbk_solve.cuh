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
// Column-oriented: step i solves the diagonal block of block row i, then one
// launch updates every target block row k with the stored blocks of block
// column i: r_k -= B_ki y_i — distinct targets per block, 64-row chunks per
// item, so no atomics and a fixed summation order.  FULL diagonal blocks run
// on a cluster of 8 CTAs (distributed shared memory) with the inverses of
// their 64x64 diagonal tiles (computed at the start of every solve), CSC
// diagonal blocks on one CTA sweeping the columns.  2p + 2p launches per
// solve, captured once into a CUDA graph.  C2: 79 ms (was 536 ms with one
// CTA and triangular tile solves per diagonal block).

#pragma once

#include <cooperative_groups.h>

#include "lbk_common.cuh"
#include "lbk_exec.cuh"

namespace lbk {

constexpr int SOLVE_CHUNK = 64;     // rows per diagonal-solve chunk
constexpr int UPD_ROWS = 64;        // block rows per update item

struct SolveStep {
  int32_t diag;   // diagonal block id
  int32_t off;    // global offset of the block row
  int32_t span;
  int32_t nupd;   // update items of this step
  int64_t upd_off;
  int64_t tinv;   // FULL diagonal blocks: offset of its inverse 64x64 diagonal tiles (-1: none)
  int64_t ext;    // offset of the per-chunk (row hi, row lo) pattern extents
  int32_t bl, bu; // banded FULL diagonal block: bandwidths (-1: not banded)
  int32_t nseg;   // its independent segments
  int64_t seg_off;  // offset of their (s0, s1) pairs
};

constexpr int BAND_SOLVE_ROWS = 1024;  // rows of a segment staged per chunk

// One thread's sweep over a staged chunk of a band segment (solve_band_kernel).  The last
// B solution values live in registers (win[k-1] = x at distance k), so each row costs one
// FMA on the dependency chain: the terms of the older values are summed first.  The
// backward sweep multiplies by the reciprocal of U(r, r) (formed off the chain).
// nb = the band width when it is below the template bound (B = 8 / 15 buckets).
template <int B>
__device__ __forceinline__ void band_sweep(double* ys, const double* band, int W, int rn, int upper,
                                           const double* carry, int before, int after, int nb = B) {
  double win[B > 0 ? B : 1];
#pragma unroll
  for (int k = 0; k < B; ++k) {  // values of the previous chunk (0 outside the segment)
    if (!upper) win[k] = (k < nb && k < before) ? carry[nb - 1 - k] : 0.0;
    else win[k] = (k < nb && k < after) ? carry[k] : 0.0;
  }
#pragma unroll 4
  for (int q = 0; q < rn; ++q) {
    const int r = upper ? rn - 1 - q : q;
    const double* br = band + r * W;
    double acc = ys[r];
#pragma unroll
    for (int k = B; k >= 2; --k)
      if (k <= nb) acc = fma(-br[k], win[k - 1], acc);
    double x = B >= 1 && nb >= 1 ? fma(-br[1], win[0], acc) : acc;
    if (upper) x *= br[0];  // staged as 1 / U(r, r)
#pragma unroll
    for (int k = B - 1; k >= 1; --k) win[k] = win[k - 1];
    if (B > 0) win[0] = x;
    ys[r] = x;
  }
}

// Banded FULL diagonal block (the filled pattern within |r - c| <= bl / bu, e.g. the
// bodies of a bordered-block-diagonal matrix): one CTA per independent segment stages
// the band of up to 1,024 rows into shared memory (row-oriented: the sweep reads
// contiguous entries) and one thread sweeps it, carrying the last bw solution values
// across chunks.  Forward: x_r = y_r - sum_q L(r, r-q) x_{r-q} (unit lower);
// backward: x_r = (y_r - sum_q U(r, r+q) x_{r+q}) / U(r, r).  Same row operations as the
// dense chunked solve restricted to the band (entries outside it are exact zeros).
__global__ void __launch_bounds__(256) solve_band_kernel(DevPools P, const SolveStep* __restrict__ steps, int s,
                                                        double* __restrict__ v, int upper,
                                                        const int32_t* __restrict__ segs) {
  extern __shared__ double sm[];
  const SolveStep S = steps[s];
  const BlockDev D = P.blk[S.diag];
  const int s0 = segs[S.seg_off + 2 * blockIdx.x], s1 = segs[S.seg_off + 2 * blockIdx.x + 1];
  const int bw = upper ? S.bu : S.bl, W = bw + 1, ld = D.nR;
  const double* G = P.vals + D.ent;
  double* band = sm;                              // [BAND_SOLVE_ROWS][W]
  double* ys = sm + BAND_SOLVE_ROWS * W;          // [BAND_SOLVE_ROWS]
  double* carry = ys + BAND_SOLVE_ROWS;           // last bw solved values of the previous chunk
  const int m = s1 - s0, nch = (m + BAND_SOLVE_ROWS - 1) / BAND_SOLVE_ROWS;
  for (int q = 0; q < nch; ++q) {
    const int cq = upper ? nch - 1 - q : q;
    const int r0 = s0 + cq * BAND_SOLVE_ROWS, rn = min(BAND_SOLVE_ROWS, s1 - r0);
    // staged column by column: column c holds L(c + q, c) (forward) / U(c - q, c) (backward),
    // q = 0..bw, contiguous in the column-major tile -> one thread, up to 16 loads in flight
    {
      const int cb = upper ? r0 : r0 - bw, ce = upper ? r0 + rn + bw : r0 + rn;
      for (int c = cb + static_cast<int>(threadIdx.x); c < ce; c += blockDim.x) {
        double vq[BAND_MAX + 1];
#pragma unroll
        for (int q = 0; q <= BAND_MAX; ++q) {
          const int r = upper ? c - q : c + q;
          vq[q] = (q < W && c >= s0 && c < s1 && r >= s0 && r < s1) ? G[static_cast<size_t>(c) * ld + r] : 0.0;
        }
        if (upper) vq[0] = 1.0 / vq[0];  // the backward sweep multiplies by 1 / U(c, c)
#pragma unroll
        for (int q = 0; q <= BAND_MAX; ++q) {
          const int r = upper ? c - q : c + q;
          if (q < W && r >= r0 && r < r0 + rn) band[(r - r0) * W + q] = vq[q];
        }
      }
      // (every slot (r, k) of the chunk has its column in [cb, ce): columns outside the
      // segment write their zeros there too)
    }
    for (int r = threadIdx.x; r < rn; r += blockDim.x) ys[r] = v[S.off + r0 + r];
    __syncthreads();
    if (threadIdx.x == 0) {
      switch (bw) {
        case 0: band_sweep<0>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn); break;
        case 1: band_sweep<1>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn); break;
        case 2: band_sweep<2>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn); break;
        case 3: band_sweep<3>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn); break;
        case 4: band_sweep<4>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn); break;
        case 5: case 6: case 7: case 8: band_sweep<8>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn, bw); break;
        default: band_sweep<15>(ys, band, W, rn, upper, carry, r0 - s0, s1 - r0 - rn, bw); break;
      }
      // the values the next chunk reaches back to (forward: the last bw rows, backward: the first)
      for (int k = 0; k < bw; ++k) {
        if (!upper) carry[k] = rn - bw + k >= 0 ? ys[rn - bw + k] : 0.0;
        else carry[k] = k < rn ? ys[k] : 0.0;
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rn; r += blockDim.x) v[S.off + r0 + r] = ys[r];
    __syncthreads();
  }
}

constexpr int SOLVE_CL = 8;  // CTAs per cluster of the diagonal solve

// Inverses of the 64x64 diagonal tiles of a factored FULL diagonal block:
// Linv = (unit lower of tile)^-1, Uinv = (upper of tile)^-1, column-major 64x64
// each, at inv[2 * 4096 * tile + {0, 4096}].  Edge tiles are padded with the
// identity.  One CTA per tile (the compact blocked tile solves of the executor
// applied to an identity right-hand side).
__global__ void __launch_bounds__(256) tile_inverse_kernel(DevPools P, const SolveStep* __restrict__ steps,
                                                          const int32_t* __restrict__ tstep,
                                                          const int32_t* __restrict__ ttile, double* inv) {
  extern __shared__ double sm[];
  const SolveStep S = steps[tstep[blockIdx.x]];
  const int t = ttile[blockIdx.x];
  const BlockDev D = P.blk[S.diag];
  const int m = S.span, c0 = t * XT, cn = min(XT, m - c0), ld = D.nR;
  double* X = sm;             // XTP stride
  double* T = sm + XREG;      // the factored tile
  double* rinv = sm + 2 * XREG;
  const double* G = P.vals + D.ent + static_cast<size_t>(c0) * ld + c0;
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) {
    const int r = e & (XT - 1), c = e >> 6;
    T[c * XTP + r] = (r < cn && c < cn) ? G[static_cast<size_t>(c) * ld + r] : (r == c ? 1.0 : 0.0);
    X[c * XTP + r] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  double* out = inv + S.tinv + static_cast<int64_t>(t) * 2 * XT * XT;
  tile_left_solve_blk(X, T, XT);  // X = L^-1
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) out[e] = X[(e >> 6) * XTP + (e & (XT - 1))];
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) X[(e >> 6) * XTP + (e & (XT - 1))] = (e >> 6) == (e & 63) ? 1.0 : 0.0;
  if (threadIdx.x < XT) rinv[threadIdx.x] = 1.0 / T[threadIdx.x * XTP + threadIdx.x];
  __syncthreads();
  tile_right_solve_blk<false>(X, T, rinv, nullptr, XT);  // X = U^-1
  for (int e = threadIdx.x; e < XT * XT; e += blockDim.x) out[XT * XT + e] = X[(e >> 6) * XTP + (e & (XT - 1))];
}

// Diagonal block of one step on a cluster of SOLVE_CL CTAs (FULL storage).
// CTA q owns rows [q*rpc, (q+1)*rpc) of the segment (rpc a multiple of 64, so
// every 64-row chunk has one owner).  Per chunk: the owner forms x_c = Tinv_c
// r_c from its shared memory and publishes it; one cluster barrier; every CTA
// reads x_c through distributed shared memory and updates its own rows below
// (forward) / above (backward) the chunk.  x buffers alternate by chunk
// parity, so one barrier per chunk suffices.
__global__ void __cluster_dims__(SOLVE_CL, 1, 1) __launch_bounds__(256)
    solve_diag_cluster_kernel(DevPools P, const SolveStep* __restrict__ steps, int s, double* __restrict__ v,
                              int upper, const double* __restrict__ inv, const int32_t* __restrict__ ext) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  const SolveStep S = steps[s];
  const BlockDev D = P.blk[S.diag];
  const int m = S.span, tid = threadIdx.x, q = static_cast<int>(cl.block_rank());
  const int nch = (m + XT - 1) / XT, rpc = ((nch + SOLVE_CL - 1) / SOLVE_CL) * XT;
  const int r0 = q * rpc, r1 = min(m, r0 + rpc);
  double* y = sm;                 // my rows
  double* xb = sm + rpc;          // [2][64] published chunk solution
  double* xs = xb + 2 * XT;       // chunk solution read from the owner
  double* part = xs + XT;         // 256 matvec partial sums
  for (int r = r0 + tid; r < r1; r += blockDim.x) y[r - r0] = v[S.off + r];
  const double* G = P.vals + D.ent;
  const int ld = D.nR;
  cl.sync();
  for (int qq = 0; qq < nch; ++qq) {
    const int c = upper ? nch - 1 - qq : qq;
    const int c0 = c * XT, cn = min(XT, m - c0), owner = c0 / rpc;
    double* xbuf = xb + (qq & 1) * XT;
    if (q == owner) {
      // x_c = Tinv_c r_c: thread (row, k-quarter) -> 16 independent loads
      const double* Ti = inv + S.tinv + static_cast<int64_t>(c) * 2 * XT * XT + (upper ? XT * XT : 0);
      const int row = tid & (XT - 1), kq = (tid >> 6) * 16;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (kq + k < cn) acc = fma(Ti[(kq + k) * XT + row], y[c0 - r0 + kq + k], acc);
      part[tid] = acc;
      __syncthreads();
      if (tid < XT) xbuf[tid] = tid < cn ? (part[tid] + part[XT + tid]) + (part[2 * XT + tid] + part[3 * XT + tid]) : 0.0;
      __syncthreads();
      if (tid < cn) y[c0 - r0 + tid] = xbuf[tid];
    }
    cl.sync();
    const double* src = cl.map_shared_rank(xbuf, owner);
    if (tid < XT) xs[tid] = tid < cn ? src[tid] : 0.0;
    __syncthreads();
    // my rows strictly below (forward) / above (backward) the chunk
    // ... limited to the rows the chunk's pattern reaches (banded blocks: a few)
    const int lo = upper ? max(r0, ext[S.ext + 2 * c + 1]) : max(r0, c0 + cn);
    const int hi = upper ? min(r1, c0) : min(r1, ext[S.ext + 2 * c]);
    for (int r = lo + tid; r < hi; r += blockDim.x) {
      const double* col = G + static_cast<size_t>(c0) * ld + r;
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      if (cn == XT) {
#pragma unroll
        for (int k = 0; k < XT; ++k) a4[k & 3] = fma(col[static_cast<size_t>(k) * ld], xs[k], a4[k & 3]);
      } else {
        for (int k = 0; k < cn; ++k) a4[k & 3] = fma(col[static_cast<size_t>(k) * ld], xs[k], a4[k & 3]);
      }
      y[r - r0] -= (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while another may still read its x buffer
  for (int r = r0 + tid; r < r1; r += blockDim.x) v[S.off + r] = y[r - r0];
}

#ifndef LBK_SOLVE_FLAGS
#define LBK_SOLVE_FLAGS 0  // 1: dense diagonal solve with per-chunk flags in distributed shared memory + lookahead (measured slower: C2 solve 68 -> 85 ms)
#endif

__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_cluster(int* p, int v) {
  asm volatile("st.release.cluster.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Same solve as solve_diag_cluster_kernel, without a cluster barrier per chunk: the
// owner of chunk c publishes x_c in its own row segment (y) and raises done[c]
// (st.release.cluster); a consumer waits on that flag through distributed shared
// memory (ld.acquire.cluster) and reads x_c from the owner's y.  Lookahead: a CTA that
// owns the next chunk applies x_c to that chunk's rows first, forms and publishes x_next,
// and only then applies x_c to the rest of its rows - the critical path per chunk is one
// 64x64 update, one 64x64 matvec and one flag hop.  Every row still receives its updates
// in chunk order, each the same 4-way partial-sum matvec as before.
__global__ void __cluster_dims__(SOLVE_CL, 1, 1) __launch_bounds__(256)
    solve_diag_flag_kernel(DevPools P, const SolveStep* __restrict__ steps, int s, double* __restrict__ v,
                           int upper, const double* __restrict__ inv, const int32_t* __restrict__ ext) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double sm[];
  const SolveStep S = steps[s];
  const BlockDev D = P.blk[S.diag];
  const int m = S.span, tid = threadIdx.x, q = static_cast<int>(cl.block_rank());
  const int nch = (m + XT - 1) / XT, rpc = ((nch + SOLVE_CL - 1) / SOLVE_CL) * XT;
  const int r0 = q * rpc, r1 = min(m, r0 + rpc);
  double* y = sm;                 // my rows (x once solved)
  double* xs = sm + rpc;          // the current chunk's solution
  double* part = xs + XT;         // 256 matvec partial sums
  int* done = reinterpret_cast<int*>(part + 4 * XT);  // per chunk: x published (own chunks)
  for (int r = r0 + tid; r < r1; r += blockDim.x) y[r - r0] = v[S.off + r];
  for (int c = tid; c < nch; c += blockDim.x) done[c] = 0;
  const double* G = P.vals + D.ent;
  const int ld = D.nR;
  cl.sync();  // every CTA's flags are zero before anyone polls them
  auto chunk = [&](int qq) { return upper ? nch - 1 - qq : qq; };
  auto owner_of = [&](int c) { return (c * XT) / rpc; };
  // x_c = Tinv_c r_c on the owner (its rows of chunk c are fully updated), then publish
  auto solve_chunk = [&](int c) {
    const int c0 = c * XT, cn = min(XT, m - c0);
    const double* Ti = inv + S.tinv + static_cast<int64_t>(c) * 2 * XT * XT + (upper ? XT * XT : 0);
    const int row = tid & (XT - 1), kq = (tid >> 6) * 16;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (kq + k < cn) acc = fma(Ti[(kq + k) * XT + row], y[c0 - r0 + kq + k], acc);
    part[tid] = acc;
    __syncthreads();
    double xv = 0.0;
    if (tid < cn) xv = (part[tid] + part[XT + tid]) + (part[2 * XT + tid] + part[3 * XT + tid]);
    __syncthreads();
    if (tid < cn) y[c0 - r0 + tid] = xv;
    __syncthreads();
    if (tid == 0) st_release_cluster(done + c, 1);
  };
  // y[r - r0] -= L[r, c0:c0+cn] xs for r in [lo, hi) (rows of this CTA)
  auto apply = [&](int c, int lo, int hi) {
    const int c0 = c * XT, cn = min(XT, m - c0);
    for (int r = lo + tid; r < hi; r += blockDim.x) {
      const double* col = G + static_cast<size_t>(c0) * ld + r;
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      if (cn == XT) {
#pragma unroll
        for (int k = 0; k < XT; ++k) a4[k & 3] = fma(col[static_cast<size_t>(k) * ld], xs[k], a4[k & 3]);
      } else {
        for (int k = 0; k < cn; ++k) a4[k & 3] = fma(col[static_cast<size_t>(k) * ld], xs[k], a4[k & 3]);
      }
      y[r - r0] -= (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
  };
  if (owner_of(chunk(0)) == q) solve_chunk(chunk(0));
  for (int qq = 0; qq < nch; ++qq) {
    const int c = chunk(qq), c0 = c * XT, cn = min(XT, m - c0), own = owner_of(c);
    // rows this chunk reaches inside my range (banded patterns: a few)
    const int lo = upper ? max(r0, ext[S.ext + 2 * c + 1]) : max(r0, c0 + cn);
    const int hi = upper ? min(r1, c0) : min(r1, ext[S.ext + 2 * c]);
    const bool need = lo < hi;
    if (need) {
      if (own == q) {
        if (tid < XT) xs[tid] = tid < cn ? y[c0 - r0 + tid] : 0.0;
      } else {
        if (tid == 0) {
          const int* f = cl.map_shared_rank(done, own) + c;
          while (ld_acquire_cluster(f) == 0) {
          }
        }
        __syncthreads();
        const double* src = cl.map_shared_rank(y, own) + (c0 - own * rpc);
        if (tid < XT) xs[tid] = tid < cn ? src[tid] : 0.0;
      }
      __syncthreads();
    }
    // lookahead: when the next chunk is mine, its rows get x_c first and it is solved and
    // published before x_c reaches the rest of my rows
    int n0 = m, n1 = m;
    if (qq + 1 < nch && owner_of(chunk(qq + 1)) == q) {
      n0 = chunk(qq + 1) * XT;
      n1 = min(m, n0 + XT);
      if (need) apply(c, max(lo, n0), min(hi, n1));
      __syncthreads();
      solve_chunk(chunk(qq + 1));
    }
    if (need) {
      apply(c, lo, min(hi, n0));
      apply(c, max(lo, n1), hi);
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while another may still read its rows
  for (int r = r0 + tid; r < r1; r += blockDim.x) v[S.off + r] = y[r - r0];
}

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
      // four independent partial sums and a fully unrolled k loop: the 64
      // column loads of a row are all in flight at once (HBM latency bound)
      for (int r = rb0 + tid; r < rb1; r += blockDim.x) {
        const double* col = G + static_cast<size_t>(c0) * ld + r;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (cn == SOLVE_CHUNK) {
#pragma unroll
          for (int k = 0; k < SOLVE_CHUNK; ++k) acc[k & 3] = fma(col[static_cast<size_t>(k) * ld], y[c0 + k], acc[k & 3]);
        } else {
          for (int k = 0; k < cn; ++k) acc[k & 3] = fma(col[static_cast<size_t>(k) * ld], y[c0 + k], acc[k & 3]);
        }
        y[r] -= (acc[0] + acc[1]) + (acc[2] + acc[3]);
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < m; r += blockDim.x) v[S.off + r] = y[r];
}

// r_k -= B_ki y_i for one 64-row chunk of one stored block (dense tiles: 64 rows
// x 4 column quarters, partial sums reduced in smem; CSC: one row per thread).
// Dynamic smem: the source segment (block column span) + 256 partial sums.
__global__ void __launch_bounds__(256) solve_upd_kernel(DevPools P, const SolveUpd* __restrict__ items,
                                                       double* __restrict__ v) {
  extern __shared__ double ys[];
  const SolveUpd it = items[blockIdx.x];
  const BlockDev B = P.blk[it.blk];
  const int tid = threadIdx.x;
  const int32_t* cl = B.store == STORE_RECT ? P.clist + B.coff : nullptr;
  // the source values this block reads: a RECT block only its stored columns (compressed)
  if (cl) {
    for (int a = tid; a < B.nC; a += blockDim.x) ys[a] = v[it.src_off + cl[a]];
  } else {
    for (int c = tid; c < B.ncols; c += blockDim.x) ys[c] = v[it.src_off + c];
  }
  __syncthreads();
  const double* G = P.vals + B.ent;
  const int a = it.r0 + tid;
  if (B.store == STORE_SPARSE) {
    if (tid >= UPD_ROWS || a >= B.nrows) return;
    const int32_t* rp = P.csr_ptr + B.rp;
    const int32_t* cc = P.csr_col + B.csr;
    const int32_t* ps = P.csr_pos + B.csr;
    double acc = 0.0;
    for (int g = rp[a]; g < rp[a + 1]; ++g) acc = fma(G[ps[g]], ys[cc[g]], acc);
    v[it.tgt_off + a] -= acc;
  } else {
    // 64 rows x 4 column quarters per CTA: 4x shorter dependent load chains
    const int ar = it.r0 + (tid & 63), quarter = tid >> 6;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (ar < B.nR) {
      const int cq = (B.nC + 3) / 4, cb = quarter * cq, ce = min(B.nC, cb + cq);
      const double* col = G + ar;
      int c = cb;
      for (; c + 8 <= ce; c += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q & 3] = fma(col[static_cast<size_t>(c + q) * B.nR], ys[c + q], acc[q & 3]);
      }
      for (; c < ce; ++c) acc[0] = fma(col[static_cast<size_t>(c) * B.nR], ys[c], acc[0]);
    }
    double* part = ys + ((B.ncols + 1) & ~1);  // 4 x 64 partial sums after the source segment
    part[quarter * 64 + (tid & 63)] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    __syncthreads();
    if (tid < 64 && ar < B.nR) {
      const int row = B.store == STORE_RECT ? P.rlist[B.roff + ar] : ar;
      v[it.tgt_off + row] -= (part[tid] + part[64 + tid]) + (part[128 + tid] + part[192 + tid]);
    }
  }
}

}  // namespace lbk
