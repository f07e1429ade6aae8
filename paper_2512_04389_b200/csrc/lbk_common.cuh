// lbk_common.cuh — device data model shared by the sparse and dense kernels.
//
// Every stored block of the grid (grid.py:62-82) lives in one pooled
// "working" array in one of three storage kinds, chosen once at plan time:
//   SPARSE  local CSC on the filled pattern (reference layout);
//   RECT    dense column-major tile over (R x C), R = the block's nonempty
//           local rows, C = its nonempty local columns (supernodal-style
//           compression of a block whose rectangle is >= tau dense);
//   FULL    dense column-major tile over the whole nrows x ncols block
//           (every diagonal block, and everything in dense-scratch mode).
// RECT/FULL blocks are also valid CSC (empty columns outside C, row list R
// repeated), so the sparse kernels read any block through the CSC view while
// the DMMA kernels use the tile view.  Entries of a tile outside the filled
// pattern stay exactly zero (the pattern is elimination-closed, grid.py:3-5)
// and are dropped again on export (factorize.py:179-192).

#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace lbk {

constexpr int KIND_GETRF = 0, KIND_GESSM = 1, KIND_TSTRF = 2, KIND_SSSSM = 3;
constexpr int STORE_SPARSE = 0, STORE_RECT = 1, STORE_FULL = 2;
constexpr int MAX_SMEM = 227 * 1024;

struct BlockDev {
  int32_t nrows, ncols;  // block span
  int32_t store;         // STORE_*
  int32_t nR, nC;        // tile dims (RECT/FULL); nR = ld of the tile
  int32_t nlev;          // sparse diagonal GETRF: intra-block column levels
  int64_t cp;            // colptr pool offset (ncols+1 entries): CSC view of every block
  int64_t ent;           // rows / vals pool offset
  int64_t rp;            // CSR rowptr pool offset (nrows+1), -1 if no CSR index
  int64_t csr;           // CSR entry pool offset (csr_col / csr_pos), -1 if none
  int64_t roff, coff;    // R / C list offsets (RECT), -1 otherwise
  int64_t dg;            // diagonal blocks: offset into the per-diagonal-row pools
  int64_t lvc, lvp;      // sparse diagonal GETRF: level-column / level-pointer offsets
  int64_t xtb1;          // executor-tiled diagonal blocks: 1 + offset of the tile boundaries (0: uniform 64)
};

struct Item {  // generic (sparse) work item: `chunk` columns/rows of one task
  int32_t kind;
  int32_t a, b, c;  // block ids (see lbk_plan)
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
  const int32_t* diag_csc;  // sparse diagonal blocks: local CSC index of (c,c)
  const int32_t* diag_csr;  // sparse diagonal blocks: local CSR index of (r,r)
  const int32_t* lv_cols;
  const int32_t* lv_ptr;
  const int32_t* rlist;     // RECT row lists
  const int32_t* clist;     // RECT column lists
  const int32_t* maps;      // SSSSM gather/scatter maps of the DMMA path
  const int32_t* kchunks;   // SSSSM DMMA tiles: lists of active inner-dimension chunks
  double* gemm_ws;          // split-K partial products of the DMMA SSSSM tiles
  int32_t* perm;            // per diagonal-block row: local permutation
  double* colmax;           // per diagonal-block column: max |entry| at GETRF entry
  unsigned long long* bmax; // per diagonal-block column: max |d_qc| over rows below c (bits)
  unsigned long long* err;  // [0] zero-pivot key, [1] swap key (block<<32 | col), min wins
  const int32_t* xtb;       // tile boundaries of executor-tiled diagonal blocks (subtree-aligned)
};

__device__ __forceinline__ double dsub_mul(double x, double l, double u) {
  // x - (l*u) with both operations separately rounded, like numpy's x -= outer(l, u)
  return __dsub_rn(x, __dmul_rn(l, u));
}

__device__ __forceinline__ void record(unsigned long long* w, int block, int col) {
  unsigned long long key = (static_cast<unsigned long long>(block) << 32) | static_cast<unsigned>(col);
  atomicMin(w, key);
}

// non-negative doubles order like their bit patterns
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* w, double v) {
  atomicMax(w, static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace lbk
