// Host-side structure path of the block LU engine (native, bit-exact with the
// reference's Python structure path).
//
//   lbk_symbolic_*      ~ lublock.symbolic.symbolic_factorize   pkg/src/lublock/symbolic.py:57-108
//   lbk_partition_*     ~ lublock.grid.partition                pkg/src/lublock/grid.py:85-148
//   lbk_levels_*        ~ lublock.grid.dependency_levels        pkg/src/lublock/grid.py:223-378
//
// All integer outputs must equal the reference arrays element for element;
// the Python wrappers in paper_2512_04389_b200/{symbolic,grid}.py check that
// against committed golden fixtures.  No floating point is produced here
// except the value scatter in partition (pure copies).
//
// Memory model: each "run" call allocates a result object owned by C++ and
// returns an opaque handle plus the sizes; the caller allocates numpy arrays
// of those sizes and calls the matching "fetch", then "free".

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/lbk.h"

namespace {

// --------------------------------------------------------------------------
// symbolic factorization: elimination-tree row-subtree walk in natural order
// --------------------------------------------------------------------------
struct SymbolicResult {
  int64_t n = 0;
  std::vector<int64_t> col_ptr;  // n+1
  std::vector<int64_t> row_idx;  // nnz(L+U)
  std::vector<int64_t> parent;   // elimination tree
};

// Row pattern of L for row i = the set of etree nodes reached by walking up
// from every j<i with A(i,j) != 0 until a node already marked for row i.
// The union pattern of column c is [sorted row-pattern(c)] ++ [c] ++
// [rows i>c whose pattern contains c, ascending] which is exactly the (col,
// row)-sorted order the reference builds with a stable argsort.
int symbolic_run(int64_t n, const int64_t* cp, const int64_t* ri, SymbolicResult* out) {
  std::vector<int64_t> parent(n, -1), mark(n, -1);
  std::vector<int64_t> rp_ptr(n + 1, 0);
  std::vector<int32_t> rp;  // row patterns (strict lower), concatenated
  rp.reserve(static_cast<size_t>(cp[n]) * 2 + 16);
  std::vector<int64_t> lcount(n, 0);  // column counts of strict L
  for (int64_t i = 0; i < n; ++i) {
    mark[i] = i;
    size_t start = rp.size();
    for (int64_t e = cp[i]; e < cp[i + 1]; ++e) {
      int64_t j = ri[e];
      if (j >= i) break;  // rows sorted: remaining entries are >= i
      while (mark[j] != i) {
        rp.push_back(static_cast<int32_t>(j));
        mark[j] = i;
        if (parent[j] == -1) parent[j] = i;
        j = parent[j];
      }
    }
    std::sort(rp.begin() + start, rp.end());
    for (size_t k = start; k < rp.size(); ++k) lcount[rp[k]]++;
    rp_ptr[i + 1] = static_cast<int64_t>(rp.size());
  }
  out->n = n;
  out->col_ptr.assign(n + 1, 0);
  for (int64_t c = 0; c < n; ++c)
    out->col_ptr[c + 1] = out->col_ptr[c] + (rp_ptr[c + 1] - rp_ptr[c]) + 1 + lcount[c];
  out->row_idx.resize(static_cast<size_t>(out->col_ptr[n]));
  // fill: upper part + diagonal first, remember the write cursor for the lower part
  std::vector<int64_t> cur(n);
  for (int64_t c = 0; c < n; ++c) {
    int64_t w = out->col_ptr[c];
    for (int64_t k = rp_ptr[c]; k < rp_ptr[c + 1]; ++k) out->row_idx[w++] = rp[k];
    out->row_idx[w++] = c;
    cur[c] = w;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp_ptr[i]; k < rp_ptr[i + 1]; ++k) out->row_idx[cur[rp[k]]++] = i;
  out->parent = std::move(parent);
  return 0;
}

// --------------------------------------------------------------------------
// partition: cut the filled pattern into local-index CSC blocks
// --------------------------------------------------------------------------
struct PartitionResult {
  int64_t p = 0;
  int64_t nblocks = 0;
  // block table, column-major block order (key = bj*p + bi ascending)
  std::vector<int64_t> bi, bj, nrows, ncols, nnz, cp_off, ent_off;
  std::vector<int64_t> col_ptr;  // sum over blocks of (ncols+1)
  std::vector<int64_t> row_idx;  // local rows, nnz_filled
  std::vector<double> values;    // nnz_filled
  std::vector<int64_t> block_nnz;  // p*p row-major
};

int partition_run(int64_t n, const int64_t* fcp, const int64_t* fri, const int64_t* acp,
                  const int64_t* ari, const double* aval, int64_t p, const int64_t* pos,
                  PartitionResult* out) {
  std::vector<int32_t> rowblk(n);
  for (int64_t b = 0; b < p; ++b)
    for (int64_t r = pos[b]; r < pos[b + 1]; ++r) rowblk[r] = static_cast<int32_t>(b);
  const int64_t nnzf = fcp[n];
  // scatter A values into the filled pattern (0.0 at fill); A must be covered
  std::vector<double> fval(static_cast<size_t>(nnzf), 0.0);
  for (int64_t c = 0; c < n; ++c) {
    int64_t f = fcp[c], fe = fcp[c + 1];
    for (int64_t e = acp[c]; e < acp[c + 1]; ++e) {
      int64_t r = ari[e];
      while (f < fe && fri[f] < r) ++f;
      if (f == fe || fri[f] != r) return LBK_ERR_DIM_MISMATCH;
      fval[f] = aval[e];
    }
  }
  out->p = p;
  out->block_nnz.assign(static_cast<size_t>(p * p), 0);
  out->row_idx.resize(nnzf);
  out->values.resize(nnzf);
  std::vector<int64_t> cnt(p), colcnt;  // per block-row counts in this block column
  int64_t ent = 0;
  for (int64_t bj = 0; bj < p; ++bj) {
    const int64_t c0 = pos[bj], c1 = pos[bj + 1], nc = c1 - c0;
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int64_t e = fcp[c0]; e < fcp[c1]; ++e) cnt[rowblk[fri[e]]]++;
    // block start offsets within this block column (blocks ordered by bi)
    std::vector<int64_t> start(p), blk_id(p, -1);
    int64_t acc = ent;
    for (int64_t b = 0; b < p; ++b) {
      if (cnt[b] == 0) continue;
      start[b] = acc;
      acc += cnt[b];
      blk_id[b] = out->nblocks++;
      out->bi.push_back(b);
      out->bj.push_back(bj);
      out->nrows.push_back(pos[b + 1] - pos[b]);
      out->ncols.push_back(nc);
      out->nnz.push_back(cnt[b]);
      out->ent_off.push_back(start[b]);
      out->cp_off.push_back(static_cast<int64_t>(out->col_ptr.size()));
      out->col_ptr.resize(out->col_ptr.size() + nc + 1, 0);
      out->block_nnz[b * p + bj] = cnt[b];
    }
    // write entries, in (col,row) order within each block; build local col_ptr
    std::vector<int64_t> w(start);
    for (int64_t c = c0; c < c1; ++c) {
      for (int64_t e = fcp[c]; e < fcp[c + 1]; ++e) {
        int64_t r = fri[e];
        int32_t b = rowblk[r];
        int64_t k = w[b]++;
        out->row_idx[k] = r - pos[b];
        out->values[k] = fval[e];
        out->col_ptr[out->cp_off[blk_id[b]] + (c - c0) + 1]++;
      }
    }
    for (int64_t b = 0; b < p; ++b) {
      if (blk_id[b] < 0) continue;
      int64_t* cpb = &out->col_ptr[out->cp_off[blk_id[b]]];
      for (int64_t c = 0; c < nc; ++c) cpb[c + 1] += cpb[c];
    }
    ent = acc;
  }
  return 0;
}

// --------------------------------------------------------------------------
// dependency levels: static task DAG in construction order with ASAP levels
// --------------------------------------------------------------------------
struct LevelsResult {
  std::vector<int8_t> kinds;
  std::vector<int32_t> steps, rows, cols, levels;
  std::vector<int64_t> weights, costs, pred_ptr;
  std::vector<int32_t> pred_idx;
};

// Inputs: the block table of a partition (any order) with per-block col
// counts (from col_ptr) and row counts (bincount of local rows).
int levels_run(int64_t p, int64_t nblocks, const int64_t* bi, const int64_t* bj,
               const int64_t* nrows, const int64_t* ncols, const int64_t* cp_off,
               const int64_t* ent_off, const int64_t* col_ptr, const int64_t* row_idx,
               LevelsResult* out) {
  std::vector<int64_t> bid(static_cast<size_t>(p * p), -1);
  for (int64_t b = 0; b < nblocks; ++b) bid[bi[b] * p + bj[b]] = b;
  auto bnnz = [&](int64_t r, int64_t c) -> int64_t {
    int64_t b = bid[r * p + c];
    if (b < 0) return 0;
    return col_ptr[cp_off[b] + ncols[b]];
  };
  // per-block column counts and row counts (int64)
  std::vector<int64_t> ccoff(nblocks + 1, 0), rcoff(nblocks + 1, 0);
  for (int64_t b = 0; b < nblocks; ++b) {
    ccoff[b + 1] = ccoff[b] + ncols[b];
    rcoff[b + 1] = rcoff[b] + nrows[b];
  }
  std::vector<int64_t> ccnt(ccoff[nblocks]), rcnt(rcoff[nblocks], 0);
  for (int64_t b = 0; b < nblocks; ++b) {
    const int64_t* cpb = col_ptr + cp_off[b];
    for (int64_t c = 0; c < ncols[b]; ++c) ccnt[ccoff[b] + c] = cpb[c + 1] - cpb[c];
    const int64_t base = ent_off[b];
    for (int64_t e = 0; e < cpb[ncols[b]]; ++e) rcnt[rcoff[b] + row_idx[base + e]]++;
  }
  std::vector<int32_t> last_id(static_cast<size_t>(p * p), -1), last_lv(static_cast<size_t>(p * p), -1);
  std::vector<int64_t> pred_cnt;
  int32_t tid = 0;
  std::vector<int64_t> lows, ups;
  std::vector<int32_t> u_id(p), u_lv(p), l_id(p), l_lv(p);
  auto push = [&](int8_t k, int64_t s, int64_t r, int64_t c, int64_t w, int64_t cost, int32_t lv) {
    out->kinds.push_back(k);
    out->steps.push_back(static_cast<int32_t>(s));
    out->rows.push_back(static_cast<int32_t>(r));
    out->cols.push_back(static_cast<int32_t>(c));
    out->weights.push_back(w);
    out->costs.push_back(cost);
    out->levels.push_back(lv);
  };
  for (int64_t i = 0; i < p; ++i) {
    lows.clear();
    ups.clear();
    for (int64_t k = i + 1; k < p; ++k)
      if (bnnz(k, i)) lows.push_back(k);
    for (int64_t j = i + 1; j < p; ++j)
      if (bnnz(i, j)) ups.push_back(j);
    const int64_t dnnz = bnnz(i, i);
    int32_t prev = last_id[i * p + i];
    int32_t glv = last_lv[i * p + i] + 1;
    push(0, i, i, i, dnnz, dnnz, glv);
    if (prev >= 0) { out->pred_idx.push_back(prev); pred_cnt.push_back(1); }
    else pred_cnt.push_back(0);
    const int32_t gid = tid++;
    for (int64_t j : ups) {
      prev = last_id[i * p + j];
      int32_t lv = std::max(glv, last_lv[i * p + j]) + 1;
      const int64_t w = bnnz(i, j);
      push(1, i, i, j, w, w, lv);
      out->pred_idx.push_back(gid);
      if (prev >= 0) { out->pred_idx.push_back(prev); pred_cnt.push_back(2); }
      else pred_cnt.push_back(1);
      u_id[j] = tid++;
      u_lv[j] = lv;
    }
    for (int64_t k : lows) {
      prev = last_id[k * p + i];
      int32_t lv = std::max(glv, last_lv[k * p + i]) + 1;
      const int64_t w = bnnz(k, i);
      push(2, i, k, i, w, w, lv);
      out->pred_idx.push_back(gid);
      if (prev >= 0) { out->pred_idx.push_back(prev); pred_cnt.push_back(2); }
      else pred_cnt.push_back(1);
      l_id[k] = tid++;
      l_lv[k] = lv;
    }
    for (int64_t k : lows) {
      const int64_t bl = bid[k * p + i];
      const int64_t nnz_l = bnnz(k, i);
      const int64_t* cl = &ccnt[ccoff[bl]];
      for (int64_t j : ups) {
        const int64_t bu = bid[i * p + j];
        const int64_t* ru = &rcnt[rcoff[bu]];
        int64_t madds = 0;
        for (int64_t r = 0; r < ncols[bl]; ++r) madds += cl[r] * ru[r];
        prev = last_id[k * p + j];
        int32_t plv = last_lv[k * p + j];
        int32_t lv = std::max(l_lv[k], u_lv[j]);
        if (plv > lv) lv = plv;
        lv += 1;
        const int64_t nnz_u = bnnz(i, j);
        const int64_t tgt = bnnz(k, j);
        int64_t w = nnz_l < nnz_u ? nnz_l : nnz_u;
        if (tgt > 0 && tgt < w) w = tgt;
        push(3, i, k, j, w, madds, lv);
        out->pred_idx.push_back(l_id[k]);
        out->pred_idx.push_back(u_id[j]);
        if (prev >= 0) { out->pred_idx.push_back(prev); pred_cnt.push_back(3); }
        else pred_cnt.push_back(2);
        last_id[k * p + j] = tid;
        last_lv[k * p + j] = lv;
        ++tid;
      }
    }
  }
  out->pred_ptr.assign(static_cast<size_t>(tid) + 1, 0);
  for (int32_t t = 0; t < tid; ++t) out->pred_ptr[t + 1] = out->pred_ptr[t] + pred_cnt[t];
  return 0;
}

template <class T>
void copy_out(const std::vector<T>& v, T* dst) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
}

}  // namespace

extern "C" {

int lbk_symbolic_run(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, void** handle,
                     int64_t* nnz_filled) {
  auto* r = new (std::nothrow) SymbolicResult();
  if (!r) return LBK_ERR_OOM;
  try {
    int rc = symbolic_run(n, col_ptr, row_idx, r);
    if (rc) { delete r; return rc; }
  } catch (const std::bad_alloc&) {
    delete r;
    return LBK_ERR_OOM;
  }
  *handle = r;
  *nnz_filled = r->col_ptr[n];
  return 0;
}

int lbk_symbolic_fetch(void* handle, int64_t* col_ptr, int64_t* row_idx, int64_t* parent) {
  auto* r = static_cast<SymbolicResult*>(handle);
  copy_out(r->col_ptr, col_ptr);
  copy_out(r->row_idx, row_idx);
  copy_out(r->parent, parent);
  return 0;
}

void lbk_symbolic_free(void* handle) { delete static_cast<SymbolicResult*>(handle); }

// symbolic.py:46-54 (_require_symmetric_full_diag) in O(nnz): returns 0 if the
// pattern has a full diagonal and is structurally symmetric, 1 for a missing
// diagonal (*ndiag = count), 2 for asymmetry, 3 for unsorted/duplicate rows.
int lbk_check_symmetric(int64_t n, const int64_t* cp, const int64_t* ri, int64_t* ndiag) {
  int64_t nd = 0;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
      if (ri[e] == c) ++nd;
      if (e > cp[c] && ri[e] <= ri[e - 1]) return 3;
    }
  *ndiag = nd;
  if (nd != n) return 1;
  // transpose by counting sort; rows come out ascending per column because
  // source columns are scanned in order
  std::vector<int64_t> tp(n + 1, 0);
  for (int64_t e = 0; e < cp[n]; ++e) tp[ri[e] + 1]++;
  for (int64_t r = 0; r < n; ++r) tp[r + 1] += tp[r];
  for (int64_t c = 0; c <= n; ++c)
    if (tp[c] != cp[c]) return 2;
  std::vector<int64_t> w(tp.begin(), tp.end() - 1);
  std::vector<int64_t> ti(static_cast<size_t>(cp[n]));
  for (int64_t c = 0; c < n; ++c)
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e) ti[w[ri[e]]++] = c;
  for (int64_t e = 0; e < cp[n]; ++e)
    if (ti[e] != ri[e]) return 2;
  return 0;
}

int lbk_partition_run(int64_t n, const int64_t* f_col_ptr, const int64_t* f_row_idx,
                      const int64_t* a_col_ptr, const int64_t* a_row_idx, const double* a_values,
                      int64_t p, const int64_t* positions, void** handle, int64_t* nblocks,
                      int64_t* colptr_len) {
  auto* r = new (std::nothrow) PartitionResult();
  if (!r) return LBK_ERR_OOM;
  int rc;
  try {
    rc = partition_run(n, f_col_ptr, f_row_idx, a_col_ptr, a_row_idx, a_values, p, positions, r);
  } catch (const std::bad_alloc&) {
    rc = LBK_ERR_OOM;
  }
  if (rc) { delete r; return rc; }
  *handle = r;
  *nblocks = r->nblocks;
  *colptr_len = static_cast<int64_t>(r->col_ptr.size());
  return 0;
}

int lbk_partition_fetch(void* handle, int64_t* table /* 7 x nblocks */, int64_t* col_ptr,
                        int64_t* row_idx, double* values, int64_t* block_nnz) {
  auto* r = static_cast<PartitionResult*>(handle);
  const int64_t nb = r->nblocks;
  const std::vector<int64_t>* cols[7] = {&r->bi, &r->bj, &r->nrows, &r->ncols,
                                         &r->nnz, &r->cp_off, &r->ent_off};
  for (int k = 0; k < 7; ++k) copy_out(*cols[k], table + k * nb);
  copy_out(r->col_ptr, col_ptr);
  copy_out(r->row_idx, row_idx);
  copy_out(r->values, values);
  copy_out(r->block_nnz, block_nnz);
  return 0;
}

void lbk_partition_free(void* handle) { delete static_cast<PartitionResult*>(handle); }

int lbk_levels_run(int64_t p, int64_t nblocks, const int64_t* table /* 7 x nblocks */,
                   const int64_t* col_ptr, const int64_t* row_idx, void** handle,
                   int64_t* ntasks, int64_t* npreds) {
  auto* r = new (std::nothrow) LevelsResult();
  if (!r) return LBK_ERR_OOM;
  const int64_t nb = nblocks;
  int rc;
  try {
    rc = levels_run(p, nb, table, table + nb, table + 2 * nb, table + 3 * nb, table + 5 * nb,
                    table + 6 * nb, col_ptr, row_idx, r);
  } catch (const std::bad_alloc&) {
    rc = LBK_ERR_OOM;
  }
  if (rc) { delete r; return rc; }
  *handle = r;
  *ntasks = static_cast<int64_t>(r->kinds.size());
  *npreds = static_cast<int64_t>(r->pred_idx.size());
  return 0;
}

int lbk_levels_fetch(void* handle, int8_t* kinds, int32_t* steps, int32_t* rows, int32_t* cols,
                     int64_t* weights, int64_t* costs, int32_t* levels, int64_t* pred_ptr,
                     int32_t* pred_idx) {
  auto* r = static_cast<LevelsResult*>(handle);
  copy_out(r->kinds, kinds);
  copy_out(r->steps, steps);
  copy_out(r->rows, rows);
  copy_out(r->cols, cols);
  copy_out(r->weights, weights);
  copy_out(r->costs, costs);
  copy_out(r->levels, levels);
  copy_out(r->pred_ptr, pred_ptr);
  copy_out(r->pred_idx, pred_idx);
  return 0;
}

void lbk_levels_free(void* handle) { delete static_cast<LevelsResult*>(handle); }

}  // extern "C"
