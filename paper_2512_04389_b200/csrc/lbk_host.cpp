// Host-side structure path of the block LU engine (native, bit-exact with the
// reference's Python structure path).
//
//   lbk_symbolic_nnz/fill   ~ lublock.symbolic.symbolic_factorize   pkg/src/lublock/symbolic.py:57-108
//   lbk_check_symmetric     ~ symbolic._require_symmetric_full_diag  symbolic.py:46-54
//   lbk_blockptr            ~ lublock.features.diag_block_pointer    features.py:44-54 (Alg. 2)
//   lbk_partition_*         ~ lublock.grid.partition                 grid.py:85-148
//   lbk_levels_*            ~ lublock.grid.dependency_levels         grid.py:223-378
//
// All integer outputs equal the reference arrays element for element; the
// Python wrappers are tested against golden fixtures the reference produced.
// Large outputs are written straight into caller-allocated buffers (count
// first, then fill) so multi-GB patterns (C2: 347M entries) are produced in
// one pass without intermediate copies.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/lbk.h"

namespace {

// Row pattern of L for row i = the etree nodes reached by walking up from
// every j < i with A(i,j) != 0 until a node already marked for row i.  The
// walk is run twice: once to count, once to fill the caller's buffers.
// Column c of the union pattern is [sorted row pattern of c] ++ [c] ++
// [rows i > c whose pattern contains c, ascending] — exactly the
// (col,row)-sorted order the reference builds with a stable argsort.
template <class Visit>
void etree_walk(int64_t n, const int64_t* cp, const int64_t* ri, std::vector<int64_t>& parent,
                std::vector<int64_t>& mark, Visit visit) {
  std::fill(parent.begin(), parent.end(), -1);
  std::fill(mark.begin(), mark.end(), -1);
  for (int64_t i = 0; i < n; ++i) {
    mark[i] = i;
    for (int64_t e = cp[i]; e < cp[i + 1]; ++e) {
      int64_t j = ri[e];
      if (j >= i) break;  // rows sorted: the rest are >= i
      while (mark[j] != i) {
        visit(i, j);
        mark[j] = i;
        if (parent[j] == -1) parent[j] = i;
        j = parent[j];
      }
    }
  }
}

struct PartitionPlan {
  int64_t nblocks = 0, colptr_len = 0;
};

int partition_count(int64_t n, const int64_t* fcp, const int64_t* fri, int64_t p, const int64_t* pos,
                    PartitionPlan* out) {
  std::vector<int32_t> rowblk(n);
  for (int64_t b = 0; b < p; ++b)
    for (int64_t r = pos[b]; r < pos[b + 1]; ++r) rowblk[r] = static_cast<int32_t>(b);
  std::vector<char> seen(p);
  for (int64_t bj = 0; bj < p; ++bj) {
    std::fill(seen.begin(), seen.end(), 0);
    for (int64_t e = fcp[pos[bj]]; e < fcp[pos[bj + 1]]; ++e) seen[rowblk[fri[e]]] = 1;
    for (int64_t b = 0; b < p; ++b)
      if (seen[b]) {
        out->nblocks++;
        out->colptr_len += pos[bj + 1] - pos[bj] + 1;
      }
  }
  return 0;
}

int partition_fill(int64_t n, const int64_t* fcp, const int64_t* fri, const int64_t* acp, const int64_t* ari,
                   const double* aval, int64_t p, const int64_t* pos, int64_t* table, int64_t nb_total,
                   int64_t* col_ptr, int64_t* row_idx, double* values, int64_t* block_nnz, int64_t* apos) {
  std::vector<int32_t> rowblk(n);
  for (int64_t b = 0; b < p; ++b)
    for (int64_t r = pos[b]; r < pos[b + 1]; ++r) rowblk[r] = static_cast<int32_t>(b);
  std::fill(block_nnz, block_nnz + p * p, 0);
  int64_t *T_bi = table, *T_bj = table + nb_total, *T_nr = table + 2 * nb_total, *T_nc = table + 3 * nb_total,
          *T_nz = table + 4 * nb_total, *T_cp = table + 5 * nb_total, *T_ent = table + 6 * nb_total;
  std::vector<int64_t> cnt(p), start(p), w(p), blk_id(p);
  int64_t ent = 0, cpo = 0, nbk = 0;
  for (int64_t bj = 0; bj < p; ++bj) {
    const int64_t c0 = pos[bj], c1 = pos[bj + 1], nc = c1 - c0;
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int64_t e = fcp[c0]; e < fcp[c1]; ++e) cnt[rowblk[fri[e]]]++;
    int64_t acc = ent;
    for (int64_t b = 0; b < p; ++b) {
      blk_id[b] = -1;
      if (!cnt[b]) continue;
      start[b] = acc;
      acc += cnt[b];
      blk_id[b] = nbk;
      T_bi[nbk] = b;
      T_bj[nbk] = bj;
      T_nr[nbk] = pos[b + 1] - pos[b];
      T_nc[nbk] = nc;
      T_nz[nbk] = cnt[b];
      T_cp[nbk] = cpo;
      T_ent[nbk] = start[b];
      std::fill(col_ptr + cpo, col_ptr + cpo + nc + 1, 0);
      cpo += nc + 1;
      block_nnz[b * p + bj] = cnt[b];
      ++nbk;
    }
    std::copy(start.begin(), start.end(), w.begin());
    for (int64_t c = c0; c < c1; ++c) {
      int64_t a = acp[c];
      const int64_t a1 = acp[c + 1];
      for (int64_t e = fcp[c]; e < fcp[c + 1]; ++e) {
        const int64_t r = fri[e];
        const int32_t b = rowblk[r];
        const int64_t k = w[b]++;
        row_idx[k] = r - pos[b];
        // A's entries of this column are a sorted subset of the filled column
        double v = 0.0;
        if (a < a1 && ari[a] == r) {
          if (apos) apos[a] = k;  // pool position of A's entry a
          v = aval[a++];
        }
        values[k] = v;
        col_ptr[T_cp[blk_id[b]] + (c - c0) + 1]++;
      }
      if (a != a1) return LBK_ERR_DIM_MISMATCH;  // A not covered by the filled pattern
    }
    for (int64_t b = 0; b < p; ++b) {
      if (blk_id[b] < 0) continue;
      int64_t* cpb = col_ptr + T_cp[blk_id[b]];
      for (int64_t c = 0; c < nc; ++c) cpb[c + 1] += cpb[c];
    }
    ent = acc;
  }
  return nbk == nb_total ? 0 : LBK_ERR_BAD_ARG;
}

struct LevelsResult {
  std::vector<int8_t> kinds;
  std::vector<int32_t> steps, rows, cols, levels;
  std::vector<int64_t> weights, costs, pred_ptr;
  std::vector<int32_t> pred_idx;
};

// Static task DAG in construction order with ASAP levels (grid.py:223-378).
int levels_run(int64_t p, int64_t nblocks, const int64_t* bi, const int64_t* bj, const int64_t* nrows,
               const int64_t* ncols, const int64_t* cp_off, const int64_t* ent_off, const int64_t* col_ptr,
               const int64_t* row_idx, LevelsResult* out) {
  std::vector<int64_t> bid(static_cast<size_t>(p * p), -1);
  for (int64_t b = 0; b < nblocks; ++b) bid[bi[b] * p + bj[b]] = b;
  auto bnnz = [&](int64_t r, int64_t c) -> int64_t {
    const int64_t b = bid[r * p + c];
    return b < 0 ? 0 : col_ptr[cp_off[b] + ncols[b]];
  };
  std::vector<int64_t> ccoff(nblocks + 1, 0), rcoff(nblocks + 1, 0);
  for (int64_t b = 0; b < nblocks; ++b) {
    ccoff[b + 1] = ccoff[b] + ncols[b];
    rcoff[b + 1] = rcoff[b] + nrows[b];
  }
  std::vector<int64_t> ccnt(ccoff[nblocks]), rcnt(rcoff[nblocks], 0);
  for (int64_t b = 0; b < nblocks; ++b) {
    const int64_t* cpb = col_ptr + cp_off[b];
    for (int64_t c = 0; c < ncols[b]; ++c) ccnt[ccoff[b] + c] = cpb[c + 1] - cpb[c];
    for (int64_t e = 0; e < cpb[ncols[b]]; ++e) rcnt[rcoff[b] + row_idx[ent_off[b] + e]]++;
  }
  std::vector<int32_t> last_id(static_cast<size_t>(p * p), -1), last_lv(static_cast<size_t>(p * p), -1);
  std::vector<int64_t> pred_cnt, lows, ups;
  std::vector<int32_t> u_id(p), u_lv(p), l_id(p), l_lv(p);
  int32_t tid = 0;
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
    const int32_t glv = last_lv[i * p + i] + 1;
    push(0, i, i, i, dnnz, dnnz, glv);
    if (prev >= 0) {
      out->pred_idx.push_back(prev);
      pred_cnt.push_back(1);
    } else {
      pred_cnt.push_back(0);
    }
    const int32_t gid = tid++;
    for (int64_t j : ups) {
      prev = last_id[i * p + j];
      const int32_t lv = std::max(glv, last_lv[i * p + j]) + 1;
      const int64_t w = bnnz(i, j);
      push(1, i, i, j, w, w, lv);
      out->pred_idx.push_back(gid);
      if (prev >= 0) {
        out->pred_idx.push_back(prev);
        pred_cnt.push_back(2);
      } else {
        pred_cnt.push_back(1);
      }
      u_id[j] = tid++;
      u_lv[j] = lv;
    }
    for (int64_t k : lows) {
      prev = last_id[k * p + i];
      const int32_t lv = std::max(glv, last_lv[k * p + i]) + 1;
      const int64_t w = bnnz(k, i);
      push(2, i, k, i, w, w, lv);
      out->pred_idx.push_back(gid);
      if (prev >= 0) {
        out->pred_idx.push_back(prev);
        pred_cnt.push_back(2);
      } else {
        pred_cnt.push_back(1);
      }
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
        int64_t madds = 0;  // structural multiply-adds: dot(colcounts(L_ki), rowcounts(U_ij))
        for (int64_t r = 0; r < ncols[bl]; ++r) madds += cl[r] * ru[r];
        prev = last_id[k * p + j];
        const int32_t plv = last_lv[k * p + j];
        int32_t lv = std::max(l_lv[k], u_lv[j]);
        if (plv > lv) lv = plv;
        lv += 1;
        const int64_t nnz_u = bnnz(i, j), tgt = bnnz(k, j);
        int64_t w = nnz_l < nnz_u ? nnz_l : nnz_u;
        if (tgt > 0 && tgt < w) w = tgt;
        push(3, i, k, j, w, madds, lv);
        out->pred_idx.push_back(l_id[k]);
        out->pred_idx.push_back(u_id[j]);
        if (prev >= 0) {
          out->pred_idx.push_back(prev);
          pred_cnt.push_back(3);
        } else {
          pred_cnt.push_back(2);
        }
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

int lbk_symbolic_nnz(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* nnz_filled) {
  try {
    std::vector<int64_t> parent(n), mark(n);
    int64_t cnt = 0;
    etree_walk(n, col_ptr, row_idx, parent, mark, [&](int64_t, int64_t) { ++cnt; });
    *nnz_filled = 2 * cnt + n;
  } catch (const std::bad_alloc&) {
    return LBK_ERR_OOM;
  }
  return 0;
}

int lbk_symbolic_fill(int64_t n, const int64_t* cp, const int64_t* ri, int64_t* out_cp, int64_t* out_ri,
                      int64_t* parent_out) {
  try {
    std::vector<int64_t> parent(n), mark(n), rcount(n, 0), lcount(n, 0);
    etree_walk(n, cp, ri, parent, mark, [&](int64_t i, int64_t j) {
      rcount[i]++;
      lcount[j]++;
    });
    out_cp[0] = 0;
    for (int64_t c = 0; c < n; ++c) out_cp[c + 1] = out_cp[c] + rcount[c] + 1 + lcount[c];
    // U part (row pattern of c, unsorted then sorted in place) + diagonal;
    // the L part of column j is appended in ascending row order by the walk
    std::vector<int64_t> ucur(n), lcur(n);
    for (int64_t c = 0; c < n; ++c) {
      ucur[c] = out_cp[c];
      out_ri[out_cp[c] + rcount[c]] = c;
      lcur[c] = out_cp[c] + rcount[c] + 1;
    }
    etree_walk(n, cp, ri, parent, mark, [&](int64_t i, int64_t j) {
      out_ri[ucur[i]++] = j;
      out_ri[lcur[j]++] = i;
    });
    for (int64_t c = 0; c < n; ++c) std::sort(out_ri + out_cp[c], out_ri + out_cp[c] + rcount[c]);
    if (parent_out) std::copy(parent.begin(), parent.end(), parent_out);
  } catch (const std::bad_alloc&) {
    return LBK_ERR_OOM;
  }
  return 0;
}

// symbolic.py:46-54 in O(nnz): 0 ok, 1 missing diagonal (*ndiag = count),
// 2 asymmetric, 3 unsorted/duplicate rows.
int lbk_check_symmetric(int64_t n, const int64_t* cp, const int64_t* ri, int64_t* ndiag) {
  int64_t nd = 0;
  for (int64_t c = 0; c < n; ++c)
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e) {
      if (ri[e] == c) ++nd;
      if (e > cp[c] && ri[e] <= ri[e - 1]) return 3;
    }
  *ndiag = nd;
  if (nd != n) return 1;
  try {
    // transpose by counting sort; compare with the original pattern
    std::vector<int64_t> tp(n + 1, 0);
    for (int64_t e = 0; e < cp[n]; ++e) tp[ri[e] + 1]++;
    for (int64_t r = 0; r < n; ++r) tp[r + 1] += tp[r];
    for (int64_t c = 0; c <= n; ++c)
      if (tp[c] != cp[c]) return 2;
    std::vector<int64_t> w(tp.begin(), tp.end() - 1);
    std::vector<int32_t> ti(static_cast<size_t>(cp[n]));
    for (int64_t c = 0; c < n; ++c)
      for (int64_t e = cp[c]; e < cp[c + 1]; ++e) ti[w[ri[e]]++] = static_cast<int32_t>(c);
    for (int64_t e = 0; e < cp[n]; ++e)
      if (ti[e] != ri[e]) return 2;
  } catch (const std::bad_alloc&) {
    return LBK_ERR_OOM;
  }
  return 0;
}

// Alg. 2: num[r] = strictly-lower entries of row r; blockptr = prefix of 2*num+1.
int lbk_blockptr(int64_t n, const int64_t* cp, const int64_t* ri, int64_t* blockptr) {
  std::fill(blockptr, blockptr + n + 1, 0);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t e = cp[c]; e < cp[c + 1]; ++e)
      if (ri[e] > c) blockptr[ri[e] + 1]++;
  for (int64_t r = 0; r < n; ++r) blockptr[r + 1] = blockptr[r] + 2 * blockptr[r + 1] + 1;
  return 0;
}

int lbk_partition_count(int64_t n, const int64_t* f_col_ptr, const int64_t* f_row_idx, int64_t p,
                        const int64_t* positions, int64_t* nblocks, int64_t* colptr_len) {
  PartitionPlan pp;
  try {
    partition_count(n, f_col_ptr, f_row_idx, p, positions, &pp);
  } catch (const std::bad_alloc&) {
    return LBK_ERR_OOM;
  }
  *nblocks = pp.nblocks;
  *colptr_len = pp.colptr_len;
  return 0;
}

int lbk_partition_fill(int64_t n, const int64_t* f_col_ptr, const int64_t* f_row_idx, const int64_t* a_col_ptr,
                       const int64_t* a_row_idx, const double* a_values, int64_t p, const int64_t* positions,
                       int64_t nblocks, int64_t* table, int64_t* col_ptr, int64_t* row_idx, double* values,
                       int64_t* block_nnz, int64_t* a_pos) {
  try {
    return partition_fill(n, f_col_ptr, f_row_idx, a_col_ptr, a_row_idx, a_values, p, positions, table, nblocks,
                          col_ptr, row_idx, values, block_nnz, a_pos);
  } catch (const std::bad_alloc&) {
    return LBK_ERR_OOM;
  }
}

int lbk_levels_run(int64_t p, int64_t nblocks, const int64_t* table, const int64_t* col_ptr,
                   const int64_t* row_idx, void** handle, int64_t* ntasks, int64_t* npreds) {
  auto* r = new (std::nothrow) LevelsResult();
  if (!r) return LBK_ERR_OOM;
  const int64_t nb = nblocks;
  int rc;
  try {
    rc = levels_run(p, nb, table, table + nb, table + 2 * nb, table + 3 * nb, table + 5 * nb, table + 6 * nb,
                    col_ptr, row_idx, r);
  } catch (const std::bad_alloc&) {
    rc = LBK_ERR_OOM;
  }
  if (rc) {
    delete r;
    return rc;
  }
  *handle = r;
  *ntasks = static_cast<int64_t>(r->kinds.size());
  *npreds = static_cast<int64_t>(r->pred_idx.size());
  return 0;
}

int lbk_levels_fetch(void* handle, int8_t* kinds, int32_t* steps, int32_t* rows, int32_t* cols, int64_t* weights,
                     int64_t* costs, int32_t* levels, int64_t* pred_ptr, int32_t* pred_idx) {
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
