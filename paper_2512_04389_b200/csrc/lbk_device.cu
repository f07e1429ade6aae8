// lbk_device.cu — sm_100a block-LU engine behind the C-ABI of include/lbk.h.
//
// Replaces the numerical factorization of the reference,
//   lublock.factorize.factorize(grid, tree, ...)   pkg/src/lublock/factorize.py:245-384
// with a level-by-level device scheduler: every dependency level of the task
// DAG (grid.py:223-378) becomes one batch of launches over work lists of
// (task, tile / column / row range) items, forked onto parallel graph
// branches by kernel family and joined before the next level; all levels are
// captured once into a CUDA graph and replayed.
//
// Per factorization the graph runs: zero the working pool, scatter A's values
// (reference pool order) into it, all levels, gather the factors back into
// reference pool order.  The block storage kinds and kernels are described in
// lbk_common.cuh, lbk_sparse.cuh and lbk_dense.cuh.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>
#include <set>
#include <queue>
#include <functional>

#include "../../include/lbk.h"
#include <iterator>
#include <limits>
#include <map>

#include "lbk_common.cuh"
#include "lbk_dense.cuh"
#include "lbk_exec.cuh"
#include "lbk_solve.cuh"
#include "lbk_sparse.cuh"

#include <array>
#include <cstdlib>

using namespace lbk;

namespace {

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    release();
    n = count;
    return cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
  }
  cudaError_t upload(const std::vector<T>& v) {
    cudaError_t e = alloc(v.size());
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    // a pageable cudaMemcpy may return before its DMA lands, and it is not ordered
    // with the non-blocking engine streams: finish it before any kernel reads p
    if (e == cudaSuccess && !v.empty()) e = cudaDeviceSynchronize();
    return e;
  }
};

struct SubStep {  // one sub-step kb of the tiled GETRFs of a level
  int64_t getrf_off, trsm_off, gemm_off;
  int32_t ngetrf, ntrsm, ngemm;
};

struct Level {
  int64_t item_off;  // generic items
  int32_t nitems, warps, acc_len;
  int64_t gemm_off;  // SSSSM DMMA tiles
  int32_t ngemm;
  int64_t gemmD_off;  // deferred SSSSM DMMA tiles (every successor exactly 2 tree levels later)
  int32_t ngemmD;
  int64_t gemmE_off;  // deferred SSSSM DMMA tiles with >= 3 levels of slack
  int32_t ngemmE;
  int64_t gred_off;   // split-K reductions of the critical SSSSM tiles
  int32_t ngred;
  int64_t absorb_off;  // SSSSM tiles run as tasks of the next executor launch (exact mode: launched here)
  int32_t nabsorb;
  int64_t panel_off;  // dense GESSM/TSTRF strips
  int32_t npanel;
  int32_t panel_smem;
  int64_t exact_off;  // exact single-CTA GETRF items (dense-scratch / static pivot)
  int32_t nexact;
  int32_t exact_smem;
  int64_t tcol_off;   // tiled GETRF: colmax items
  int32_t ntcol;
  int64_t sub_off;    // index into subs
  int32_t nsub;
  int64_t tfin_off;   // finalize items
  int32_t ntfin;
  int64_t exec_off, sptr_off, succ_off;  // persistent tile-DAG executor (tiled mode)
  int32_t nexec;
  int32_t band4 = 0;      // holds band sweeps of half-bandwidth 4: exec_band_kernel
  int32_t tree_level;     // ASAP level of the task DAG this launch level runs
  int32_t tree_level_hi;  // last tree level whose executor work runs in this launch (merged panel level)
};

constexpr int NBRANCH = 3;

// Builds one level's tile-DAG for the persistent executor: tasks get a
// priority key (elimination sub-step first); flush() orders them by key
// (topological within every DAG) and emits counters and successor lists.
#ifndef LBK_TWO_PHASE
#define LBK_TWO_PHASE 1  // GETRF_UPD / TRSM tiles load their target before their operands are ready
#endif

#ifndef LBK_SPLITK
#define LBK_SPLITK 1  // split-K for critical DMMA SSSSM launches with few tiles
#endif
constexpr int SPLITK_TILES = 2 * 148 * 2;  // fill ~2 waves of 2 CTAs per SM
constexpr int SPLITK_MIN_CHUNKS = 4;       // inner chunks per part at least

#ifndef LBK_CHAIN_TRSM
#define LBK_CHAIN_TRSM 0  // 1: the diagonal LU task also solves the next step's two update operands (measured slower: the two solves then run one after the other instead of on two CTAs)
#endif

// Tile boundaries of a diagonal block for the executor (block-local CSC of its filled,
// structurally symmetric pattern): at most XT columns per tile, and a new tile wherever a
// new elimination subtree starts while the current tile holds an ancestor of earlier
// columns.  Uniform 64-column tiles straddle subtree boundaries, so tile (k+1, k) is
// nonempty for almost every k and the LU runs as one chain through all diagonal tiles;
// with subtree-aligned tiles independent subtrees (nested-dissection leaves inside a
// block) become independent tile chains.  Any partition is correct: only the schedule
// and the operation order inside the tiles change (C2 model: sum of the blocks' critical
// paths 148 -> 65 ms).  parent(j) = min{i > j : (i, j) in the pattern},
// fd(j) = first column of j's subtree (contiguous when the order is a postorder).
// seg[j] (optional): index of the subtree-cut region holding column j (the panel solves
// of the block's row / column cut their chain dimension where it changes).
static std::vector<int32_t> subtree_tiles(int m, const int64_t* cp, const int64_t* ri, int T, int minw,
                                          std::vector<int32_t>* seg = nullptr) {
  std::vector<int32_t> par(m, -1), fd(m), b{0};
  if (seg) seg->assign(m, 0);
  for (int j = 0; j < m; ++j) {
    fd[j] = j;
    for (int64_t e = cp[j]; e < cp[j + 1]; ++e) {
      const int r = static_cast<int>(ri[e]);
      if (r > j && (par[j] < 0 || r < par[j])) par[j] = r;
    }
  }
  for (int j = 0; j < m; ++j)
    if (par[j] >= 0) fd[par[j]] = std::min(fd[par[j]], fd[j]);
  int s = 0, mfd = m;
  for (int j = 1; j < m; ++j) {
    mfd = std::min(mfd, fd[j - 1]);  // tile [s, j) holds an ancestor of a column < s iff mfd < s
    const bool new_subtree = par[j - 1] != j;
    const bool cut = new_subtree && mfd < s && j - s >= minw;
    if (j - s == T || cut) {
      b.push_back(j);
      s = j;
      mfd = m;
    }
    if (seg) (*seg)[j] = (*seg)[j - 1] + (cut ? 1 : 0);
  }
  if (m > 0) b.push_back(m);
  return b;
}

// Modelled critical path (us) of a diagonal block's tile LU under tiling tb: the executor's
// tile DAG (GETRF -> TRSM_L / TRSM_U -> GEMM updates, per-tile update chains, structurally
// empty tiles skipped) with per-task latencies measured on B200 (a task costs a fixed part
// plus a part per column of its elimination tile, ~0.8 us per handoff).  Used to keep the
// subtree-aligned tiling only where it shortens the chain: on blocks whose subtrees are
// tiny it fragments the tiles and lengthens it (C5's border blocks).
static double tile_cp_model(int m, const int64_t* cp, const int64_t* ri, const std::vector<int32_t>& tb) {
  const int nt = static_cast<int>(tb.size()) - 1;
  if (nt <= 0) return 0.0;
  std::vector<int32_t> tid(m);
  for (int x = 0; x < nt; ++x)
    for (int y = tb[x]; y < tb[x + 1]; ++y) tid[y] = x;
  std::vector<char> occ(static_cast<size_t>(nt) * nt, 0);  // [row tile * nt + col tile]
  for (int j = 0; j < m; ++j)
    for (int64_t e = cp[j]; e < cp[j + 1]; ++e) occ[static_cast<size_t>(tid[ri[e]]) * nt + tid[j]] = 1;
  std::vector<double> rd(static_cast<size_t>(nt) * nt, 0.0);
  auto R = [&](int r, int c) -> double& { return rd[static_cast<size_t>(r) * nt + c]; };
  auto O = [&](int r, int c) { return occ[static_cast<size_t>(r) * nt + c] != 0; };
  constexpr double H = 0.8;
  for (int k = 0; k < nt; ++k) {
    const double w = tb[k + 1] - tb[k];
    const double tg = R(k, k) + H + 5.0 + 0.27 * w;
    R(k, k) = tg;
    for (int r = k + 1; r < nt; ++r) {
      if (O(r, k)) R(r, k) = std::max(R(r, k), tg) + H + 3.0 + 0.1 * w;
      if (O(k, r)) R(k, r) = std::max(R(k, r), tg) + H + 3.0 + 0.1 * w;
    }
    for (int c = k + 1; c < nt; ++c) {
      if (!O(k, c)) continue;
      for (int r = k + 1; r < nt; ++r)
        if (O(r, k)) R(r, c) = std::max({R(r, c), R(r, k), R(k, c)}) + H + 4.0 + 0.06 * w;
    }
  }
  return *std::max_element(rd.begin(), rd.end());
}

struct ExecBuilder {
  std::vector<XTask> t;
  std::vector<int64_t> key;
  std::vector<std::vector<int>> preds, preds2;  // phase-1 / phase-2 dependencies
  std::set<std::pair<int, int>> early;          // (chain-2 GETRF task, successor released after its LU)
  void mark_early(int p, int s) { early.insert({p, s}); }
  // deps2: dependencies the task waits for only after its phase-1 loads (the target tile of
  // GETRF_UPD / TRSM is loaded while its operands are still being produced)
  int add(int type, int64_t a, int64_t d, int r, int c, int k, int32_t step, int64_t prio, std::vector<int> deps,
          std::vector<int> deps2 = {}) {
    XTask x{};
    x.type = static_cast<int8_t>(type);
    x.r = static_cast<int16_t>(r);
    x.c = static_cast<int16_t>(c);
    x.k = static_cast<int16_t>(k);
    x.a = static_cast<int32_t>(a);
    x.d = static_cast<int32_t>(d);
    x.step = step;
    t.push_back(x);
    key.push_back(prio);
    auto clean = [](std::vector<int>& v) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      while (!v.empty() && v.front() < 0) v.erase(v.begin());
    };
    clean(deps);
    clean(deps2);
    if (!LBK_TWO_PHASE) {  // everything in phase 1
      deps.insert(deps.end(), deps2.begin(), deps2.end());
      deps2.clear();
      clean(deps);
    }
    std::vector<int> d1;
    std::set_difference(deps.begin(), deps.end(), deps2.begin(), deps2.end(), std::back_inserter(d1));
    preds.push_back(std::move(d1));
    preds2.push_back(std::move(deps2));
    return static_cast<int>(t.size()) - 1;
  }
  // Dequeue order = descending upward rank (longest cost path to the end of
  // the level's DAG; per-type costs are measured tile latencies in 0.1 us).
  // That is a topological order (a task outranks all its successors) and it
  // is the lookahead schedule: the next panel's GETRF/TRSM tiles and the
  // GEMMs feeding them overtake the bulk trailing updates of the current
  // step, which a plain step-major order would dequeue first.
  static int cost_of(int type) {
    static const int c[15] = {150, 360, 180, 130, 64, 60, 130, 64, 180, 64, 100000, 420, 190, 240, 1};
    return type >= 0 && type < 15 ? c[type] : 64;
  }
  void flush(Level* L, std::vector<XTask>* tasks, std::vector<int32_t>* sptr, std::vector<int32_t>* succ,
             std::vector<int32_t>* deps0) {
    const int n = static_cast<int>(t.size());
    std::vector<int> order(n), pos(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    {
      // insertion order is topological (deps always name earlier tasks)
      std::vector<std::vector<int>> fwd(n);
      for (int i = 0; i < n; ++i) {
        for (int p : preds[i]) fwd[p].push_back(i);
        for (int p : preds2[i]) fwd[p].push_back(i);
      }
      std::vector<int64_t> rank(n, 0);
      for (int i = n - 1; i >= 0; --i) {
        int64_t m = 0;
        for (int s2 : fwd[i]) m = std::max(m, rank[s2]);
        rank[i] = m + (t[i].type == X_SSSSM ? 30 + 26 * t[i].k : cost_of(t[i].type)) +
                  (t[i].chain == 1 ? cost_of(X_TRSM_L) + cost_of(X_TRSM_U) : t[i].chain == 2 ? cost_of(X_TRSM_L) : 0);
      }
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return rank[x] > rank[y]; });
    }
    for (int i = 0; i < n; ++i) pos[order[i]] = i;
    // successor entries: (task << 1) | phase; a chain-2 GETRF task lists its early successors
    // first and records their count in pad1
    std::vector<std::vector<int>> out(n), out_early(n);
    for (int i = 0; i < n; ++i) {
      for (int p : preds[i]) (early.count({p, i}) ? out_early : out)[pos[p]].push_back(pos[i] << 1);
      for (int p : preds2[i]) (early.count({p, i}) ? out_early : out)[pos[p]].push_back((pos[i] << 1) | 1);
    }
    for (int q = 0; q < n; ++q) {
      if (out_early[pos[q]].empty()) continue;  // (pad1 of other task types keeps its own meaning)
      t[q].pad1 = static_cast<int16_t>(out_early[pos[q]].size());
      out[pos[q]].insert(out[pos[q]].begin(), out_early[pos[q]].begin(), out_early[pos[q]].end());
    }
    L->exec_off = static_cast<int64_t>(tasks->size());
    L->nexec = n;
    L->band4 = 0;
    for (int i = 0; i < n; ++i) L->band4 |= t[i].type == X_BAND && t[i].r == 4 && t[i].c == 4;
    L->sptr_off = static_cast<int64_t>(sptr->size());
    L->succ_off = static_cast<int64_t>(succ->size());
    int32_t acc = 0;
    for (int i = 0; i < n; ++i) {
      tasks->push_back(t[order[i]]);
      deps0->push_back(static_cast<int32_t>(preds[order[i]].size()));
      deps0->push_back(static_cast<int32_t>(preds2[order[i]].size()));
      sptr->push_back(acc);
      for (int s2 : out[i]) succ->push_back(s2);
      acc += static_cast<int32_t>(out[i].size());
    }
    sptr->push_back(acc);
  }
};

}  // namespace

struct lbk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux[NBRANCH] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork = nullptr, join[NBRANCH] = {nullptr, nullptr, nullptr};
  cudaStream_t dstream = nullptr;     // deferred SSSSM branch (lowest priority)
  cudaEvent_t dfork = nullptr;
  std::vector<cudaEvent_t> dev, dev2; // per launch level: deferred work done (slack 2 / >= 3)
  cudaStream_t dstream2 = nullptr;
  std::vector<int8_t> defer;          // per task: may run concurrently with the next level
  int exec_per_sm = 2;
  int band_per_sm = 1;  // exec_band_kernel residency (register bound)
  bool use_bandreg = true;  // LBK_NO_BANDREG: band levels on the plain executor (A/B experiments)
  int defer_ctas = 0;  // > 0: deferred SSSSM work on this many looping CTAs (LBK_DEFER_CTAS)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaGraphExec_t> graphs;  // one per segment (see lbk_set_cuts)
  double g_tol = NAN, g_eps = NAN;
  int32_t flags = 0;
  // plan
  int64_t n = 0, p = 0, nblocks = 0, nnz = 0, nnz_work = 0, ndiag_rows = 0;
  std::vector<BlockDev> hblk;
  std::vector<Level> levels;
  std::vector<SubStep> subs;
  std::vector<int8_t> route;  // per task: -1 skipped, 0 CSC kernel, 1 DMMA SSSSM, 2 panel, 3 tiled GETRF
  int64_t n_generic = 0, n_gemm = 0, n_panel = 0, n_tile = 0;
  int64_t store_count[3] = {0, 0, 0};
  // device
  DevBuf<BlockDev> blk;
  DevBuf<int32_t> colptr, rows, csr_ptr, csr_col, csr_pos, diag_csc, diag_csr, lv_cols, lv_ptr, rlist, clist,
      maps, perm;
  DevBuf<int64_t> map;
  DevBuf<double> vals, vin, vout, colmax;
  DevBuf<unsigned long long> bmax, err;
  DevBuf<int> dirty;  // [0]: working pool needs zeroing before the next run; [1]: non-finite input seen
  DevBuf<Item> items;
  DevBuf<GemmTask> gtasks;
  DevBuf<GemmItem> gitems;
  DevBuf<int32_t> kchunks;
  DevBuf<double> gemm_ws;  // split-K partial products
  DevBuf<DenseItem> ditems;
  DevBuf<TileItem> titems;
  DevBuf<XTask> xtasks;
  DevBuf<int32_t> xsptr, xsucc, xdeps0;
  DevBuf<int32_t> xtb;  // executor tile boundaries per tiled diagonal block (BlockDev::xtb1)
  DevBuf<int> xdeps, xheads;
  DevBuf<int32_t> perm0;  // identity permutation per diagonal row
  int64_t n_exec = 0;
  double dmma_flops = 0, exec_flops = 0;  // executed (tile-shaped) flops per factorization
  bool use_exec = true;
  // distribution (lbk_set_task_mask / lbk_set_cuts): tasks this rank runs, and
  // the tree levels after which the graph is cut for a block exchange
  std::vector<int8_t> mask, cut_after;
  std::vector<int32_t> seg_begin;  // launch-level index where each segment starts (+ end sentinel)
  std::vector<int64_t> wlen;       // working entries per block
  std::vector<char> isdiag;
  // device triangular solve (lbk_solve): block grid + lazily built graph
  std::vector<int64_t> pos, hbi, hbj;
  // streamed end-to-end output: each block's factor values leave for the host
  // as soon as the level that finishes it is done (lbk_factorize_host)
  std::vector<int32_t> blk_final_tl;  // tree level of the task that finishes each block

  std::vector<int64_t> ref_off, ref_len;  // reference pool range of each block
  std::vector<char> resident;             // block has working storage on this rank
  bool refined = false;                   // segment-refined levels (lbk_plan flags bit 2)
  // output layout (lbk_set_export): entries nout, per-block range, omap[x] = working
  // position of output entry x (-1: a constant 1.0, the unit diagonal of L)
  int64_t nout = 0;
  std::vector<int64_t> out_off, out_len;
  DevBuf<int64_t> omap, zcount, out_off_d;
  cudaStream_t cstream = nullptr;
  cudaEvent_t cev = nullptr;
  std::vector<cudaEvent_t> lev;     // per launch level: critical work done (copy-stream fork)
  // streamed-output graphs, one per host output buffer (two slots: a caller
  // alternating between two buffers - the previous factors still alive - does
  // not recapture)
  struct SGraph {
    cudaGraphExec_t g = nullptr;
    double* out = nullptr;
    double tol = NAN, eps = NAN;
    uint64_t used = 0;
  } sg[2];
  uint64_t sg_clock = 0;
  DevBuf<int64_t> sranges;          // (offset, length) pairs, grouped by launch level
  std::vector<int64_t> hsranges;
  std::vector<int64_t> spiece_off;  // per launch level: first gather piece (+ sentinel)
  // refactorization input: A's entries (CSC order) -> reference pool positions
  DevBuf<int64_t> amap;
  DevBuf<double> avals;
  int64_t nnz_a = 0;
  std::vector<int64_t> srange_off;  // per launch level: first pair index (+ sentinel)
  std::vector<int32_t> dext;       // per diagonal block, per 64-col chunk: (row hi, row lo) of its pattern
  std::vector<int64_t> dext_off;   // per block: offset into dext (diagonal blocks)
  DevBuf<int32_t> sdext;
  // banded FULL diagonal blocks (from lbk_plan): bandwidths and segments for the band solve
  std::vector<int32_t> band_bl, band_bu, band_seg;
  std::vector<int64_t> band_off;
  DevBuf<int32_t> sbandseg;
  DevBuf<SolveStep> sfw, sbw;
  DevBuf<SolveUpd> ufw, ubw;
  DevBuf<int32_t> sbstart, tistep, titile;
  DevBuf<int64_t> sdgrow;
  DevBuf<double> sb, sv, stinv;
  int64_t n_tinv = 0;
  cudaGraphExec_t solve_graph = nullptr;
  DevBuf<unsigned long long> xtrace;  // executor task timeline (instrumented replays only)
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

#define LBK_CUDA(call, st)                                    \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
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
  P.rlist = c->rlist.p;
  P.clist = c->clist.p;
  P.maps = c->maps.p;
  P.kchunks = c->kchunks.p;
  P.gemm_ws = c->gemm_ws.p;
  P.perm = c->perm.p;
  P.colmax = c->colmax.p;
  P.bmax = c->bmax.p;
  P.err = c->err.p;
  P.xtb = c->xtb.p;
  return P;
}

// output map: the export map when set, else the reference-pool map
const int64_t* out_map(const lbk_ctx* c) { return c->omap.p ? c->omap.p : c->map.p; }

void drop_sgraphs(lbk_ctx* c) {
  for (auto& q : c->sg) {
    if (q.g) cudaGraphExecDestroy(q.g);
    q = lbk_ctx::SGraph{};
  }
}

void drop_graphs(lbk_ctx* c) {
  for (auto g : c->graphs)
    if (g) cudaGraphExecDestroy(g);
  c->graphs.clear();
}

constexpr double RECT_SMALL = 64.0 * 64.0;
constexpr size_t DEFER_MIN_TILES = 64;  // smaller deferred groups run with the level's critical SSSSM launch

int choose_warps(int acc_len) { return std::max(1, std::min(4, MAX_SMEM / (acc_len * 8))); }

// positions of `sub` inside sorted `sup` (-1 if absent); identity flag
std::vector<int32_t> positions_in(const std::vector<int32_t>& sub, const std::vector<int32_t>& sup, bool* identity) {
  std::vector<int32_t> out(sub.size());
  size_t j = 0;
  bool id = sub.size() == sup.size();
  for (size_t i = 0; i < sub.size(); ++i) {
    while (j < sup.size() && sup[j] < sub[i]) ++j;
    out[i] = (j < sup.size() && sup[j] == sub[i]) ? static_cast<int32_t>(j) : -1;
    if (out[i] != static_cast<int32_t>(i)) id = false;
  }
  *identity = id;
  return out;
}

}  // namespace

extern "C" {

int lbk_create(lbk_ctx** out, int device, lbk_status* st) {
  auto* c = new (std::nothrow) lbk_ctx();
  if (!c) return fail(st, LBK_ERR_OOM, "ctx alloc");
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  int prio_lo = 0, prio_hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  // critical-path streams at the highest priority: graph kernel nodes inherit
  // it (instantiated with cudaGraphInstantiateFlagUseNodePriority), so the
  // block scheduler serves them before the deferred SSSSM branch
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(gemm_map_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tile_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSM_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tile_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TGEMM_SMEM);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(exec_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM);
  if (e == cudaSuccess) {
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, exec_band_kernel, 256, EXEC_SMEM);
    c->band_per_sm = std::max(1, nb);
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(solve_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(solve_upd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(solve_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(tile_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (2 * XREG + XT) * sizeof(double));
  c->use_exec = std::getenv("LBK_NO_EXEC") == nullptr;
  for (int k = 0; k < NBRANCH && e == cudaSuccess; ++k) {
    e = cudaStreamCreateWithPriority(&c->aux[k], cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join[k], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->dstream, cudaStreamNonBlocking, prio_lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->dstream2, cudaStreamNonBlocking, prio_lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking);

  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->cev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->dfork, cudaEventDisableTiming);
  if (const char* x = std::getenv("LBK_EXEC_PER_SM")) c->exec_per_sm = std::max(1, std::atoi(x));
  c->use_bandreg = std::getenv("LBK_NO_BANDREG") == nullptr;
  if (const char* x = std::getenv("LBK_DEFER_CTAS")) c->defer_ctas = std::max(0, std::atoi(x));
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
  for (auto g : c->graphs)
    if (g) cudaGraphExecDestroy(g);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (int k = 0; k < NBRANCH; ++k) {
    if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
    if (c->join[k]) cudaEventDestroy(c->join[k]);
  }
  if (c->fork) cudaEventDestroy(c->fork);
  for (auto ev : c->dev) cudaEventDestroy(ev);
  for (auto ev : c->dev2) cudaEventDestroy(ev);
  if (c->dstream) cudaStreamDestroy(c->dstream);
  if (c->dstream2) cudaStreamDestroy(c->dstream2);
  if (c->cstream) cudaStreamDestroy(c->cstream);

  if (c->cev) cudaEventDestroy(c->cev);
  for (auto ev : c->lev) cudaEventDestroy(ev);
  for (auto& q : c->sg)
    if (q.g) cudaGraphExecDestroy(q.g);
  if (c->dfork) cudaEventDestroy(c->dfork);
  if (c->solve_graph) cudaGraphExecDestroy(c->solve_graph);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"

namespace {
// Per launch level: the output ranges (c->out_off / out_len: reference pool order,
// or the export layout) of the blocks the level finishes, for the streamed output.
int build_out_ranges(lbk_ctx* c, lbk_status* st) {
  const int64_t nb = static_cast<int64_t>(c->out_off.size());
  {
    // per launch level: the output ranges of the blocks it finishes
    // (adjacent blocks merged; pool order is column-major block order)
    std::vector<std::vector<std::pair<int64_t, int64_t>>> per(c->levels.size());
    std::vector<int32_t> tl_to_l;
    for (size_t l = 0; l < c->levels.size(); ++l) {
      const int32_t hi = c->levels[l].tree_level_hi;
      if (static_cast<int32_t>(tl_to_l.size()) <= hi) tl_to_l.resize(hi + 1, -1);
      for (int32_t tl = c->levels[l].tree_level; tl <= hi; ++tl)
        if (tl_to_l[tl] < 0 || tl == c->levels[l].tree_level) tl_to_l[tl] = static_cast<int32_t>(l);
    }
    for (int64_t b = 0; b < nb; ++b) {
      const int32_t tl = c->blk_final_tl[b];
      if (tl < 0 || tl >= static_cast<int32_t>(tl_to_l.size()) || tl_to_l[tl] < 0 || c->out_len[b] == 0) continue;
      auto& v = per[tl_to_l[tl]];
      if (!v.empty() && v.back().first + v.back().second == c->out_off[b]) v.back().second += c->out_len[b];
      else v.push_back({c->out_off[b], c->out_len[b]});
    }
    std::vector<int64_t> flat, pieces;  // copy ranges; gather pieces of <= 64K entries (one CTA each)
    c->srange_off.assign(1, 0);
    c->spiece_off.assign(1, 0);
    constexpr int64_t PIECE = 1 << 16;
    for (auto& v : per) {
      for (auto& pr : v) {
        flat.push_back(pr.first);
        flat.push_back(pr.second);
        for (int64_t o = 0; o < pr.second; o += PIECE) {
          pieces.push_back(pr.first + o);
          pieces.push_back(std::min(PIECE, pr.second - o));
        }
      }
      c->srange_off.push_back(static_cast<int64_t>(flat.size() / 2));
      c->spiece_off.push_back(static_cast<int64_t>(pieces.size() / 2));
    }
    LBK_CUDA(c->sranges.upload(pieces.empty() ? std::vector<int64_t>(2, 0) : pieces), st);
    c->hsranges = flat;
  }
  ok(st);
  return 0;
}

}  // namespace

extern "C" {

// Build the device plan.  flags bit 0: DMMA storage/kernels (diagonal blocks
// FULL, blocks whose R x C rectangle is >= tau dense RECT); bit 1: dense-
// scratch mode (every block FULL, true row swaps).  Without bit 0 every
// block stays SPARSE (CSC kernels only).
int lbk_plan(lbk_ctx* c, int64_t n, int64_t p, const int64_t* positions, int64_t nblocks, const int64_t* table,
             const int64_t* colptr, const int64_t* rowidx, int64_t ntasks, const int8_t* kinds,
             const int32_t* steps, const int32_t* trows, const int32_t* tcols, const int32_t* tlevels,
             const int64_t* costs, int32_t chunk, int32_t flags, double tau, lbk_status* st) {
  if (!c) return fail(st, LBK_ERR_BAD_ARG, "null ctx");
  LBK_CUDA(cudaSetDevice(c->device), st);
  c->pos.assign(positions, positions + p + 1);
  c->hbi.assign(table, table + nblocks);
  c->hbj.assign(table + nblocks, table + 2 * nblocks);
  if (c->solve_graph) {
    cudaGraphExecDestroy(c->solve_graph);
    c->solve_graph = nullptr;
  }
  const int64_t nb = nblocks;
  const int64_t *T_bi = table, *T_bj = table + nb, *T_nr = table + 2 * nb, *T_nc = table + 3 * nb,
                *T_nz = table + 4 * nb, *T_cp = table + 5 * nb, *T_ent = table + 6 * nb;
  const bool dense_on = (flags & 1) != 0, all_full = (flags & 2) != 0;
  c->flags = flags;
  c->dmma_flops = c->exec_flops = 0;
  c->n = n;
  c->p = p;
  c->nblocks = nb;
  if (chunk < 1) chunk = 8;
  std::vector<int64_t> bid(static_cast<size_t>(p * p), -1);
  for (int64_t b = 0; b < nb; ++b) bid[T_bi[b] * p + T_bj[b]] = b;
  for (int64_t i = 0; i < p; ++i)
    if (bid[i * p + i] < 0) return fail(st, LBK_ERR_DIM_MISMATCH, "missing diagonal block");
  try {
    // ---- storage kind, R / C lists ------------------------------------------------
    std::vector<BlockDev> hb(nb);
    c->wlen.assign(nb, 0);
    c->ref_off.assign(T_ent, T_ent + nb);
    c->ref_len.assign(T_nz, T_nz + nb);
    c->out_off = c->ref_off;
    c->out_len = c->ref_len;
    c->omap.release();
    c->zcount.release();
    c->blk_final_tl.assign(nb, -1);
    for (int64_t t = 0; t < ntasks; ++t) {
      const int64_t i = steps[t];
      int64_t fb = -1;
      if (kinds[t] == KIND_GETRF) fb = bid[i * p + i];
      else if (kinds[t] == KIND_GESSM) fb = bid[i * p + tcols[t]];
      else if (kinds[t] == KIND_TSTRF) fb = bid[trows[t] * p + i];
      if (fb >= 0) c->blk_final_tl[fb] = tlevels[t];  // (refined plans: reset below)
    }

    c->dext.clear();
    c->dext_off.assign(nb, -1);
    c->isdiag.assign(nb, 0);
    for (int64_t b = 0; b < nb; ++b) c->isdiag[b] = T_bi[b] == T_bj[b];
    if (!c->mask.empty() && static_cast<int64_t>(c->mask.size()) != ntasks)
      return fail(st, LBK_ERR_DIM_MISMATCH, "task mask length differs from the task count");
    std::vector<std::vector<int32_t>> Rl(nb), Cl(nb);
    // distributed plans (task mask): working storage only for the blocks this rank's
    // tasks write or read (owned blocks + received operands); other blocks get none
    // and their pool entries map to -2 (skipped by the scatter, zero in the output)
    std::vector<char> resident(nb, c->mask.empty() ? 1 : 0);
    if (!c->mask.empty()) {
      auto mark = [&](int64_t bi, int64_t bj) {
        if (bi >= 0 && bj >= 0 && bid[bi * p + bj] >= 0) resident[bid[bi * p + bj]] = 1;
      };
      for (int64_t t = 0; t < ntasks; ++t) {
        if (!c->mask[t]) continue;
        const int64_t i = steps[t], r = trows[t], cc = tcols[t];
        mark(i, i);
        if (kinds[t] == KIND_GESSM) mark(i, cc);
        else if (kinds[t] == KIND_TSTRF) mark(r, i);
        else if (kinds[t] == KIND_SSSSM) {
          mark(r, i);
          mark(i, cc);
          mark(r, cc);
        }
      }
    }
    c->resident.assign(resident.begin(), resident.end());
    int64_t nnz = 0, nnz_w = 0, ncp = 0;
    for (int64_t b = 0; b < nb; ++b) {
      BlockDev& d = hb[b];
      std::memset(&d, 0, sizeof(d));
      d.nrows = static_cast<int32_t>(T_nr[b]);
      d.ncols = static_cast<int32_t>(T_nc[b]);
      d.rp = d.csr = d.roff = d.coff = -1;
      const int64_t* scp = colptr + T_cp[b];
      const int64_t* sri = rowidx + T_ent[b];
      const int64_t nzb = T_nz[b];
      nnz += nzb;
      const bool diag = T_bi[b] == T_bj[b];
      const int64_t area = static_cast<int64_t>(d.nrows) * d.ncols;
      int store = STORE_SPARSE;
      if (all_full || (dense_on && (diag || nzb == area))) {
        store = STORE_FULL;
      } else if (dense_on && nzb > 0) {
        std::vector<char> rmark(d.nrows, 0);
        for (int64_t e = 0; e < nzb; ++e) rmark[sri[e]] = 1;
        std::vector<int32_t> R, Cc;
        for (int r = 0; r < d.nrows; ++r)
          if (rmark[r]) R.push_back(r);
        for (int col = 0; col < d.ncols; ++col)
          if (scp[col + 1] > scp[col]) Cc.push_back(col);
        const double rect = static_cast<double>(R.size()) * Cc.size();
        // small rectangles go dense regardless of their fill: a <= 64 x 64 tile
        // costs at most 32 KB and turns scattered few-entry updates (BBD ports
        // into a dense border) into one DMMA tile instead of CSC column sweeps
        if (static_cast<double>(nzb) >= tau * rect || rect <= RECT_SMALL) {
          if (static_cast<int>(R.size()) == d.nrows && static_cast<int>(Cc.size()) == d.ncols) {
            store = STORE_FULL;
          } else {
            store = STORE_RECT;
            Rl[b] = std::move(R);
            Cl[b] = std::move(Cc);
          }
        }
      }
      d.store = store;
      if (store == STORE_FULL) {
        d.nR = d.nrows;
        d.nC = d.ncols;
      } else if (store == STORE_RECT) {
        d.nR = static_cast<int32_t>(Rl[b].size());
        d.nC = static_cast<int32_t>(Cl[b].size());
      }
      d.cp = ncp;
      d.ent = nnz_w;
      c->wlen[b] = !resident[b] ? 0 : store == STORE_SPARSE ? nzb : static_cast<int64_t>(d.nR) * d.nC;
      ncp += d.ncols + 1;
      nnz_w += c->wlen[b];
      c->store_count[store]++;
    }
    c->nnz = nnz;
    c->nout = nnz;
    c->nnz_work = nnz_w;
    // ---- working CSC view, orig -> work map, R/C lists, CSR for sparse blocks ------
    std::vector<int32_t> hcp(ncp), hrows(nnz_w);
    std::vector<int64_t> hmap(nnz);
    std::vector<int32_t> hrl, hcl, hrp, hcc, hcpos;
    std::vector<int32_t> hdcsc, hdcsr, hlvc, hlvp;
    int64_t ndiag = 0;
    for (int64_t b = 0; b < nb; ++b) {
      BlockDev& d = hb[b];
      const int64_t* scp = colptr + T_cp[b];
      const int64_t* sri = rowidx + T_ent[b];
      const int64_t nzb = T_nz[b];
      const int64_t eo = T_ent[b];  // index into the reference pool (A values, factor output)
      int32_t* cp = &hcp[d.cp];
      const bool res = resident[b];
      if (!res)
        for (int64_t e = 0; e < nzb; ++e) hmap[eo + e] = -2;  // no storage on this rank
      if (d.store == STORE_SPARSE) {
        for (int k = 0; k <= d.ncols; ++k) cp[k] = static_cast<int32_t>(scp[k]);
        for (int64_t e = 0; res && e < nzb; ++e) {
          hrows[d.ent + e] = static_cast<int32_t>(sri[e]);
          hmap[eo + e] = d.ent + e;
        }
        // CSR transpose (rows ascending, columns ascending within a row)
        d.rp = static_cast<int64_t>(hrp.size());
        d.csr = static_cast<int64_t>(hcc.size());
        hrp.resize(hrp.size() + d.nrows + 1, 0);
        hcc.resize(hcc.size() + nzb);
        hcpos.resize(hcpos.size() + nzb);
        int32_t* rp = &hrp[d.rp];
        for (int64_t e = 0; e < nzb; ++e) rp[sri[e] + 1]++;
        for (int r = 0; r < d.nrows; ++r) rp[r + 1] += rp[r];
        std::vector<int32_t> w(rp, rp + d.nrows);
        for (int col = 0; col < d.ncols; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e) {
            const int32_t g = w[sri[e]]++;
            hcc[d.csr + g] = col;
            hcpos[d.csr + g] = static_cast<int32_t>(e);
          }
      } else if (d.store == STORE_FULL) {
        for (int k = 0; k <= d.ncols; ++k) cp[k] = k * d.nrows;
        for (int col = 0; res && col < d.ncols; ++col)
          for (int r = 0; r < d.nrows; ++r) hrows[d.ent + static_cast<int64_t>(col) * d.nrows + r] = r;
        for (int col = 0; res && col < d.ncols; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
            hmap[eo + e] = d.ent + static_cast<int64_t>(col) * d.nrows + sri[e];
      } else {
        const std::vector<int32_t>& R = Rl[b];
        const std::vector<int32_t>& Cc = Cl[b];
        d.roff = static_cast<int64_t>(hrl.size());
        d.coff = static_cast<int64_t>(hcl.size());
        hrl.insert(hrl.end(), R.begin(), R.end());
        hcl.insert(hcl.end(), Cc.begin(), Cc.end());
        std::vector<int32_t> rpos(d.nrows, -1), cpos(d.ncols, -1);
        for (int a = 0; a < d.nR; ++a) rpos[R[a]] = a;
        for (int a = 0; a < d.nC; ++a) cpos[Cc[a]] = a;
        int32_t acc = 0;
        for (int col = 0; col < d.ncols; ++col) {
          cp[col] = acc;
          if (cpos[col] >= 0) {
            for (int a = 0; res && a < d.nR; ++a) hrows[d.ent + acc + a] = R[a];
            acc += d.nR;
          }
        }
        cp[d.ncols] = acc;
        for (int col = 0; res && col < d.ncols; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
            hmap[eo + e] = d.ent + static_cast<int64_t>(cpos[col]) * d.nR + rpos[sri[e]];
      }
      if (T_bi[b] == T_bj[b]) {
        // row extent of every 64-column chunk of the diagonal block's pattern
        // (the device solve only touches rows the chunk can reach)
        {
          const int nch = (d.ncols + 63) / 64;
          c->dext_off[b] = static_cast<int64_t>(c->dext.size());
          std::vector<int32_t> hi(nch, 0), lo(nch, d.nrows);
          for (int col = 0; col < d.ncols; ++col)
            for (int64_t e = scp[col]; e < scp[col + 1]; ++e) {
              const int r = static_cast<int>(sri[e]), ch = col / 64;
              hi[ch] = std::max(hi[ch], r + 1);
              lo[ch] = std::min(lo[ch], r);
            }
          for (int ch = 0; ch < nch; ++ch) {
            c->dext.push_back(hi[ch]);
            c->dext.push_back(lo[ch]);
          }
        }
        d.dg = ndiag;
        ndiag += d.nrows;
        if (d.store == STORE_SPARSE) {
          // sparse diagonal block (all-sparse mode): diagonal positions + column levels
          const int64_t base = static_cast<int64_t>(hdcsc.size());
          if (base != d.dg) {
            hdcsc.resize(d.dg, -1);
            hdcsr.resize(d.dg, -1);
          }
          hdcsc.resize(d.dg + d.ncols, -1);
          hdcsr.resize(d.dg + d.nrows, -1);
          for (int col = 0; col < d.ncols; ++col)
            for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
              if (sri[e] == col) hdcsc[d.dg + col] = static_cast<int32_t>(e);
          const int32_t* rp = &hrp[d.rp];
          for (int r = 0; r < d.nrows; ++r)
            for (int32_t g = rp[r]; g < rp[r + 1]; ++g)
              if (hcc[d.csr + g] == r) hdcsr[d.dg + r] = g;
          for (int col = 0; col < d.ncols; ++col)
            if (hdcsc[d.dg + col] < 0 || hdcsr[d.dg + col] < 0)
              return fail(st, LBK_ERR_DIM_MISMATCH, "diagonal block without full diagonal");
          std::vector<int32_t> lev(d.ncols, 0);
          int32_t nlev = 0;
          for (int col = 0; col < d.ncols; ++col) {
            int32_t lv = 0;
            for (int64_t e = scp[col]; e < scp[col + 1] && sri[e] < col; ++e) lv = std::max(lv, lev[sri[e]] + 1);
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
      }
    }
    hdcsc.resize(ndiag, -1);
    hdcsr.resize(ndiag, -1);
    c->ndiag_rows = ndiag;
    auto rows_of = [&](int64_t b) {
      const BlockDev& d = hb[b];
      if (d.store == STORE_RECT) return Rl[b];
      std::vector<int32_t> v(d.nrows);
      for (int r = 0; r < d.nrows; ++r) v[r] = r;
      return v;
    };
    auto cols_of = [&](int64_t b) {
      const BlockDev& d = hb[b];
      if (d.store == STORE_RECT) return Cl[b];
      std::vector<int32_t> v(d.ncols);
      for (int r = 0; r < d.ncols; ++r) v[r] = r;
      return v;
    };
    // ---- banded diagonal blocks: independent segments --------------------------------
    // A FULL diagonal block whose filled pattern lies in a band <= BAND_MAX is swept
    // segment by segment (X_BAND); a segment boundary at s when no entry couples
    // [.., s) with [s, ..) (block-diagonal bodies inside one block), segments >= 64.
    struct BandInfo {
      int bl = 0, bu = 0;
      std::vector<std::pair<int32_t, int32_t>> seg;  // [s0, s1)
      std::vector<int32_t> segof;                    // local index -> segment
      std::vector<int32_t> lev;                      // refined launch level of each segment
    };
    std::map<int64_t, BandInfo> band;
    if (!all_full && dense_on && c->use_exec)
      for (int64_t b = 0; b < nb; ++b) {
        const int m = static_cast<int>(T_nr[b]);
        if (T_bi[b] != T_bj[b] || hb[b].store != STORE_FULL || m <= 2 * XT || m > 32767) continue;
        int bl = 0, bu = 0;
        const int64_t* scp = colptr + T_cp[b];
        const int64_t* sri = rowidx + T_ent[b];
        for (int col = 0; col < m; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e) {
            const int r = static_cast<int>(sri[e]);
            bl = std::max(bl, r - col);
            bu = std::max(bu, col - r);
          }
        if (bl > BAND_MAX || bu > BAND_MAX) continue;
        BandInfo bi;
        bi.bl = bl;
        bi.bu = bu;
        std::vector<int> lo(m, m);  // lowest row/col index coupled to index x from the other side
        for (int col = 0; col < m; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e) {
            const int r = static_cast<int>(sri[e]);
            lo[std::max(r, col)] = std::min(lo[std::max(r, col)], std::min(r, col));
          }
        std::vector<int> sufmin(m + 1, m);
        for (int x = m - 1; x >= 0; --x) sufmin[x] = std::min(sufmin[x + 1], lo[x]);
        bi.segof.assign(m, 0);
        int s0 = 0;
        for (int s1 = 1; s1 <= m; ++s1)
          if (s1 == m || (sufmin[s1] >= s1 && s1 - s0 >= 64)) {
            for (int x = s0; x < s1; ++x) bi.segof[x] = static_cast<int32_t>(bi.seg.size());
            bi.seg.push_back({s0, s1});
            s0 = s1;
          }
        bi.lev.assign(bi.seg.size(), -1);
        band.emplace(b, std::move(bi));
      }
    c->band_bl.assign(nb, -1);
    c->band_bu.assign(nb, -1);
    c->band_off.assign(nb, -1);
    c->band_seg.clear();
    for (const auto& kv : band) {
      c->band_bl[kv.first] = kv.second.bl;
      c->band_bu[kv.first] = kv.second.bu;
      c->band_off[kv.first] = static_cast<int64_t>(c->band_seg.size());
      for (const auto& sg : kv.second.seg) {
        c->band_seg.push_back(sg.first);
        c->band_seg.push_back(sg.second);
      }
    }
    // ---- refined ASAP levels ----------------------------------------------------------
    // The reference's DAG (grid.py:223-378) orders whole blocks.  Inside a banded
    // diagonal block the segments are independent sub-LUs, so: an update into the block
    // waits only for the last update into the segments its product rows reach, each
    // segment's sweep only for those updates, and a panel (GESSM / TSTRF) only for the
    // segments its rows / columns read.  Every per-entry operation order is unchanged
    // (the ascending-step chain is kept per segment), so the factors are bitwise the same;
    // the chain of coupled band blocks of a bordered-block-diagonal matrix falls apart into
    // short per-body chains.  Off for distributed plans (their cuts follow tree levels),
    // static pivoting (the exact single-CTA GETRF factors whole blocks) and the tile path.
    const bool refine = (flags & 4) != 0 && c->mask.empty() && c->use_exec && !all_full && !band.empty() &&
                        std::getenv("LBK_NO_REFINE") == nullptr;
    std::vector<int32_t> rlev(tlevels, tlevels + ntasks);
    std::vector<int8_t> rdefer;
    c->refined = refine;
    if (refine) {
      constexpr int32_t NONE = std::numeric_limits<int32_t>::max();
      std::vector<int32_t> lastlv(nb, -1), lastid(nb, -1), minsucc(ntasks, NONE);
      std::map<int64_t, std::vector<int32_t>> slastlv, slastid;
      for (auto& kv : band) {
        slastlv[kv.first].assign(kv.second.seg.size(), -1);
        slastid[kv.first].assign(kv.second.seg.size(), -1);
      }
      std::vector<int32_t> getrf_of(p, -1), gessm_of(p, -1), tstrf_of(p, -1);
      auto pred = [&](int32_t& lvl, int32_t plv, int32_t pid, std::vector<int32_t>& ps) {
        lvl = std::max(lvl, plv + 1);
        if (pid >= 0) ps.push_back(pid);
      };
      // segments of band block d reached by the rows (rows = true) / columns of block x
      auto segs_of = [&](int64_t d, int64_t x, bool rows_dim) {
        const BandInfo& bi = band.at(d);
        std::vector<char> hit(bi.seg.size(), 0);
        const int64_t* scp = colptr + T_cp[x];
        const int64_t* sri = rowidx + T_ent[x];
        if (rows_dim) {
          for (int64_t e = 0; e < T_nz[x]; ++e) hit[bi.segof[sri[e]]] = 1;
        } else {
          for (int col = 0; col < T_nc[x]; ++col)
            if (scp[col + 1] > scp[col]) hit[bi.segof[col]] = 1;
        }
        return hit;
      };
      std::vector<int32_t> ps;
      for (int64_t t = 0; t < ntasks; ++t) {
        const int kind = kinds[t];
        const int64_t i = steps[t], r = trows[t], cc = tcols[t];
        const int64_t d = bid[i * p + i];
        const bool dband = band.count(d) != 0;
        int32_t lvl = 0;
        ps.clear();
        if (kind == KIND_GETRF) {
          getrf_of[i] = static_cast<int32_t>(t);
          if (dband) {
            BandInfo& bi = band.at(d);
            auto& sl = slastlv[d];
            auto& si = slastid[d];
            for (size_t q = 0; q < bi.seg.size(); ++q) {
              bi.lev[q] = sl[q] + 1;
              if (si[q] >= 0) minsucc[si[q]] = std::min(minsucc[si[q]], bi.lev[q]);
              lvl = std::max(lvl, bi.lev[q]);
            }
          } else {
            pred(lvl, lastlv[d], lastid[d], ps);
          }
        } else if (kind == KIND_GESSM || kind == KIND_TSTRF) {
          const int64_t x = kind == KIND_GESSM ? bid[i * p + cc] : bid[r * p + i];
          if (kind == KIND_GESSM) gessm_of[cc] = static_cast<int32_t>(t);
          else tstrf_of[r] = static_cast<int32_t>(t);
          if (dband) {
            const std::vector<char> hit = segs_of(d, x, kind == KIND_GESSM);
            const BandInfo& bi = band.at(d);
            for (size_t q = 0; q < hit.size(); ++q)
              if (hit[q]) lvl = std::max(lvl, bi.lev[q] + 1);
          } else {
            lvl = std::max(lvl, rlev[getrf_of[i]] + 1);
          }
          pred(lvl, lastlv[x], lastid[x], ps);
        } else {  // SSSSM(r, cc, i)
          const int64_t tgt = bid[r * p + cc];
          if (tgt < 0 || costs[t] == 0) {  // skipped at run time (zero work): not a writer
            rlev[t] = 0;
            continue;
          }
          lvl = std::max(rlev[tstrf_of[r]], rlev[gessm_of[cc]]) + 1;
          if (band.count(tgt)) {
            const std::vector<char> hit = segs_of(tgt, bid[r * p + i], true);  // product rows = L's rows
            auto& sl = slastlv[tgt];
            auto& si = slastid[tgt];
            for (size_t q = 0; q < hit.size(); ++q)
              if (hit[q]) pred(lvl, sl[q], si[q], ps);
            for (int32_t pid : ps) minsucc[pid] = std::min(minsucc[pid], lvl);
            for (size_t q = 0; q < hit.size(); ++q)
              if (hit[q]) {
                sl[q] = lvl;
                si[q] = static_cast<int32_t>(t);
              }
            rlev[t] = lvl;
            continue;
          }
          pred(lvl, lastlv[tgt], lastid[tgt], ps);
          lastlv[tgt] = lvl;
          for (int32_t pid : ps) minsucc[pid] = std::min(minsucc[pid], lvl);
          lastid[tgt] = static_cast<int32_t>(t);
          rlev[t] = lvl;
          continue;
        }
        for (int32_t pid : ps) minsucc[pid] = std::min(minsucc[pid], lvl);
        rlev[t] = lvl;
      }
      // lookahead slack of the updates under the refined levels (numeric.defer_flags semantics)
      rdefer.assign(ntasks, 0);
      for (int64_t t = 0; t < ntasks; ++t)
        if (kinds[t] == KIND_SSSSM && minsucc[t] != NONE)
          rdefer[t] = static_cast<int8_t>(std::clamp(minsucc[t] - rlev[t], 0, 100));
    }
    const int32_t* tlev = rlev.data();
    if (refine)  // the level after which each block is final (streamed output)
      for (int64_t t = 0; t < ntasks; ++t) {
        const int64_t i = steps[t];
        int64_t fb = -1;
        if (kinds[t] == KIND_GETRF) fb = bid[i * p + i];
        else if (kinds[t] == KIND_GESSM) fb = bid[i * p + tcols[t]];
        else if (kinds[t] == KIND_TSTRF) fb = bid[trows[t] * p + i];
        if (fb >= 0) c->blk_final_tl[fb] = tlev[t];
      }
    // ---- per-level work lists ------------------------------------------------------
    int32_t nlevels = 0;
    for (int64_t t = 0; t < ntasks; ++t) nlevels = std::max(nlevels, tlev[t] + 1);
    for (auto& kv : band)
      for (int32_t l : kv.second.lev) nlevels = std::max(nlevels, l + 1);
    std::vector<std::vector<Item>> gen(nlevels);
    std::vector<int32_t> acc_len(nlevels, 1);
    std::vector<std::vector<GemmItem>> gem(nlevels), gemD(nlevels), gemE(nlevels);
    std::vector<GemmTask> gtasks;
    std::vector<int64_t> gtask_t;  // tree task of each GemmTask
    std::vector<int32_t> hmaps;
    std::vector<std::vector<DenseItem>> pan(nlevels), exa(nlevels);
    std::vector<std::vector<std::array<int32_t, 4>>> ptask(nlevels);  // (kind, diag blk, panel blk, step)
    std::vector<int32_t> pan_smem(nlevels, 0), exa_smem(nlevels, 0);
    std::vector<std::vector<int64_t>> tgetrf(nlevels);  // FULL diagonal blocks factored by the tiled GETRF
    c->route.assign(ntasks, -1);
    // items of min(chunk, warps) NONEMPTY columns/rows each (the kernels skip empty ones
    // in a few instructions; a CTA per 8 positions of a 2000-wide, 2%-occupied
    // panel would launch 250 CTAs with 64 KB accumulators for nothing)
    // materialized after the task loop, when the level's warps per CTA are
    // known: one nonempty column/row per warp and item
    struct PendingRange {
      int32_t lv;
      Item base;
      int32_t count;
      std::vector<char> nonempty;
    };
    std::vector<PendingRange> pending_ranges;
    auto add_range = [&](int32_t lv, Item base, int32_t count, std::vector<char> nonempty) {
      pending_ranges.push_back(PendingRange{lv, base, count, std::move(nonempty)});
    };
    auto emit_range = [&](int32_t lv, Item base, int32_t count, const std::vector<char>& nonempty,
                          int32_t chunk_nz) {
      int32_t s = 0, have = 0;
      for (int32_t x = 0; x < count; ++x) {
        if (!nonempty[x]) {
          if (have == 0) s = x + 1;
          continue;
        }
        if (++have == chunk_nz) {
          Item it = base;
          it.begin = s;
          it.end = x + 1;
          gen[lv].push_back(it);
          s = x + 1;
          have = 0;
        }
      }
      if (have) {
        Item it = base;
        it.begin = s;
        it.end = count;
        gen[lv].push_back(it);
      }
    };
    auto col_nonempty = [&](int64_t b) {
      std::vector<char> v(hb[b].ncols, 0);
      const int64_t* scp = colptr + T_cp[b];
      for (int x = 0; x < hb[b].ncols; ++x) v[x] = scp[x + 1] > scp[x];
      return v;
    };
    auto row_nonempty = [&](int64_t b) {
      std::vector<char> v(hb[b].nrows, 0);
      const int64_t* sri = rowidx + T_ent[b];
      for (int64_t e = 0; e < T_nz[b]; ++e) v[sri[e]] = 1;
      return v;
    };
    auto tile_like = [&](int64_t b) { return hb[b].store != STORE_SPARSE; };
    // pattern occupancy of a FULL/RECT block in its stored (compressed) coordinates:
    // lmask[c] = 128-row tiles holding entries of stored column c (as an SSSSM L operand),
    // umask[r] = 64-column tiles holding entries of stored row r (as a U operand)
    std::map<int64_t, std::vector<uint64_t>> lmask_c, umask_c;
    std::vector<int32_t> hkch;
    auto stored_pos = [&](int64_t b, bool rows_dim) {
      const BlockDev& d = hb[b];
      const int n = rows_dim ? d.nrows : d.ncols;
      std::vector<int32_t> pos(n);
      if (d.store == STORE_RECT) {
        std::fill(pos.begin(), pos.end(), -1);
        const std::vector<int32_t>& lst = rows_dim ? Rl[b] : Cl[b];
        for (size_t q = 0; q < lst.size(); ++q) pos[lst[q]] = static_cast<int32_t>(q);
      } else {
        for (int q = 0; q < n; ++q) pos[q] = q;
      }
      return pos;
    };
    auto lmask = [&](int64_t b) -> const std::vector<uint64_t>& {
      auto it = lmask_c.find(b);
      if (it != lmask_c.end()) return it->second;
      std::vector<uint64_t> m(hb[b].nC, 0);
      const std::vector<int32_t> rp = stored_pos(b, true), cpn = stored_pos(b, false);
      const int64_t* scp = colptr + T_cp[b];
      const int64_t* sri = rowidx + T_ent[b];
      for (int col = 0; col < hb[b].ncols; ++col)
        for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
          m[cpn[col]] |= 1ull << std::min(rp[sri[e]] / GBM, 63);
      return lmask_c.emplace(b, std::move(m)).first->second;
    };
    auto umask = [&](int64_t b) -> const std::vector<uint64_t>& {
      auto it = umask_c.find(b);
      if (it != umask_c.end()) return it->second;
      std::vector<uint64_t> m(hb[b].nR, 0);
      const std::vector<int32_t> rp = stored_pos(b, true), cpn = stored_pos(b, false);
      const int64_t* scp = colptr + T_cp[b];
      const int64_t* sri = rowidx + T_ent[b];
      for (int col = 0; col < hb[b].ncols; ++col)
        for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
          m[rp[sri[e]]] |= 1ull << std::min(cpn[col] / GBN, 63);
      return umask_c.emplace(b, std::move(m)).first->second;
    };
    for (int64_t t = 0; t < ntasks; ++t) {
      if (!c->mask.empty() && !c->mask[t]) continue;  // another rank's task (owner-computes)
      const int kind = kinds[t];
      const int64_t i = steps[t], r = trows[t], cc = tcols[t];
      const int32_t lv = tlev[t];
      const int64_t dblk = bid[i * p + i];
      Item it{};
      it.kind = kind;
      if (kind == KIND_GETRF) {
        if (hb[dblk].store == STORE_FULL) {
          // tiled multi-CTA GETRF (no-swap speculation, verified); the exact
          // single-CTA variant is kept for dense-scratch / static pivoting.
          // Refined band blocks: listed at every level holding one of their segments.
          if (refine && band.count(dblk)) {
            std::vector<int32_t> ls = band.at(dblk).lev;
            std::sort(ls.begin(), ls.end());
            ls.erase(std::unique(ls.begin(), ls.end()), ls.end());
            for (int32_t l : ls) tgetrf[l].push_back(dblk);
          } else {
            tgetrf[lv].push_back(dblk);
          }
          c->route[t] = 3;
          DenseItem d{0, static_cast<int32_t>(dblk), static_cast<int32_t>(i), all_full ? 1 : 0, 0,
                      static_cast<int32_t>(i)};
          exa[lv].push_back(d);
          exa_smem[lv] = std::max(exa_smem[lv], (hb[dblk].nrows + 64) * 8);
        } else {
          it.a = static_cast<int32_t>(dblk);
          it.b = static_cast<int32_t>(i);
          c->route[t] = 0;
          it.begin = 0;
          it.end = 1;
          gen[lv].push_back(it);
          acc_len[lv] = std::max(acc_len[lv], hb[dblk].nrows);
        }
      } else if (kind == KIND_GESSM) {
        const int64_t x = bid[i * p + cc];
        it.a = static_cast<int32_t>(dblk);
        it.b = static_cast<int32_t>(x);
        it.c = all_full ? 1 : 0;  // row permutation of FULL panels (dense-scratch mode)
        if (hb[dblk].store == STORE_FULL && tile_like(x)) {
          c->route[t] = 2;
          for (int32_t s = 0; s < hb[x].nC; s += STRIP)
            pan[lv].push_back(DenseItem{1, it.a, it.b, it.c, s, static_cast<int32_t>(i)});
          ptask[lv].push_back({1, it.a, it.b, static_cast<int32_t>(i)});
          pan_smem[lv] = std::max(pan_smem[lv], (hb[x].nR + 64) * 8);
          continue;
        }
        acc_len[lv] = std::max(acc_len[lv], hb[x].nrows);
        c->route[t] = 0;
        add_range(lv, it, hb[x].ncols, col_nonempty(x));
      } else if (kind == KIND_TSTRF) {
        const int64_t x = bid[r * p + i];
        it.a = static_cast<int32_t>(dblk);
        it.b = static_cast<int32_t>(x);
        if (hb[dblk].store == STORE_FULL && tile_like(x)) {
          c->route[t] = 2;
          for (int32_t s = 0; s < hb[x].nR; s += STRIP)
            pan[lv].push_back(DenseItem{2, it.a, it.b, 0, s, static_cast<int32_t>(i)});
          ptask[lv].push_back({2, it.a, it.b, static_cast<int32_t>(i)});
          pan_smem[lv] = std::max(pan_smem[lv], 64 * 8);
          continue;
        }
        if (hb[x].store != STORE_SPARSE || (hb[dblk].store == STORE_SPARSE && hb[dblk].rp < 0))
          return fail(st, LBK_ERR_BAD_ARG, "TSTRF operand without a CSR index");
        acc_len[lv] = std::max(acc_len[lv], hb[x].ncols);
        c->route[t] = 0;
        add_range(lv, it, hb[x].nrows, row_nonempty(x));
      } else {
        const int64_t tgt = bid[r * p + cc];
        if (tgt < 0) {
          if (costs[t] > 0) return fail(st, LBK_ERR_SUPPORT, "update hits an empty block");
          continue;  // zero-work update into an absent block (grid.py:332-362)
        }
        if (costs[t] == 0) continue;  // structurally empty product
        const int64_t lb = bid[r * p + i], ub = bid[i * p + cc];
        it.a = static_cast<int32_t>(lb);
        it.b = static_cast<int32_t>(ub);
        it.c = static_cast<int32_t>(tgt);
        if (tile_like(lb) && tile_like(ub) && tile_like(tgt)) {
          const std::vector<int32_t> RL = rows_of(lb), CL = cols_of(lb), RU = rows_of(ub), CU = cols_of(ub),
                                     RC = rows_of(tgt), CC = cols_of(tgt);
          // inner index: intersection of L's columns and U's rows
          std::vector<int32_t> kl, ku;
          size_t a = 0, bb = 0;
          while (a < CL.size() && bb < RU.size()) {
            if (CL[a] == RU[bb]) {
              kl.push_back(static_cast<int32_t>(a));
              ku.push_back(static_cast<int32_t>(bb));
              ++a;
              ++bb;
            } else if (CL[a] < RU[bb]) {
              ++a;
            } else {
              ++bb;
            }
          }
          if (kl.empty()) continue;
          GemmTask gt{};
          gt.a = it.a;
          gt.b = it.b;
          gt.c = it.c;
          gt.K = static_cast<int32_t>(kl.size());
          const bool kid = kl.size() == CL.size() && ku.size() == RU.size();
          gt.kL = gt.kU = -1;
          if (!kid) {
            gt.kL = static_cast<int64_t>(hmaps.size());
            hmaps.insert(hmaps.end(), kl.begin(), kl.end());
            gt.kU = static_cast<int64_t>(hmaps.size());
            hmaps.insert(hmaps.end(), ku.begin(), ku.end());
          }
          bool rid = false, cid = false;
          std::vector<int32_t> rm = positions_in(RL, RC, &rid), cm = positions_in(CU, CC, &cid);
          gt.rmap = gt.cmap = -1;
          if (!rid) {
            gt.rmap = static_cast<int64_t>(hmaps.size());
            hmaps.insert(hmaps.end(), rm.begin(), rm.end());
          }
          if (!cid) {
            gt.cmap = static_cast<int64_t>(hmaps.size());
            hmaps.insert(hmaps.end(), cm.begin(), cm.end());
          }
          const int32_t task = static_cast<int32_t>(gtasks.size());
          c->route[t] = 1;
          gtasks.push_back(gt);
          gtask_t.push_back(t);
          const int slack = refine ? rdefer[t] : c->defer.empty() ? 0 : c->defer[t];
          auto& dst = slack >= 3 ? gemE[lv] : slack == 2 ? gemD[lv] : gem[lv];
          // k-chunk skipping: per GBK-chunk of the inner index, the 128-row tiles of L and the
          // 64-column tiles of U holding pattern entries (bit per tile, saturating at 63)
          // (dense-scratch mode: row swaps move the support, so every chunk runs)
          const int nkch = (gt.K + GBK - 1) / GBK;
          std::vector<uint64_t> chL(nkch, ~0ull), chU(nkch, ~0ull);
          if (!all_full) {
            const std::vector<uint64_t>& lm = lmask(lb);
            const std::vector<uint64_t>& um = umask(ub);
            std::fill(chL.begin(), chL.end(), 0);
            std::fill(chU.begin(), chU.end(), 0);
            for (int32_t k = 0; k < gt.K; ++k) {
              chL[k / GBK] |= lm[kid ? k : kl[k]];
              chU[k / GBK] |= um[kid ? k : ku[k]];
            }
          }
          std::vector<int32_t> act;
          for (int32_t n0 = 0; n0 < hb[ub].nC; n0 += GBN)
            for (int32_t m0 = 0; m0 < hb[lb].nR; m0 += GBM) {
              const uint64_t bm = 1ull << std::min(m0 / GBM, 63), bn = 1ull << std::min(n0 / GBN, 63);
              act.clear();
              int64_t klen = 0;
              for (int q = 0; q < nkch; ++q)
                if ((chL[q] & bm) && (chU[q] & bn)) {
                  act.push_back(q);
                  klen += std::min(GBK, gt.K - q * GBK);
                }
              if (act.empty()) continue;  // the tile's product is structurally zero
              GemmItem gi{task, m0, n0, -1, 0, 0, nkch, -1, 0};
              if (static_cast<int>(act.size()) < nkch) {
                gi.nkc = static_cast<int32_t>(act.size());
                gi.kc_off = static_cast<int64_t>(hkch.size());
                gi.ke = gi.nkc;
                hkch.insert(hkch.end(), act.begin(), act.end());
              }
              dst.push_back(gi);
              c->dmma_flops += 2.0 * std::min(GBM, hb[lb].nR - m0) * static_cast<double>(klen) *
                               std::min(GBN, hb[ub].nC - n0);
            }
          continue;
        }
        acc_len[lv] = std::max(acc_len[lv], hb[tgt].nrows);
        c->route[t] = 0;
        add_range(lv, it, hb[tgt].ncols, col_nonempty(ub));
      }
    }
    for (const PendingRange& pr : pending_ranges)
      emit_range(pr.lv, pr.base, pr.count, pr.nonempty, std::min(chunk, choose_warps(acc_len[pr.lv])));
    pending_ranges.clear();
    // ---- flatten ---------------------------------------------------------------------
    std::vector<Item> gall;
    std::vector<GemmItem> mall;
    int64_t max_ws_slots = 0;  // split-K workspace slots (levels run one after another)
    std::vector<DenseItem> dall;
    std::vector<TileItem> tall;
    std::vector<XTask> xtasks;
    std::vector<int32_t> xsucc_ptr, xsucc, xdeps0;
    std::vector<int32_t> hxtb;            // executor tile boundaries (BlockDev::xtb1)
    std::map<int64_t, int64_t> xtb_of;
    // executor tiling of a diagonal block: subtree-aligned boundaries + subtree-cut region
    // per column (uniform 64 columns / one region in dense-scratch mode or LBK_UNIFORM_TILES)
    struct DiagTiling {
      std::vector<int32_t> tb, seg;
    };
    std::map<int64_t, DiagTiling> dtiling;
    auto diag_tiling = [&](int64_t b) -> const DiagTiling& {
      auto it = dtiling.find(b);
      if (it != dtiling.end()) return it->second;
      DiagTiling& t = dtiling[b];
      const int m = hb[b].nrows;
      if (all_full || std::getenv("LBK_UNIFORM_TILES")) {
        for (int x = 0; x < m; x += XT) t.tb.push_back(x);
        t.tb.push_back(m);
        t.seg.assign(m, 0);
      } else {
        const int64_t* bcp = colptr + T_cp[b];
        const int64_t* bri = rowidx + T_ent[b];
        // candidates: uniform 64-column tiles and subtree-aligned tiles with a minimum width
        // before a cut of 1 / 8 / 16 / 32 columns; the one with the shortest modelled chain
        // wins (uniform unless an aligned one is >= 5 % shorter and not fragmented)
        for (int x = 0; x < m; x += XT) t.tb.push_back(x);
        t.tb.push_back(m);
        t.seg.assign(m, 0);
        double best = 0.95 * tile_cp_model(m, bcp, bri, t.tb);
        const size_t max_tiles = t.tb.size() * 3 / 2 + 1;
        for (int minw : {1, 8, 16, 32}) {
          std::vector<int32_t> sg;
          std::vector<int32_t> tb = subtree_tiles(m, bcp, bri, XT, minw, &sg);
          if (tb.size() > max_tiles) continue;
          const double cpm = tile_cp_model(m, bcp, bri, tb);
          if (cpm < best) {
            best = cpm;
            t.tb.swap(tb);
            t.seg.swap(sg);
          }
        }
      }
      return t;
    };
    c->levels.clear();
    c->subs.clear();
    // A GETRF-only level followed by a panel-only level run in ONE executor
    // launch: each panel tile waits only for the tile columns (GESSM) / rows
    // (TSTRF) of the diagonal factor it reads, so the panel substitution
    // chains trail the GETRF chain instead of starting after it.
    auto only_exec = [&](int32_t l) {
      return gen[l].empty() && gem[l].empty() && gemD[l].empty() && gemE[l].empty();
    };
    std::vector<char> merged_into_prev(nlevels, 0);
    const bool chain_l = std::getenv("LBK_CHAIN_L") != nullptr;  // chain-2 GETRF tasks (A/B)
    const int panel_agg = std::getenv("LBK_PANEL_AGG") ? std::max(1, std::atoi(std::getenv("LBK_PANEL_AGG"))) : 4;
    int32_t absorbed_lv = -2;  // SSSSM level whose DMMA tiles run inside the next executor launch
    int64_t absorbed_off = 0, absorbed_n = 0;
    for (int32_t lv = 0; lv < nlevels; ++lv) {
      if (gen[lv].empty() && gem[lv].empty() && gemD[lv].empty() && gemE[lv].empty() && pan[lv].empty() &&
          exa[lv].empty())
        continue;
      const bool merge_next = c->use_exec && !all_full && lv + 1 < nlevels && only_exec(lv) && only_exec(lv + 1) &&
                              !tgetrf[lv].empty() && ptask[lv].empty() && tgetrf[lv + 1].empty() &&
                              !ptask[lv + 1].empty() &&
                              (c->cut_after.empty() || !c->cut_after[lv]) && std::getenv("LBK_NO_MERGE") == nullptr;
      if (static_cast<int64_t>(acc_len[lv]) * 8 > MAX_SMEM || pan_smem[lv] > MAX_SMEM || exa_smem[lv] > MAX_SMEM)
        return fail(st, LBK_ERR_BAD_ARG, "block span too large for the shared-memory accumulator");
      Level L{};
      L.tree_level = lv;
      L.tree_level_hi = merge_next ? lv + 1 : lv;
      L.item_off = static_cast<int64_t>(gall.size());
      L.nitems = static_cast<int32_t>(gen[lv].size());
      L.acc_len = acc_len[lv];
      L.warps = choose_warps(L.acc_len);
      gall.insert(gall.end(), gen[lv].begin(), gen[lv].end());
      if (gemD[lv].size() + gemE[lv].size() < DEFER_MIN_TILES) {  // not worth separate launches
        gem[lv].insert(gem[lv].end(), gemD[lv].begin(), gemD[lv].end());
        gem[lv].insert(gem[lv].end(), gemE[lv].begin(), gemE[lv].end());
        gemD[lv].clear();
        gemE[lv].clear();
      }
      // An SSSSM-only level followed by an executor-only GETRF level: its DMMA tiles become
      // executor tasks of the next launch (X_SSSSM), and only the tasks of that launch that
      // touch an updated block wait for them (the column tiles' COLMAX tasks of a diagonal
      // block, the first writes into a panel) - no launch barrier between the updates and
      // the next factorizations, and the executor's idle CTAs (its chains are latency-bound)
      // run the remaining updates.  Off for distributed plans (cuts at level boundaries),
      // dense-scratch plans and band launches.  Measured slower (C2 118.7 -> 119.9 ms, C5 7.04 ->
      // 7.27 ms, profiles/r2_absorb_ab.txt): the updates feeding the next diagonal block's
      // first column tiles are the longest tiles and outrank every chain task, so the chain
      // starts no earlier - kept as a variant (-DLBK_ABSORB_TILES=1 and LBK_ABSORB=1).
      auto no_band = [&](int32_t l) {
        for (int64_t b : tgetrf[l])
          if (band.count(b)) return false;
        return true;
      };
      const bool absorb = LBK_ABSORB_TILES && c->use_exec && !all_full && c->cut_after.empty() && std::getenv("LBK_ABSORB") &&
                          lv + 1 < nlevels && !gem[lv].empty() && gen[lv].empty() && exa[lv].empty() &&
                          tgetrf[lv].empty() && ptask[lv].empty() && !merged_into_prev[lv] &&
                          !tgetrf[lv + 1].empty() && gen[lv + 1].empty() && gem[lv + 1].empty() &&
                          gemD[lv + 1].empty() && gemE[lv + 1].empty() && no_band(lv + 1);
      if (absorb) {
        std::stable_sort(gem[lv].begin(), gem[lv].end(),
                         [&](const GemmItem& x, const GemmItem& y) { return x.ke - x.ks > y.ke - y.ks; });
        absorbed_lv = lv;
        absorbed_off = static_cast<int64_t>(mall.size());
        absorbed_n = static_cast<int64_t>(gem[lv].size());
        L.absorb_off = absorbed_off;
        L.nabsorb = static_cast<int32_t>(absorbed_n);
        mall.insert(mall.end(), gem[lv].begin(), gem[lv].end());
        for (const GemmItem& gi : gem[lv]) {
          const GemmTask& gt = gtasks[gi.task];
          c->route[gtask_t[gi.task]] = 3;
          const int64_t klen = gi.nkc < 0 ? gt.K : [&] {
            int64_t kl = 0;
            for (int q = 0; q < gi.nkc; ++q) kl += std::min(GBK, gt.K - hkch[gi.kc_off + q] * GBK);
            return kl;
          }();
          const double xf = 2.0 * std::min(GBM, hb[gt.a].nR - gi.m0) * static_cast<double>(klen) *
                            std::min(GBN, hb[gt.b].nC - gi.n0);
          c->dmma_flops -= xf;
          c->exec_flops += xf;
        }
        gem[lv].clear();
      }
      // longest tiles first (LPT): the block scheduler hands out CTAs in index order,
      // so the long inner loops start early and the level's tail is made of short tiles
      // (items write disjoint output tiles: the order does not touch the floating point)
      // split-K for a critical launch with too few tiles to fill the GPU: a tile with enough
      // inner chunks is cut into up to 8 parts writing partial products to a workspace, and
      // a reduction launch adds them in slot order (deterministic) and scatters into C
      std::vector<GemmItem> red;
      // Part length: the candidate (unsplit, or parts of about 1, 1/2, 1/4, 1/8 of the level's
      // mean chunks per CTA slot) whose greedy longest-first schedule over the 296 CTA slots
      // has the shortest makespan, a split tile paying one extra chunk for its reduction
      // (a level of 360 equal tiles otherwise runs as 1 full wave + a 22 % wave).
      // LBK_SPLITK_OLD: the round-2 rule (only launches under 592 tiles).
      int split_len = 0;  // 0: no split; else target chunks per part
      if (LBK_SPLITK && !gem[lv].empty() && !std::getenv("LBK_SPLITK_OLD")) {
        constexpr int SLOTS = 296;
        int64_t total = 0;
        for (const GemmItem& g0 : gem[lv]) total += g0.ke - g0.ks;
        auto makespan = [&](int len) {
          std::vector<int64_t> w;
          for (const GemmItem& g0 : gem[lv]) {
            const int nk = g0.ke - g0.ks;
            const int parts = len ? std::min(8, nk / std::max(len, SPLITK_MIN_CHUNKS)) : 1;
            if (parts < 2) {
              w.push_back(nk);
              continue;
            }
            for (int q = 0; q < parts; ++q) w.push_back((nk * (q + 1)) / parts - (nk * q) / parts + 1);
          }
          std::sort(w.begin(), w.end(), std::greater<int64_t>());
          std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> pq;
          for (int q = 0; q < SLOTS; ++q) pq.push(0);
          int64_t mk = 0;
          for (int64_t x : w) {
            const int64_t t0 = pq.top();
            pq.pop();
            pq.push(t0 + x);
            mk = std::max(mk, t0 + x);
          }
          return mk;
        };
        int64_t best = makespan(0);
        const int64_t mean = std::max<int64_t>(1, total / SLOTS);
        for (int64_t div : {1, 2, 4, 8}) {
          const int len = static_cast<int>(std::max<int64_t>(SPLITK_MIN_CHUNKS, mean / div));
          const int64_t mk = makespan(len);
          if (mk * 20 < best * 19) {  // >= 5 % shorter
            best = mk;
            split_len = len;
          }
        }
      }
      const bool old_rule = LBK_SPLITK && std::getenv("LBK_SPLITK_OLD") && !gem[lv].empty() &&
                            static_cast<int>(gem[lv].size()) < SPLITK_TILES;
      if (split_len > 0 || old_rule) {
        const int S = old_rule ? std::min(8, SPLITK_TILES / static_cast<int>(gem[lv].size())) : 8;
        std::vector<GemmItem> out;
        int32_t slots = 0;
        for (const GemmItem& g0 : gem[lv]) {
          const int nk = g0.ke - g0.ks;
          const int parts = old_rule ? std::min(S, nk / SPLITK_MIN_CHUNKS)
                                     : std::min(S, nk / std::max(split_len, SPLITK_MIN_CHUNKS));
          if (parts < 2) {
            out.push_back(g0);
            continue;
          }
          GemmItem r = g0;
          r.wslot = slots;
          r.nsplit = parts;
          red.push_back(r);
          for (int q = 0; q < parts; ++q) {
            GemmItem part = g0;
            part.ks = g0.ks + static_cast<int32_t>((static_cast<int64_t>(nk) * q) / parts);
            part.ke = g0.ks + static_cast<int32_t>((static_cast<int64_t>(nk) * (q + 1)) / parts);
            part.wslot = slots++;
            out.push_back(part);
          }
        }
        gem[lv].swap(out);
        max_ws_slots = std::max<int64_t>(max_ws_slots, slots);
      }
      for (auto* v : {&gem[lv], &gemD[lv], &gemE[lv]})
        std::stable_sort(v->begin(), v->end(),
                         [&](const GemmItem& x, const GemmItem& y) { return x.ke - x.ks > y.ke - y.ks; });
      L.gemm_off = static_cast<int64_t>(mall.size());
      L.ngemm = static_cast<int32_t>(gem[lv].size());
      mall.insert(mall.end(), gem[lv].begin(), gem[lv].end());
      L.gemmD_off = static_cast<int64_t>(mall.size());
      L.ngemmD = static_cast<int32_t>(gemD[lv].size());
      mall.insert(mall.end(), gemD[lv].begin(), gemD[lv].end());
      L.gemmE_off = static_cast<int64_t>(mall.size());
      L.ngemmE = static_cast<int32_t>(gemE[lv].size());
      mall.insert(mall.end(), gemE[lv].begin(), gemE[lv].end());
      L.gred_off = static_cast<int64_t>(mall.size());
      L.ngred = static_cast<int32_t>(red.size());
      mall.insert(mall.end(), red.begin(), red.end());
      L.panel_off = static_cast<int64_t>(dall.size());
      L.npanel = static_cast<int32_t>(pan[lv].size());
      L.panel_smem = pan_smem[lv];
      dall.insert(dall.end(), pan[lv].begin(), pan[lv].end());
      L.exact_off = static_cast<int64_t>(dall.size());
      L.nexact = static_cast<int32_t>(exa[lv].size());
      L.exact_smem = exa_smem[lv];
      dall.insert(dall.end(), exa[lv].begin(), exa[lv].end());
      // tiled GETRF work of this level
      L.tcol_off = static_cast<int64_t>(tall.size());
      int32_t maxm = 0;
      for (int64_t b : tgetrf[lv]) {
        const int m = hb[b].nrows;
        maxm = std::max(maxm, m);
        for (int c0 = 0; c0 < m; c0 += TS) {
          TileItem ti{};
          ti.blk = static_cast<int32_t>(b);
          ti.step = static_cast<int32_t>(T_bi[b]);
          ti.c0 = c0;
          tall.push_back(ti);
        }
      }
      L.ntcol = static_cast<int32_t>(tall.size() - L.tcol_off);
      L.sub_off = static_cast<int64_t>(c->subs.size());
      // tile occupancy of each diagonal block from its filled pattern: the
      // block's own LU fills only inside the (elimination-closed) pattern, so
      // structurally zero tiles never need a TRSM or a trailing update
      std::vector<std::vector<char>> occ(tgetrf[lv].size());
      for (size_t q = 0; q < tgetrf[lv].size(); ++q) {
        const int64_t b = tgetrf[lv][q];
        const int m = hb[b].nrows, nt = (m + TS - 1) / TS;
        occ[q].assign(static_cast<size_t>(nt) * nt, all_full ? 1 : 0);
        if (all_full) continue;
        const int64_t* scp = colptr + T_cp[b];
        const int64_t* sri = rowidx + T_ent[b];
        for (int col = 0; col < m; ++col)
          for (int64_t e = scp[col]; e < scp[col + 1]; ++e) occ[q][(col / TS) * nt + sri[e] / TS] = 1;
      }
      for (int kb = 0; kb < maxm; kb += TS) {
        SubStep s{};
        const int tk = kb / TS;
        s.getrf_off = static_cast<int64_t>(tall.size());
        for (int64_t b : tgetrf[lv])
          if (kb < hb[b].nrows) tall.push_back(TileItem{static_cast<int32_t>(b), static_cast<int32_t>(T_bi[b]), kb, 0, 0, 0});
        s.ngetrf = static_cast<int32_t>(tall.size() - s.getrf_off);
        s.trsm_off = static_cast<int64_t>(tall.size());
        for (size_t q = 0; q < tgetrf[lv].size(); ++q) {
          const int64_t b = tgetrf[lv][q];
          const int m = hb[b].nrows, nt = (m + TS - 1) / TS;
          if (kb >= m) continue;
          for (int o = kb + TS; o < m; o += TS) {
            const int to = o / TS;
            if (occ[q][tk * nt + to])  // L tile (o, kb): column tk, row to
              tall.push_back(TileItem{static_cast<int32_t>(b), static_cast<int32_t>(T_bi[b]), kb, o, 0, 0});
            if (occ[q][to * nt + tk])  // U tile (kb, o): column to, row tk
              tall.push_back(TileItem{static_cast<int32_t>(b), static_cast<int32_t>(T_bi[b]), kb, 0, o, 1});
          }
        }
        s.ntrsm = static_cast<int32_t>(tall.size() - s.trsm_off);
        s.gemm_off = static_cast<int64_t>(tall.size());
        for (size_t q = 0; q < tgetrf[lv].size(); ++q) {
          const int64_t b = tgetrf[lv][q];
          const int m = hb[b].nrows, nt = (m + TS - 1) / TS;
          if (kb >= m) continue;
          for (int c0 = kb + TS; c0 < m; c0 += TS) {
            if (!occ[q][(c0 / TS) * nt + tk]) continue;  // U tile (kb, c0) empty
            for (int r0 = kb + TS; r0 < m; r0 += TS)
              if (occ[q][tk * nt + r0 / TS])  // L tile (r0, kb)
                tall.push_back(TileItem{static_cast<int32_t>(b), static_cast<int32_t>(T_bi[b]), kb, r0, c0, 0});
          }
        }
        s.ngemm = static_cast<int32_t>(tall.size() - s.gemm_off);
        c->subs.push_back(s);
      }
      L.nsub = static_cast<int32_t>(c->subs.size() - L.sub_off);
      L.tfin_off = static_cast<int64_t>(tall.size());
      for (int64_t b : tgetrf[lv])
        for (int c0 = 0; c0 < hb[b].nrows; c0 += 256)
          tall.push_back(TileItem{static_cast<int32_t>(b), static_cast<int32_t>(T_bi[b]), 0, 0, c0, 0});
      L.ntfin = static_cast<int32_t>(tall.size() - L.tfin_off);
      // ---- persistent tile-DAG executor work of this level (tiled mode) ----
      {
        ExecBuilder X;
        // per diagonal block factored in this launch: tile-column (L part) and
        // tile-row (U part) completion markers for merged panel work
        std::map<int64_t, std::vector<int>> coldone, rowdone;
        std::map<int64_t, std::vector<int32_t>> xtid_of;  // diagonal row -> executor tile
        // absorbed DMMA SSSSM tiles of the previous level: (task, first and last target column)
        // per target block
        std::map<int64_t, std::vector<std::array<int32_t, 3>>> upd_of;
        if (absorbed_lv == lv - 1) {
          // long tiles run as a chain of pieces of <= LBK_ABSORB_PIECE inner chunks (each piece
          // C -= its partial product, in k order: deterministic), so a CTA is never held for a
          // whole K loop and the chain tasks of the launch interleave with the updates
          const char* pc = std::getenv("LBK_ABSORB_PIECE");
          const int piece = pc ? std::max(1, std::atoi(pc)) : 16;
          for (int64_t q = 0; q < absorbed_n; ++q) {
            const GemmItem gi = mall[absorbed_off + q];
            const GemmTask& gt = gtasks[gi.task];
            const int nk = gi.ke - gi.ks;
            const int np_ = std::max(1, (nk + piece - 1) / piece);
            int x = -1;
            for (int pq = 0; pq < np_; ++pq) {
              int64_t idx = absorbed_off + q;
              GemmItem part = gi;
              if (np_ > 1) {
                part.ks = gi.ks + static_cast<int32_t>((static_cast<int64_t>(nk) * pq) / np_);
                part.ke = gi.ks + static_cast<int32_t>((static_cast<int64_t>(nk) * (pq + 1)) / np_);
                idx = static_cast<int64_t>(mall.size());
                mall.push_back(part);
              }
              x = X.add(X_SSSSM, idx, gt.c, 0, 0, std::min(part.ke - part.ks, 32767), 0, 0,
                        x >= 0 ? std::vector<int>{x} : std::vector<int>{});
            }
            int32_t lo = INT32_MAX, hi = -1;
            for (int n = gi.n0; n < std::min(gi.n0 + GBN, hb[gt.b].nC); ++n) {
              const int32_t cc = gt.cmap >= 0 ? hmaps[gt.cmap + n] : n;
              if (cc < 0) continue;
              lo = std::min(lo, cc);
              hi = std::max(hi, cc);
            }
            if (hi >= 0) upd_of[gt.c].push_back({x, lo, hi});
          }
        }
        auto upd_cols = [&](int64_t blk, int c0, int c1) {  // absorbed updates of target columns [c0, c1)
          std::vector<int> v;
          auto it = upd_of.find(blk);
          if (it != upd_of.end())
            for (const auto& u : it->second)
              if (u[1] < c1 && u[2] >= c0) v.push_back(u[0]);
          return v;
        };
        for (size_t q = 0; q < tgetrf[lv].size(); ++q) {
          const int64_t b = tgetrf[lv][q];
          const int m = hb[b].nrows;
          const int32_t stp = static_cast<int32_t>(T_bi[b]);
          if (band.count(b)) {
            // banded diagonal block: one sweeping task per independent segment instead of
            // the tile DAG (refined plans: only the segments whose level is this one)
            const BandInfo& bi = band.at(b);
            std::vector<int> band_tasks;
            for (size_t q = 0; q < bi.seg.size(); ++q) {
              if (refine && bi.lev[q] != lv) continue;
              const int s0 = bi.seg[q].first, s1 = bi.seg[q].second;
              band_tasks.push_back(X.add(X_BAND, b, s0, bi.bl, bi.bu, s1 - s0, stp, 0, {}));
            }
            if (merge_next) {
              const int done = X.add(X_NOP, b, b, 0, 0, 0, stp, 0, band_tasks);
              coldone[b].assign(1, done);
              rowdone[b].assign(1, done);
              xtid_of[b].assign(m, 0);
            }
            continue;
          }
          // executor tiling of this diagonal block: subtree-aligned boundaries (uniform 64
          // columns in dense-scratch mode, where every tile is full anyway)
          const std::vector<int32_t>& tb = diag_tiling(b).tb;
          const int nt = static_cast<int>(tb.size()) - 1;
          if (!xtb_of.count(b)) {
            xtb_of[b] = static_cast<int64_t>(hxtb.size());
            hb[b].xtb1 = static_cast<int64_t>(hxtb.size()) + 1;
            hxtb.insert(hxtb.end(), tb.begin(), tb.end());
          }
          std::vector<int32_t> tid_of(m);
          for (int x = 0; x < nt; ++x)
            for (int y = tb[x]; y < tb[x + 1]; ++y) tid_of[y] = x;
          xtid_of[b] = tid_of;
          // xocc[col tile * nt + row tile]: tiles holding pattern entries
          std::vector<char> xocc(static_cast<size_t>(nt) * nt, all_full ? 1 : 0);
          if (!all_full) {
            const int64_t* scp = colptr + T_cp[b];
            const int64_t* sri = rowidx + T_ent[b];
            for (int col = 0; col < m; ++col)
              for (int64_t e = scp[col]; e < scp[col + 1]; ++e)
                xocc[static_cast<size_t>(tid_of[col]) * nt + tid_of[sri[e]]] = 1;
          }
          // column maxima at GETRF entry: tasks over (column tile, row chunk of
          // COLMAX_ROWS); every first write into column tile c waits for all of
          // column c's colmax tasks
          std::vector<int> last(static_cast<size_t>(nt) * nt, -1), lt(nt, -1), ut(nt, -1), fin_deps;
          std::vector<std::vector<int>> colj(nt);
          for (int cc = 0; cc < nt; ++cc)
            for (int rc = 0; rc * COLMAX_ROWS < m; ++rc) {
              const int col = X.add(X_COLMAX, b, b, rc, cc, 0, stp, -1, upd_cols(b, tb[cc], tb[cc + 1]));
              colj[cc].push_back(col);
              fin_deps.push_back(col);
            }
          auto L_ = [&](int r, int cc) -> int& { return last[static_cast<size_t>(cc) * nt + r]; };
          auto prev_raw = [&](int r, int cc, std::vector<int> extra) {
            const int l = L_(r, cc);
            if (l >= 0) extra.push_back(l);
            else extra.insert(extra.end(), colj[cc].begin(), colj[cc].end());
            return extra;
          };
          // trailing updates of a tile from consecutive steps wait here and run as one task
          // (up to panel_agg of them, XTask::pad1, k order: bitwise identical); any use of the
          // tile's last writer (prev) emits the pending task first
          struct GPend {
            int k0 = -1, cnt = 0;
            std::vector<int> deps;
          };
          std::map<std::pair<int, int>, GPend> gpend;
          auto flush_gemm = [&](int r, int cc) {
            auto it = gpend.find({r, cc});
            if (it == gpend.end()) return;
            GPend gp = it->second;
            gpend.erase(it);
            const int tsk = X.add(X_GEMM, b, b, r, cc, gp.k0, stp, gp.k0 * 4 + 2, prev_raw(r, cc, gp.deps));
            X.t[tsk].pad1 = static_cast<int16_t>(gp.cnt);
            L_(r, cc) = tsk;
          };
          auto prev = [&](int r, int cc, std::vector<int> extra) {
            flush_gemm(r, cc);
            return prev_raw(r, cc, std::move(extra));
          };
          auto add_gemm = [&](int r, int cc, int kb, int lt_r, int ut_c) {
            if (panel_agg <= 1) {
              L_(r, cc) = X.add(X_GEMM, b, b, r, cc, kb, stp, kb * 4 + 2, prev_raw(r, cc, {lt_r, ut_c}));
              return;
            }
            auto it = gpend.find({r, cc});
            if (it != gpend.end() && (it->second.k0 + it->second.cnt != kb || it->second.cnt >= panel_agg))
              flush_gemm(r, cc);
            GPend& gp = gpend[{r, cc}];
            if (gp.cnt == 0) gp.k0 = kb;
            ++gp.cnt;
            gp.deps.push_back(lt_r);
            gp.deps.push_back(ut_c);
          };
          // the last update of diagonal tile kb (GEMM(kb, kb, kb-1)) is fused into
          // its LU task: one handoff and one tile round trip less per step of
          // the critical chain
          std::vector<int> fused_deps, fused_ops;
          bool fused = false;
          std::vector<std::vector<int>> colw(nt), roww(nt);  // writers of each tile column's L / row's U part
          for (int kb = 0; kb < nt; ++kb) {
            // chain: this step's LU task also solves L(kb+1, kb) and U(kb, kb+1), the operands
            // of the next diagonal update (both tiles present), so the critical chain has one
            // task and one handoff per step instead of three and two
            const bool chain = LBK_CHAIN_TRSM && kb + 1 < nt && xocc[static_cast<size_t>(kb) * nt + kb + 1] &&
                               xocc[static_cast<size_t>(kb + 1) * nt + kb];
            // chain-2: this step's LU task also solves L(kb+1, kb) (the operand the next diagonal
            // update waits for last), after releasing the tasks that need only the factored tile
            const bool chainL = !chain && chain_l && kb + 1 < nt && xocc[static_cast<size_t>(kb) * nt + kb + 1];
            std::vector<int> gdeps = fused ? fused_deps : prev(kb, kb, {});
            if (chain) {
              const std::vector<int> dl = prev(kb + 1, kb, {}), du = prev(kb, kb + 1, {});
              gdeps.insert(gdeps.end(), dl.begin(), dl.end());
              gdeps.insert(gdeps.end(), du.begin(), du.end());
            }
            std::vector<int> gdeps2 = fused && !chain ? fused_ops : std::vector<int>{};
            if (chainL) {  // the L tile's last update: waited for with the operands (phase 2)
              const std::vector<int> dl = prev(kb + 1, kb, {});
              gdeps.insert(gdeps.end(), dl.begin(), dl.end());
              gdeps2.insert(gdeps2.end(), dl.begin(), dl.end());
            }
            // GETRF_UPD loads its target tile before the two operand tiles exist (phase 2)
            const int g = fused ? X.add(X_GETRF_UPD, b, b, kb, kb, kb - 1, stp, kb * 4, gdeps, gdeps2)
                                : X.add(X_GETRF, b, b, kb, kb, kb, stp, kb * 4, gdeps, gdeps2);
            X.t[g].chain = chain ? 1 : chainL ? 2 : 0;
            fused = false;
            colw[kb].push_back(g);
            roww[kb].push_back(g);
            L_(kb, kb) = g;
            fin_deps.push_back(g);
            for (int r = kb + 1; r < nt; ++r) {
              lt[r] = -1;
              if (!xocc[static_cast<size_t>(kb) * nt + r]) continue;
              lt[r] = ((chain || chainL) && r == kb + 1)
                          ? g
                          : X.add(X_TRSM_L, b, b, r, kb, kb, stp, kb * 4 + 1, prev(r, kb, {g}), {g});
              if (chainL && lt[r] != g) X.mark_early(g, lt[r]);
              colw[kb].push_back(lt[r]);
              L_(r, kb) = lt[r];
              fin_deps.push_back(lt[r]);
            }
            for (int cc = kb + 1; cc < nt; ++cc) {
              ut[cc] = -1;
              if (!xocc[static_cast<size_t>(cc) * nt + kb]) continue;
              ut[cc] = (chain && cc == kb + 1) ? g
                                               : X.add(X_TRSM_U, b, b, kb, cc, kb, stp, kb * 4 + 1, prev(kb, cc, {g}), {g});
              if (chainL) X.mark_early(g, ut[cc]);
              roww[kb].push_back(ut[cc]);
              L_(kb, cc) = ut[cc];
            }
            for (int cc = kb + 1; cc < nt; ++cc) {
              if (ut[cc] < 0) continue;
              for (int r = kb + 1; r < nt; ++r) {
                if (lt[r] < 0) continue;
                if (r == kb + 1 && cc == kb + 1) {
                  fused = true;
                  fused_deps = prev(r, cc, {lt[r], ut[cc]});
                  fused_ops = {lt[r], ut[cc]};
                  continue;
                }
                add_gemm(r, cc, kb, lt[r], ut[cc]);
              }
            }
          }
          while (!gpend.empty()) flush_gemm(gpend.begin()->first.first, gpend.begin()->first.second);  // (none expected)
          X.add(X_FINAL, b, b, 0, 0, 0, stp, 1 << 30, fin_deps);
          if (merge_next) {  // chained markers: column t done implies columns < t done
            coldone[b].assign(nt, -1);
            rowdone[b].assign(nt, -1);
            for (int t2 = 0; t2 < nt; ++t2) {
              std::vector<int> dc = colw[t2], dr = roww[t2];
              if (t2) {
                dc.push_back(coldone[b][t2 - 1]);
                dr.push_back(rowdone[b][t2 - 1]);
              }
              coldone[b][t2] = X.add(X_NOP, b, b, t2, 0, 0, stp, 0, dc);
              rowdone[b][t2] = X.add(X_NOP, b, b, t2, 1, 0, stp, 0, dr);
            }
          }
        }
        const std::vector<std::array<int32_t, 4>> none;
        const auto& ptasks_here = merge_next ? ptask[lv + 1] : merged_into_prev[lv] ? none : ptask[lv];
        if (merge_next) merged_into_prev[lv + 1] = 1;
        for (const auto& pt : ptasks_here) {
          const int32_t dblk = pt[1], xb = pt[2], stp = pt[3];
          const bool gessm = pt[0] == 1;
          const std::vector<int32_t> Rx = rows_of(xb), Cx = cols_of(xb);
          // Chain dimension (GESSM: the panel's rows R_X, TSTRF: its columns C_X) tiled at
          // most XT wide and cut wherever the diagonal factor's subtree-cut region changes,
          // so the substitution chains of independent subtrees are independent (the other
          // dimension: uniform XT).  The boundaries go to BlockDev::xtb1 of the panel.
          const std::vector<int32_t>& Dpos = gessm ? Rx : Cx;
          const std::vector<int32_t>& dseg = diag_tiling(dblk).seg;
          std::vector<int32_t> cb{0}, chid(Dpos.size(), 0);
          for (size_t a = 1; a < Dpos.size(); ++a)
            if (static_cast<int>(a) - cb.back() == XT || dseg[Dpos[a]] != dseg[Dpos[a - 1]])
              cb.push_back(static_cast<int32_t>(a));
          if (!Dpos.empty()) cb.push_back(static_cast<int32_t>(Dpos.size()));
          const int nch = static_cast<int>(cb.size()) - 1;
          for (int x = 0; x < nch; ++x)
            for (int y = cb[x]; y < cb[x + 1]; ++y) chid[y] = x;
          hb[xb].xtb1 = static_cast<int64_t>(hxtb.size()) + 1;
          hxtb.insert(hxtb.end(), cb.begin(), cb.end());
          const int tr = gessm ? nch : (hb[xb].nR + XT - 1) / XT, tc = gessm ? (hb[xb].nC + XT - 1) / XT : nch;
          auto rtile = [&](int a) { return gessm ? chid[a] : a / XT; };
          auto ctile = [&](int a) { return gessm ? a / XT : chid[a]; };
          std::vector<int> last(static_cast<size_t>(tr) * tc, -1);
          auto L_ = [&](int r, int cc) -> int& { return last[static_cast<size_t>(cc) * tr + r]; };
          // Tile occupancy from the filled patterns (tiled mode: no swaps, so the
          // patterns are exact): occX = tiles of the panel that hold entries; occD
          // = tiles of the diagonal factor gathered onto the panel's rows (GESSM:
          // strict L over R_X x R_X) or columns (TSTRF: strict U over C_X x C_X).
          // A panel tile outside the pattern stays zero through the solve (fill
          // closure), and a zero factor tile contributes nothing.
          const int nd = nch;
          std::vector<char> occX(static_cast<size_t>(tr) * tc, all_full ? 1 : 0);
          std::vector<char> occD(static_cast<size_t>(nd) * nd, all_full ? 1 : 0);
          if (!all_full) {
            std::vector<int32_t> rpos(hb[xb].nrows, -1), cpos(hb[xb].ncols, -1);
            for (size_t a = 0; a < Rx.size(); ++a) rpos[Rx[a]] = static_cast<int32_t>(a);
            for (size_t a = 0; a < Cx.size(); ++a) cpos[Cx[a]] = static_cast<int32_t>(a);
            const int64_t* xcp = colptr + T_cp[xb];
            const int64_t* xri = rowidx + T_ent[xb];
            for (int col = 0; col < hb[xb].ncols; ++col)
              for (int64_t e = xcp[col]; e < xcp[col + 1]; ++e)
                occX[static_cast<size_t>(ctile(cpos[col])) * tr + rtile(rpos[xri[e]])] = 1;
            const std::vector<int32_t>& pos = gessm ? rpos : cpos;
            const int64_t* dcp = colptr + T_cp[dblk];
            const int64_t* dri = rowidx + T_ent[dblk];
            for (int col = 0; col < hb[dblk].ncols; ++col) {
              const int pc = pos[col];
              if (pc < 0) continue;
              for (int64_t e = dcp[col]; e < dcp[col + 1]; ++e) {
                const int64_t row = dri[e];
                const bool keep = gessm ? row > col : row < col;
                if (keep && pos[row] >= 0) occD[static_cast<size_t>(chid[pc]) * nd + chid[pos[row]]] = 1;
              }
            }
          }
          auto X_ = [&](int r, int cc) { return occX[static_cast<size_t>(cc) * tr + r] != 0; };
          auto D_ = [&](int r, int cc) { return occD[static_cast<size_t>(cc) * nd + r] != 0; };
          // the update of the next tile along the substitution chain is fused
          // into that tile's solve task (one handoff + one tile round trip less
          // per chain step)
          std::vector<int> pend(static_cast<size_t>(tr) * tc, -2);  // step k of a pending fused update
          std::vector<std::vector<int>> pend_deps(static_cast<size_t>(tr) * tc);
          auto P_ = [&](int r, int cc) -> int& { return pend[static_cast<size_t>(cc) * tr + r]; };
          auto PD_ = [&](int r, int cc) -> std::vector<int>& { return pend_deps[static_cast<size_t>(cc) * tr + r]; };
          // merged launch: a task whose factor tiles come from the panel's tile
          // kt (rows R_kt for GESSM, columns C_kt for TSTRF) waits for the
          // diagonal factor's columns / rows up to the last of them
          const bool has_marks = merge_next && coldone.count(dblk);
          const std::vector<int32_t>& Rd = Dpos;
          auto mark = [&](int kt) -> int {
            if (!has_marks) return -1;
            const int idx = cb[kt + 1] - 1;
            const auto& v = gessm ? coldone[dblk] : rowdone[dblk];
            return v[std::min(static_cast<int>(v.size()) - 1, xtid_of.at(dblk)[Rd[idx]])];
          };
          // first writes into a panel tile wait for the absorbed updates of the panel
          const std::vector<int> xupd = upd_cols(xb, INT32_MIN, INT32_MAX);
          auto fw = [&](std::vector<int> v, int r, int cc) {
            if (L_(r, cc) < 0) v.insert(v.end(), xupd.begin(), xupd.end());
            return v;
          };
          // Updates of a panel tile from consecutive steps k far from its own solve step are
          // aggregated into one task (up to panel_agg of them, XTask::pad1 = count): it loads the
          // target once and applies them one after another in k order (the same operations as
          // separate tasks: bitwise identical), one task, load, store and handoff instead of
          // several.  The update from the step just before the tile's solve stays fused into it.
          struct Pend {
            int k0 = -1, cnt = 0;
            std::vector<int> deps;
          };
          std::map<std::pair<int, int>, Pend> pend_upd;
          auto flush_upd = [&](int type, int r, int cc) {
            auto it = pend_upd.find({r, cc});
            if (it == pend_upd.end() || it->second.cnt == 0) return;
            Pend& pq = it->second;
            std::vector<int> dep = pq.deps;
            dep.push_back(L_(r, cc));
            const int tsk = X.add(type, xb, dblk, r, cc, pq.k0, stp, pq.k0 * 4 + 2, fw(dep, r, cc));
            X.t[tsk].pad1 = static_cast<int16_t>(pq.cnt);
            L_(r, cc) = tsk;
            pend_upd.erase(it);
          };
          auto add_upd = [&](int type, int r, int cc, int kb, int d) {
            if (panel_agg <= 1) {
              L_(r, cc) = X.add(type, xb, dblk, r, cc, kb, stp, kb * 4 + 2, fw({d, L_(r, cc), mark(kb)}, r, cc));
              return;
            }
            auto it = pend_upd.find({r, cc});
            if (it != pend_upd.end() && (it->second.k0 + it->second.cnt != kb || it->second.cnt >= panel_agg))
              flush_upd(type, r, cc);
            Pend& pq = pend_upd[{r, cc}];
            if (pq.cnt == 0) pq.k0 = kb;
            ++pq.cnt;
            pq.deps.push_back(d);
            pq.deps.push_back(mark(kb));
          };
          if (pt[0] == 1) {  // GESSM: forward substitution down the row blocks
            for (int kb = 0; kb < tr; ++kb)
              for (int cc = 0; cc < tc; ++cc) {
                if (!X_(kb, cc)) continue;
                flush_upd(X_PG_UPD, kb, cc);  // (only when the tile has no fused update)
                if (P_(kb, cc) >= 0) PD_(kb, cc).push_back(mark(kb));
                const int d = P_(kb, cc) >= 0
                                  ? X.add(X_PG_FUSED, xb, dblk, kb, cc, P_(kb, cc), stp, kb * 4 + 1, PD_(kb, cc))
                                  : X.add(X_PG_DIAG, xb, dblk, kb, cc, kb, stp, kb * 4 + 1, fw({L_(kb, cc), mark(kb)}, kb, cc));
                L_(kb, cc) = d;
                for (int r = kb + 1; r < tr; ++r)
                  if (X_(r, cc) && D_(r, kb)) {  // L tile (r, kb)
                    if (r == kb + 1) {
                      flush_upd(X_PG_UPD, r, cc);
                      P_(r, cc) = kb;
                      PD_(r, cc) = fw({d, L_(r, cc)}, r, cc);
                      continue;
                    }
                    add_upd(X_PG_UPD, r, cc, kb, d);
                  }
              }
          } else {  // TSTRF: substitution along the column blocks
            for (int kb = 0; kb < tc; ++kb)
              for (int r = 0; r < tr; ++r) {
                if (!X_(r, kb)) continue;
                flush_upd(X_PT_UPD, r, kb);
                if (P_(r, kb) >= 0) PD_(r, kb).push_back(mark(kb));
                const int d = P_(r, kb) >= 0
                                  ? X.add(X_PT_FUSED, xb, dblk, r, kb, P_(r, kb), stp, kb * 4 + 1, PD_(r, kb))
                                  : X.add(X_PT_DIAG, xb, dblk, r, kb, kb, stp, kb * 4 + 1, fw({L_(r, kb), mark(kb)}, r, kb));
                L_(r, kb) = d;
                for (int cc = kb + 1; cc < tc; ++cc)
                  if (X_(r, cc) && D_(kb, cc)) {  // U tile (kb, cc)
                    if (cc == kb + 1) {
                      flush_upd(X_PT_UPD, r, cc);
                      P_(r, cc) = kb;
                      PD_(r, cc) = fw({d, L_(r, cc)}, r, cc);
                      continue;
                    }
                    add_upd(X_PT_UPD, r, cc, kb, d);
                  }
              }
          }
          for (auto& kv : std::vector<std::pair<std::pair<int, int>, Pend>>(pend_upd.begin(), pend_upd.end()))
            flush_upd(pt[0] == 1 ? X_PG_UPD : X_PT_UPD, kv.first.first, kv.first.second);  // (none expected)
        }
        for (const XTask& x : X.t) {  // executed flops of the tile tasks (full 64-tiles)
          if (x.type == X_SSSSM) continue;  // counted when absorbed
          const double t3 = 64.0 * 64.0 * 64.0;
          if (x.chain) c->exec_flops += x.chain == 1 ? 2 * t3 : t3;  // the solved tiles of the chain
          c->exec_flops += x.type == X_GETRF_UPD                                     ? 2 * t3 + 2 * t3 / 3
                           : x.type == X_PG_FUSED || x.type == X_PT_FUSED              ? 3 * t3
                           : x.type == X_PG_UPD || x.type == X_PT_UPD                 ? 2 * t3 * std::max<int>(1, x.pad1)
                           : x.type == X_GEMM                                         ? 2 * t3 * std::max<int>(1, x.pad1)
                           : x.type == X_GETRF                                       ? 2 * t3 / 3
                           : x.type == X_COLMAX || x.type == X_FINAL                 ? 0
                                                                                     : t3;
        }
        X.flush(&L, &xtasks, &xsucc_ptr, &xsucc, &xdeps0);
      }
      c->levels.push_back(L);
    }
    c->n_generic = static_cast<int64_t>(gall.size());
    c->n_gemm = static_cast<int64_t>(mall.size());
    c->n_panel = static_cast<int64_t>(dall.size());
    c->n_tile = static_cast<int64_t>(tall.size());
    c->n_exec = static_cast<int64_t>(xtasks.size());
    c->hblk = hb;
    LBK_CUDA(c->blk.upload(hb), st);
    LBK_CUDA(c->colptr.upload(hcp), st);
    LBK_CUDA(c->rows.upload(hrows), st);
    LBK_CUDA(c->map.upload(hmap), st);
    LBK_CUDA(c->csr_ptr.upload(hrp), st);
    LBK_CUDA(c->csr_col.upload(hcc), st);
    LBK_CUDA(c->csr_pos.upload(hcpos), st);
    LBK_CUDA(c->diag_csc.upload(hdcsc), st);
    LBK_CUDA(c->diag_csr.upload(hdcsr), st);
    LBK_CUDA(c->lv_cols.upload(hlvc), st);
    LBK_CUDA(c->lv_ptr.upload(hlvp), st);
    LBK_CUDA(c->rlist.upload(hrl), st);
    LBK_CUDA(c->clist.upload(hcl), st);
    LBK_CUDA(c->maps.upload(hmaps), st);
    LBK_CUDA(c->items.upload(gall), st);
    LBK_CUDA(c->gtasks.upload(gtasks), st);
    LBK_CUDA(c->gitems.upload(mall), st);
    LBK_CUDA(c->gemm_ws.alloc(std::max<int64_t>(max_ws_slots, 1) * GEMM_PART), st);
    LBK_CUDA(c->kchunks.upload(hkch.empty() ? std::vector<int32_t>(1, 0) : hkch), st);
    LBK_CUDA(c->ditems.upload(dall), st);
    LBK_CUDA(c->titems.upload(tall), st);
    LBK_CUDA(c->xtasks.upload(xtasks), st);
    LBK_CUDA(c->xsptr.upload(xsucc_ptr), st);
    LBK_CUDA(c->xsucc.upload(xsucc), st);
    LBK_CUDA(c->xdeps0.upload(xdeps0), st);
    LBK_CUDA(c->xtb.upload(hxtb.empty() ? std::vector<int32_t>(1, 0) : hxtb), st);
    LBK_CUDA(c->xdeps.alloc(xdeps0.size()), st);
    LBK_CUDA(c->xheads.alloc(c->levels.size()), st);
    LBK_CUDA(c->perm.alloc(ndiag), st);
    LBK_CUDA(c->colmax.alloc(ndiag), st);
    LBK_CUDA(c->bmax.alloc(ndiag), st);
    LBK_CUDA(c->vals.alloc(nnz_w), st);
    LBK_CUDA(c->vin.alloc(nnz), st);
    LBK_CUDA(c->vout.alloc(nnz), st);
    LBK_CUDA(c->err.alloc(2), st);
    LBK_CUDA(c->dirty.upload(std::vector<int>{1, 0}), st);
    // identity permutations until a GETRF writes them
    std::vector<int32_t> idp(ndiag);
    for (int64_t b = 0; b < nb; ++b)
      if (T_bi[b] == T_bj[b])
        for (int r = 0; r < hb[b].nrows; ++r) idp[hb[b].dg + r] = r;
    LBK_CUDA(cudaMemcpy(c->perm.p, idp.data(), idp.size() * sizeof(int32_t), cudaMemcpyHostToDevice), st);
    LBK_CUDA(c->perm0.upload(idp), st);  // (upload synchronizes the device: both copies have landed)
  } catch (const std::bad_alloc&) {
    return fail(st, LBK_ERR_OOM, "host allocation in lbk_plan");
  }
  // graph segments: segment s runs the launch levels whose tree level lies in
  // (cut_{s-1}, cut_s]; a rank exchanges blocks between segments
  c->seg_begin.assign(1, 0);
  {
    size_t l = 0;
    for (size_t tl = 0; tl < c->cut_after.size(); ++tl) {
      if (!c->cut_after[tl]) continue;
      while (l < c->levels.size() && c->levels[l].tree_level <= static_cast<int32_t>(tl)) ++l;
      c->seg_begin.push_back(static_cast<int32_t>(l));
    }
    c->seg_begin.push_back(static_cast<int32_t>(c->levels.size()));
  }
  drop_graphs(c);
  for (auto ev : c->dev) cudaEventDestroy(ev);
  for (auto ev : c->dev2) cudaEventDestroy(ev);
  c->dev.assign(c->levels.size(), nullptr);
  c->dev2.assign(c->levels.size(), nullptr);
  for (auto ev : c->lev) cudaEventDestroy(ev);
  c->lev.assign(c->levels.size(), nullptr);
  for (auto& ev : c->lev) LBK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), st);
  drop_sgraphs(c);
  if (build_out_ranges(c, st)) return st->code;
  for (auto& ev : c->dev) LBK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), st);
  for (auto& ev : c->dev2) LBK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), st);
  ok(st);
  return 0;
}

// Pristine A values in reference pool order (host -> device, kept resident).
int lbk_upload_values(lbk_ctx* c, const double* values, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  LBK_CUDA(cudaMemcpyAsync(c->vin.p, values, c->nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

}  // extern "C"

namespace {

// Capture one full factorization into the current capture of c->stream.
// With `evs`, an external (timing-capable) event record node closes each level.
// Launch levels [lo, hi) only; the prologue (zero, scatter, counter reset)
// belongs to the first segment and the gather to the last one.
void capture_factorization(lbk_ctx* c, double pivot_tol, double static_eps, std::vector<cudaEvent_t>* evs,
                           size_t lo, size_t hi, bool first, bool last, double* stream_out = nullptr) {
  DevPools P = pools(c);
  cudaStream_t s0 = c->stream;
  const bool exact = (c->flags & 2) != 0 || !std::isnan(static_eps);
  const bool use_exec = !exact && c->use_exec;
  if (first) {
    cudaMemsetAsync(c->err.p, 0xff, 2 * sizeof(unsigned long long), s0);
    if (exact || c->seg_begin.size() > 2) {
      cudaMemsetAsync(c->vals.p, 0, c->nnz_work * sizeof(double), s0);
    } else {
      // Outside the filled pattern the working pool stays exactly zero (the pattern
      // is elimination-closed, grid.py:3-5: every product landing there is an exact
      // zero) and the scatter rewrites every in-pattern entry, so the pool is only
      // zeroed after a run that may have left non-zeros there (an error, non-finite
      // input: 0 * inf) or at the first run.
      zero_if_dirty_kernel<<<148 * 8, 256, 0, s0>>>(c->vals.p, c->nnz_work, c->dirty.p);
    }
    scatter_kernel<<<148 * 8, 256, 0, s0>>>(c->vin.p, c->map.p, c->vals.p, c->nnz, c->dirty.p + 1);
  if (use_exec && c->n_exec) {
    cudaMemcpyAsync(c->xdeps.p, c->xdeps0.p, 2 * c->n_exec * sizeof(int), cudaMemcpyDeviceToDevice, s0);
    cudaMemsetAsync(c->xheads.p, 0, c->levels.size() * sizeof(int), s0);
    if (c->ndiag_rows) {  // colmax/bmax accumulate with atomic max; perms start as identity
      cudaMemsetAsync(c->colmax.p, 0, c->ndiag_rows * sizeof(double), s0);
      cudaMemsetAsync(c->bmax.p, 0, c->ndiag_rows * sizeof(unsigned long long), s0);
      cudaMemcpyAsync(c->perm.p, c->perm0.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToDevice, s0);
    }
  }
  }
  if (evs && first) cudaEventRecordWithFlags((*evs)[0], s0, cudaEventRecordExternal);
  // deferred SSSSM work of launch level l runs beside the next tree level; a
  // level at tree level T waits for the deferred work of tree levels <= T - 2
  std::vector<std::pair<cudaEvent_t, int32_t>> pending;  // (done event, first tree level that needs it)
  int64_t pend_lv = -1, pend_bytes = 0;  // streamed output not yet flushed
  for (size_t l = lo; l < hi; ++l) {
    const Level& L = c->levels[l];
    for (size_t q = 0; q < pending.size();) {
      if (pending[q].second <= L.tree_level_hi) {
        cudaStreamWaitEvent(s0, pending[q].first, 0);
        pending.erase(pending.begin() + q);
      } else {
        ++q;
      }
    }
    const bool has_t = !exact && (use_exec ? L.nexec > 0 : L.ntcol > 0);
    // instrumented replays (evs) run the deferred SSSSM groups inside their own
    // level, after its critical DMMA launch: every kernel family is then timed
    // without the cross-level overlap (which only shares the GPU differently)
    const bool inline_defer = evs != nullptr && (L.ngemmD || L.ngemmE);
    const bool own_absorbed = L.nabsorb > 0 && (exact || !use_exec);  // no executor launch to run them
    const bool br[NBRANCH] = {L.ngemm > 0 || inline_defer || own_absorbed,
                              (!use_exec && L.npanel > 0) || (exact && L.nexact > 0), has_t};
    // instrumented replays: per level [end, gemm b/e, panel b/e, getrf b/e, csc b/e]
    auto rec = [&](int k, cudaStream_t s) {
      if (evs) cudaEventRecordWithFlags((*evs)[1 + l * 13 + k], s, cudaEventRecordExternal);
    };
    if (br[0] || br[1] || br[2]) cudaEventRecord(c->fork, s0);
    if (br[0]) {
      cudaStreamWaitEvent(c->aux[0], c->fork, 0);
      rec(1, c->aux[0]);
      if (L.ngemm) gemm_map_kernel<<<L.ngemm, 256, GEMM_SMEM, c->aux[0]>>>(c->gitems.p + L.gemm_off, c->gtasks.p, P);
      if (own_absorbed)
        gemm_map_kernel<<<L.nabsorb, 256, GEMM_SMEM, c->aux[0]>>>(c->gitems.p + L.absorb_off, c->gtasks.p, P);
      if (L.ngred) gemm_reduce_kernel<<<L.ngred, 256, 0, c->aux[0]>>>(c->gitems.p + L.gred_off, c->gtasks.p, P);
      if (inline_defer) {
        if (L.ngemmD)
          gemm_map_kernel<<<L.ngemmD, 256, GEMM_SMEM, c->aux[0]>>>(c->gitems.p + L.gemmD_off, c->gtasks.p, P);
        if (L.ngemmE)
          gemm_map_kernel<<<L.ngemmE, 256, GEMM_SMEM, c->aux[0]>>>(c->gitems.p + L.gemmE_off, c->gtasks.p, P);
      }
      rec(2, c->aux[0]);
      cudaEventRecord(c->join[0], c->aux[0]);
    }
    if (br[1]) {
      cudaStreamWaitEvent(c->aux[1], c->fork, 0);
      rec(3, c->aux[1]);
      if (L.npanel)
        panel_kernel<<<L.npanel, 256, L.panel_smem, c->aux[1]>>>(c->ditems.p + L.panel_off, P, pivot_tol,
                                                                 static_eps);
      if (exact && L.nexact)
        panel_kernel<<<L.nexact, 512, L.exact_smem, c->aux[1]>>>(c->ditems.p + L.exact_off, P, pivot_tol,
                                                                 static_eps);
      rec(4, c->aux[1]);
      cudaEventRecord(c->join[1], c->aux[1]);
    }
    if (br[2]) {
      cudaStream_t s2 = c->aux[2];
      cudaStreamWaitEvent(s2, c->fork, 0);
      rec(5, s2);
      if (use_exec) {
        XLevel X;
        X.tasks = c->xtasks.p + L.exec_off;
        X.succ_ptr = c->xsptr.p + L.sptr_off;
        X.succ = c->xsucc.p + L.succ_off;
        X.deps = c->xdeps.p + 2 * L.exec_off;
        X.head = c->xheads.p + l;
        X.ntasks = L.nexec;
        X.trace = (evs && c->xtrace.p) ? c->xtrace.p + 8 * L.exec_off : nullptr;
        X.gitems = c->gitems.p;
        X.gtasks = c->gtasks.p;
        if (L.band4 && c->use_bandreg) {
          const int grid = std::max(1, std::min(L.nexec, 148 * std::min(c->exec_per_sm, c->band_per_sm)));
          exec_band_kernel<<<grid, 256, EXEC_SMEM, s2>>>(X, P, pivot_tol);
        } else {
          const int grid = std::max(1, std::min(L.nexec, 148 * c->exec_per_sm));
          exec_kernel<<<grid, 256, EXEC_SMEM, s2>>>(X, P, pivot_tol);
        }
      } else {
        getrf_colmax_kernel<<<L.ntcol, 256, 0, s2>>>(c->titems.p + L.tcol_off, P);
        for (int k = 0; k < L.nsub; ++k) {
          const SubStep& S = c->subs[L.sub_off + k];
          if (S.ngetrf) tile_getrf_kernel<<<S.ngetrf, 256, 0, s2>>>(c->titems.p + S.getrf_off, P);
          if (S.ntrsm) tile_trsm_kernel<<<S.ntrsm, 128, TRSM_SMEM, s2>>>(c->titems.p + S.trsm_off, P);
          if (S.ngemm) tile_gemm_kernel<<<S.ngemm, 128, TGEMM_SMEM, s2>>>(c->titems.p + S.gemm_off, P);
        }
        getrf_finalize_kernel<<<L.ntfin, 256, 0, s2>>>(c->titems.p + L.tfin_off, P, pivot_tol);
      }
      rec(6, s2);
      cudaEventRecord(c->join[2], s2);
    }
    if (L.nitems) {
      const size_t smem = static_cast<size_t>(L.warps) * L.acc_len * sizeof(double);
      rec(7, s0);
      level_kernel<<<L.nitems, L.warps * 32, smem, s0>>>(c->items.p + L.item_off, P, L.acc_len, pivot_tol,
                                                         static_eps);
      rec(8, s0);
    }
    for (int k = 0; k < NBRANCH; ++k)
      if (br[k]) cudaStreamWaitEvent(s0, c->join[k], 0);
    if (stream_out && c->srange_off[l + 1] > c->srange_off[l]) {
      // the blocks finished since the last flush: gather + copy to the host on
      // the copy stream, batched over levels (>= 16 MB or 256 ranges, or the
      // last level) with ranges less than 256 KB apart merged: one small copy
      // per level and range would serialise the copy stream behind many
      // launch-latency-bound nodes.  A merged gap re-sends values whose blocks
      // are not final yet; their own (later, same-stream) copy overwrites them.
      if (pend_lv < 0) pend_lv = static_cast<int64_t>(l);
      for (int64_t q = c->srange_off[l]; q < c->srange_off[l + 1]; ++q) pend_bytes += c->hsranges[2 * q + 1] * 8;
    }
    if (stream_out && pend_lv >= 0) {
      const int64_t pend_ranges = c->srange_off[l + 1] - c->srange_off[pend_lv];
      if (pend_bytes >= (16ll << 20) || pend_ranges >= 256 || l + 1 == hi) {
        cudaEventRecord(c->lev[l], s0);
        cudaStreamWaitEvent(c->cstream, c->lev[l], 0);
        const int64_t r0 = c->srange_off[pend_lv], nr = c->srange_off[l + 1] - r0;
        const int64_t p0 = c->spiece_off[pend_lv], np_ = c->spiece_off[l + 1] - p0;
        range_gather_kernel<<<static_cast<int>(std::min<int64_t>(np_, 148 * 4)), 256, 0, c->cstream>>>(
            c->vals.p, out_map(c), c->vout.p, c->sranges.p + 2 * p0, np_);
        std::vector<std::pair<int64_t, int64_t>> rs(nr);
        for (int64_t q = 0; q < nr; ++q) rs[q] = {c->hsranges[2 * (r0 + q)], c->hsranges[2 * (r0 + q) + 1]};
        std::sort(rs.begin(), rs.end());
        for (size_t q = 0; q < rs.size();) {
          int64_t off = rs[q].first, end = off + rs[q].second;
          for (++q; q < rs.size() && rs[q].first - end <= (32 << 10); ++q) end = std::max(end, rs[q].first + rs[q].second);
          cudaMemcpyAsync(stream_out + off, c->vout.p + off, (end - off) * sizeof(double), cudaMemcpyDeviceToHost,
                          c->cstream);
        }
        pend_lv = -1;
        pend_bytes = 0;
      }
    }
    if ((L.ngemmD || L.ngemmE) && !inline_defer) {
      // deferred SSSSM updates start once this level's critical work is done
      // and run (low stream priority) beside the next one (slack 2) or two
      // (slack >= 3) levels
      cudaEventRecord(c->dfork, s0);
      for (int cls = 0; cls < 2; ++cls) {
        const int32_t nd = cls ? L.ngemmE : L.ngemmD;
        if (!nd) continue;
        cudaStream_t ds = cls ? c->dstream2 : c->dstream;
        cudaStreamWaitEvent(ds, c->dfork, 0);
        const GemmItem* items = c->gitems.p + (cls ? L.gemmE_off : L.gemmD_off);
        if (c->defer_ctas > 0)
          gemm_map_loop_kernel<<<std::min(nd, c->defer_ctas), 256, GEMM_SMEM, ds>>>(items, nd, c->gtasks.p, P);
        else
          gemm_map_kernel<<<nd, 256, GEMM_SMEM, ds>>>(items, c->gtasks.p, P);
        cudaEvent_t ev = cls ? c->dev2[l] : c->dev[l];
        cudaEventRecord(ev, ds);
        pending.push_back({ev, L.tree_level + (cls ? 3 : 2)});
      }
    }
    rec(0, s0);
  }
  for (const auto& pq : pending) cudaStreamWaitEvent(s0, pq.first, 0);
  if (last) mark_dirty_kernel<<<1, 32, 0, s0>>>(c->err.p, c->dirty.p);
  if (stream_out) {
    cudaEventRecord(c->cev, c->cstream);
    cudaStreamWaitEvent(s0, c->cev, 0);
    return;
  }
  if (last) gather_kernel<<<148 * 8, 256, 0, s0>>>(c->vals.p, out_map(c), c->vout.p, c->nout);
}

int nsegments(const lbk_ctx* c) { return static_cast<int>(c->seg_begin.size()) - 1; }

bool same(double a, double b) { return a == b || (std::isnan(a) && std::isnan(b)); }

int build_graph(lbk_ctx* c, double pivot_tol, double static_eps, lbk_status* st) {
  const int ns = nsegments(c);
  if (c->refined && !std::isnan(static_eps))
    return fail(st, LBK_ERR_BAD_ARG, "static pivoting needs a plan without segment-refined levels (lbk_plan flags bit 2)");
  if (static_cast<int>(c->graphs.size()) == ns && same(c->g_tol, pivot_tol) && same(c->g_eps, static_eps)) return 0;
  drop_graphs(c);
  for (int s = 0; s < ns; ++s) {
    cudaGraph_t g;
    LBK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), st);
    (void)cudaGetLastError();
    capture_factorization(c, pivot_tol, static_eps, nullptr, c->seg_begin[s], c->seg_begin[s + 1], s == 0,
                          s == ns - 1);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (e != cudaSuccess) return cuda_fail(st, e, "graph capture");
    e = cudaGetLastError();  // a launch rejected during capture (bad configuration)
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      return cuda_fail(st, e, "kernel launch during capture");
    }
    size_t nodes = 0;
    cudaGraphGetNodes(g, nullptr, &nodes);
    cudaGraphExec_t ge = nullptr;
    if (nodes) e = cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(st, e, "graph instantiate");
    c->graphs.push_back(ge);  // nullptr: nothing for this rank in the segment
  }
  c->g_tol = pivot_tol;
  c->g_eps = static_eps;
  return 0;
}

cudaError_t launch_all(lbk_ctx* c) {
  for (auto g : c->graphs)
    if (g) {
      const cudaError_t e = cudaGraphLaunch(g, c->stream);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

// Status from the two error words (lowest failing (block << 32 | col) of a
// zero pivot / of a needed row swap; ~0 = none).
int status_from_err(const unsigned long long* h, lbk_status* st) {
  const unsigned long long none = ~0ull;
  ok(st);
  if (h[0] != none && (h[1] == none || h[0] < h[1])) {
    st->code = LBK_ERR_ZERO_PIVOT;
    st->block = static_cast<int32_t>(h[0] >> 32);
    st->col = static_cast<int32_t>(h[0] & 0xffffffffu);
    std::snprintf(st->msg, sizeof(st->msg), "zero pivot in diagonal block %d, local column %d", st->block, st->col);
    return st->code;
  }
  if (h[1] != none) {
    st->code = LBK_ERR_PIVOT_SWAP;
    st->block = static_cast<int32_t>(h[1] >> 32);
    st->col = static_cast<int32_t>(h[1] & 0xffffffffu);
    std::snprintf(st->msg, sizeof(st->msg), "row swap needed in diagonal block %d, column %d", st->block, st->col);
    return st->code;
  }
  return 0;
}

int finish(lbk_ctx* c, lbk_status* st) {
  unsigned long long h[2];
  LBK_CUDA(cudaMemcpyAsync(h, c->err.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  return status_from_err(h, st);
}

}  // namespace

extern "C" {

// Device-resident factorization of the resident A values.  *ms = device time
// of the whole graph (zero + scatter, every level, gather).
int lbk_factorize(lbk_ctx* c, double pivot_tol, double static_eps, float* ms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (build_graph(c, pivot_tol, static_eps, st)) return st->code;
  LBK_CUDA(cudaEventRecord(c->ev0, c->stream), st);
  LBK_CUDA(launch_all(c), st);
  LBK_CUDA(cudaEventRecord(c->ev1, c->stream), st);
  const int rc = finish(c, st);
  if (rc == LBK_ERR_CUDA || rc == LBK_ERR_OOM) return rc;
  if (ms) {
    float t = 0;
    cudaEventElapsedTime(&t, c->ev0, c->ev1);
    *ms = t;
  }
  return rc;
}

// End-to-end: host A values in, host factor values (reference pool order)
// and per-diagonal-row local permutations out.
namespace {
int factorize_host_impl(lbk_ctx* c, const double* a_values, bool a_is_pool, double* lu_values, int32_t* perms,
                        double pivot_tol, double static_eps, lbk_status* st);
}

int lbk_factorize_host(lbk_ctx* c, const double* a_values, double* lu_values, int32_t* perms, double pivot_tol,
                       double static_eps, lbk_status* st) {
  return factorize_host_impl(c, a_values, true, lu_values, perms, pivot_tol, static_eps, st);
}

int lbk_bind_matrix(lbk_ctx* c, int64_t nnz_a, const int64_t* pool_pos, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  for (int64_t k = 0; k < nnz_a; ++k)
    if (pool_pos[k] < 0 || pool_pos[k] >= c->nnz) return fail(st, LBK_ERR_DIM_MISMATCH, "pool position out of range");
  LBK_CUDA(c->amap.alloc(std::max<int64_t>(nnz_a, 1)), st);
  if (nnz_a) LBK_CUDA(cudaMemcpy(c->amap.p, pool_pos, nnz_a * sizeof(int64_t), cudaMemcpyHostToDevice), st);
  LBK_CUDA(cudaDeviceSynchronize(), st);  // order the pageable copy before kernels on the engine streams
  LBK_CUDA(c->avals.alloc(std::max<int64_t>(nnz_a, 1)), st);
  c->nnz_a = nnz_a;
  ok(st);
  return 0;
}

int lbk_refactor_host(lbk_ctx* c, const double* a_values, double* lu_values, int32_t* perms, double pivot_tol,
                      double static_eps, lbk_status* st) {
  if (!c->amap.p) return fail(st, LBK_ERR_BAD_ARG, "lbk_refactor_host before lbk_bind_matrix");
  return factorize_host_impl(c, a_values, false, lu_values, perms, pivot_tol, static_eps, st);
}

}  // extern "C"

namespace {
int factorize_host_impl(lbk_ctx* c, const double* a_values, bool a_is_pool, double* lu_values, int32_t* perms,
                        double pivot_tol, double static_eps, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  // A's values into the reference pool (vin): the whole pool, or A's entries
  // expanded through the bound positions (fill entries are zero)
  auto upload_input = [&]() -> cudaError_t {
    if (a_is_pool)
      return cudaMemcpyAsync(c->vin.p, a_values, c->nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream);
    cudaError_t e = cudaMemcpyAsync(c->avals.p, a_values, c->nnz_a * sizeof(double), cudaMemcpyHostToDevice,
                                    c->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->vin.p, 0, c->nnz * sizeof(double), c->stream);
    if (e == cudaSuccess && c->nnz_a)
      expand_kernel<<<148 * 4, 256, 0, c->stream>>>(c->avals.p, c->amap.p, c->vin.p, c->nnz_a);
    return e == cudaSuccess ? cudaGetLastError() : e;
  };
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, lu_values) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  (void)cudaGetLastError();
  if (c->refined && !std::isnan(static_eps))
    return fail(st, LBK_ERR_BAD_ARG, "static pivoting needs a plan without segment-refined levels (lbk_plan flags bit 2)");
  if (pinned && nsegments(c) == 1 && c->nnz >= (int64_t{1} << 24)) {
    // streamed output: every block's factor values are copied to the host while
    // later levels still run (one graph per output buffer)
    lbk_ctx::SGraph* slot = nullptr;
    for (auto& q : c->sg)
      if (q.g && q.out == lu_values && same(q.tol, pivot_tol) && same(q.eps, static_eps)) slot = &q;
    if (!slot) {
      slot = c->sg[0].used <= c->sg[1].used ? &c->sg[0] : &c->sg[1];  // least recently used
      if (slot->g) cudaGraphExecDestroy(slot->g);
      *slot = lbk_ctx::SGraph{};
      cudaGraph_t g;
      LBK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), st);
      (void)cudaGetLastError();
      capture_factorization(c, pivot_tol, static_eps, nullptr, 0, c->levels.size(), true, true, lu_values);
      cudaError_t e = cudaStreamEndCapture(c->stream, &g);
      if (e != cudaSuccess) return cuda_fail(st, e, "streamed graph capture");
      e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaGraphInstantiate(&slot->g, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(st, e, "streamed graph");
      slot->out = lu_values;
      slot->tol = pivot_tol;
      slot->eps = static_eps;
    }
    slot->used = ++c->sg_clock;
    LBK_CUDA(upload_input(), st);
    LBK_CUDA(cudaGraphLaunch(slot->g, c->stream), st);
    if (perms && c->ndiag_rows)
      LBK_CUDA(cudaMemcpyAsync(perms, c->perm.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream),
               st);
    return finish(c, st);
  }
  if (build_graph(c, pivot_tol, static_eps, st)) return st->code;
  LBK_CUDA(upload_input(), st);
  LBK_CUDA(launch_all(c), st);
  LBK_CUDA(cudaMemcpyAsync(lu_values, c->vout.p, c->nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream), st);
  if (perms && c->ndiag_rows)
    LBK_CUDA(cudaMemcpyAsync(perms, c->perm.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream),
             st);
  return finish(c, st);
}
}  // namespace

extern "C" {

// ---- distribution hooks (2D block-cyclic owner-computes, paper_2512_04389_b200/parallel.py) ----

int lbk_set_task_mask(lbk_ctx* c, int64_t ntasks, const int8_t* mask, lbk_status* st) {
  if (!c) return fail(st, LBK_ERR_BAD_ARG, "null ctx");
  if (mask) c->mask.assign(mask, mask + ntasks);
  else c->mask.clear();
  ok(st);
  return 0;
}

int lbk_set_cuts(lbk_ctx* c, int64_t nlevels, const int8_t* cut_after, lbk_status* st) {
  if (!c) return fail(st, LBK_ERR_BAD_ARG, "null ctx");
  if (cut_after) c->cut_after.assign(cut_after, cut_after + nlevels);
  else c->cut_after.clear();
  ok(st);
  return 0;
}

int lbk_num_segments(lbk_ctx* c) { return c ? nsegments(c) : 0; }

int lbk_set_task_defer(lbk_ctx* c, int64_t ntasks, const int8_t* defer, lbk_status* st) {
  if (!c) return fail(st, LBK_ERR_BAD_ARG, "null ctx");
  if (defer) c->defer.assign(defer, defer + ntasks);
  else c->defer.clear();
  ok(st);
  return 0;
}

int lbk_run_segment(lbk_ctx* c, int32_t seg, double pivot_tol, double static_eps, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (seg < 0 || seg >= nsegments(c)) return fail(st, LBK_ERR_BAD_ARG, "segment out of range");
  if (build_graph(c, pivot_tol, static_eps, st)) return st->code;
  if (seg == 0) LBK_CUDA(cudaEventRecord(c->ev0, c->stream), st);
  if (c->graphs[seg]) LBK_CUDA(cudaGraphLaunch(c->graphs[seg], c->stream), st);
  if (seg == nsegments(c) - 1) LBK_CUDA(cudaEventRecord(c->ev1, c->stream), st);
  ok(st);
  return 0;
}

int lbk_finish_raw(lbk_ctx* c, float* ms, uint64_t* err2, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  unsigned long long h[2];
  LBK_CUDA(cudaMemcpyAsync(h, c->err.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  err2[0] = h[0];
  err2[1] = h[1];
  if (ms) {
    float t = 0;
    cudaEventElapsedTime(&t, c->ev0, c->ev1);
    *ms = t;
  }
  ok(st);
  return 0;
}

int lbk_status_from_err(const uint64_t* err2, lbk_status* st) {
  const unsigned long long h[2] = {err2[0], err2[1]};
  return status_from_err(h, st);
}

void* lbk_stream(lbk_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int lbk_work_ptrs(lbk_ctx* c, void** vals, void** perm, void** vout) {
  if (vals) *vals = c->vals.p;
  if (perm) *perm = c->perm.p;
  if (vout) *vout = c->vout.p;
  return 0;
}

// layout[3 x nblocks]: working-pool offset, working entries, diagonal-row offset (-1 off-diagonal)
int lbk_block_layout(lbk_ctx* c, int64_t* layout) {
  const int64_t nb = static_cast<int64_t>(c->hblk.size());
  for (int64_t b = 0; b < nb; ++b) {
    layout[b] = c->hblk[b].ent;
    layout[nb + b] = c->wlen[b];
    layout[2 * nb + b] = c->isdiag[b] ? c->hblk[b].dg : -1;
  }
  return 0;
}

int lbk_download(lbk_ctx* c, double* lu_values, int32_t* perms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  LBK_CUDA(cudaMemcpyAsync(lu_values, c->vout.p, c->nout * sizeof(double), cudaMemcpyDeviceToHost, c->stream), st);
  if (perms && c->ndiag_rows)
    LBK_CUDA(cudaMemcpyAsync(perms, c->perm.p, c->ndiag_rows * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream),
             st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

// Output in the export layout of the caller (LUFactors blocks as stored by the
// reference's export, factorize.py:370-384): nout entries, block b's output in
// [xoff[b], xoff[b+1]) (blocks in pool order), xref[x] = reference-pool entry of
// output entry x, or -1 for a constant 1.0 (the unit diagonal of L).
int lbk_set_export(lbk_ctx* c, int64_t nout, const int64_t* xref, const int64_t* xoff, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  const int64_t nb = static_cast<int64_t>(c->ref_off.size());
  if (xoff[0] != 0 || xoff[nb] != nout) return fail(st, LBK_ERR_BAD_ARG, "export offsets do not cover nout");
  for (int64_t x = 0; x < nout; ++x)
    if (xref[x] < -1 || xref[x] >= c->nnz) return fail(st, LBK_ERR_BAD_ARG, "export entry out of range");
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  DevBuf<int64_t> xr;
  std::vector<int64_t> hx(xref, xref + nout);
  LBK_CUDA(xr.upload(hx), st);
  LBK_CUDA(c->omap.alloc(std::max<int64_t>(nout, 1)), st);
  compose_map_kernel<<<148 * 4, 256, 0, c->stream>>>(xr.p, c->map.p, c->omap.p, nout);
  LBK_CUDA(cudaGetLastError(), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  c->nout = nout;
  c->out_off.assign(xoff, xoff + nb);
  c->out_len.resize(nb);
  for (int64_t b = 0; b < nb; ++b) c->out_len[b] = xoff[b + 1] - xoff[b];
  LBK_CUDA(c->out_off_d.upload(std::vector<int64_t>(xoff, xoff + nb + 1)), st);
  LBK_CUDA(c->zcount.alloc(std::max<int64_t>(nb, 1)), st);
  LBK_CUDA(c->vout.alloc(std::max<int64_t>(nout, 1)), st);
  drop_graphs(c);  // the gather nodes captured the old output map / buffer
  drop_sgraphs(c);
  return build_out_ranges(c, st);
}

int64_t lbk_num_out(lbk_ctx* c) { return c ? c->nout : 0; }

// Exact zeros per block in the last factorization's output (export layout):
// the caller drops them like the reference's export (factorize.py:179-192)
// only where a block has any.
int lbk_export_zero_counts(lbk_ctx* c, int64_t* counts, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  const int64_t nb = static_cast<int64_t>(c->out_off.size());
  if (!c->zcount.p) {
    LBK_CUDA(c->zcount.alloc(std::max<int64_t>(nb, 1)), st);
    LBK_CUDA(c->out_off_d.upload([&] {
      std::vector<int64_t> o(c->out_off);
      o.push_back(c->nout);
      return o;
    }()), st);
  }
  if (nb) {
    zero_count_kernel<<<static_cast<int>(std::min<int64_t>(nb, 148 * 8)), 256, 0, c->stream>>>(c->vout.p, c->out_off_d.p,
                                                                                              nb, c->zcount.p);
    LBK_CUDA(cudaGetLastError(), st);
    LBK_CUDA(cudaMemcpyAsync(counts, c->zcount.p, nb * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream), st);
  }
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

// Working-layout values (every block's tile / CSC in pool block order).  In
// dense-scratch mode every block is a full column-major tile, so the caller
// can rebuild blocks whose support moved under row swaps (factorize.py:370-381).
int lbk_download_work(lbk_ctx* c, double* work, int64_t* nwork, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (nwork) *nwork = c->nnz_work;
  if (work) {
    LBK_CUDA(cudaStreamSynchronize(c->stream), st);  // the legacy-stream copy does not wait for it
    LBK_CUDA(cudaMemcpy(work, c->vals.p, c->nnz_work * sizeof(double), cudaMemcpyDeviceToHost), st);
  }
  ok(st);
  return 0;
}

int lbk_set_perms(lbk_ctx* c, const int32_t* perms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (c->ndiag_rows) {
    LBK_CUDA(cudaStreamSynchronize(c->stream), st);
    LBK_CUDA(cudaMemcpy(c->perm.p, perms, c->ndiag_rows * sizeof(int32_t), cudaMemcpyHostToDevice), st);
    LBK_CUDA(cudaDeviceSynchronize(), st);  // order the pageable copy before kernels on the engine streams
  }
  ok(st);
  return 0;
}

}  // extern "C"

namespace {

// Steps + update items of the forward (L, block rows ascending) and backward
// (U, descending) substitutions, and the graph that runs both.
int build_solve(lbk_ctx* c, lbk_status* st) {
  if (c->solve_graph) return 0;
  const int64_t p = c->p, nb = c->nblocks;
  std::vector<int64_t> bid(static_cast<size_t>(p * p), -1);
  for (int64_t b = 0; b < nb; ++b) bid[c->hbi[b] * p + c->hbj[b]] = b;
  std::vector<std::vector<int64_t>> bycol(p);
  for (int64_t b = 0; b < nb; ++b) bycol[c->hbj[b]].push_back(b);
  std::vector<SolveStep> fw, bw;
  std::vector<SolveUpd> uf, ub;
  int64_t maxspan = 1;
  // inverse diagonal tiles for the FULL diagonal blocks (cluster solve)
  std::vector<int64_t> tinv_off(p, -1);
  std::vector<int32_t> tistep, titile;
  int64_t ntinv = 0;
  for (int64_t i = 0; i < p; ++i) {
    const BlockDev& D = c->hblk[bid[i * p + i]];
    const int64_t span = c->pos[i + 1] - c->pos[i];
    if (D.store != STORE_FULL || span <= XT) continue;
    if (c->band_bl.size() == static_cast<size_t>(nb) && c->band_bl[bid[i * p + i]] >= 0) continue;  // band solve
    tinv_off[i] = ntinv;
    const int64_t nt = (span + XT - 1) / XT;
    for (int64_t t = 0; t < nt; ++t) {
      tistep.push_back(static_cast<int32_t>(i));  // forward steps are in block order
      titile.push_back(static_cast<int32_t>(t));
    }
    ntinv += nt * 2 * XT * XT;
  }
  auto items = [&](int64_t i, bool lower, std::vector<SolveUpd>* out) {
    for (int64_t b : bycol[i]) {
      const int64_t k = c->hbi[b];
      if (lower ? k <= i : k >= i) continue;
      const BlockDev& B = c->hblk[b];
      const int rows = B.store == STORE_SPARSE ? B.nrows : B.nR;
      for (int r0 = 0; r0 < rows; r0 += UPD_ROWS)
        out->push_back(SolveUpd{static_cast<int32_t>(b), static_cast<int32_t>(c->pos[k]),
                                static_cast<int32_t>(c->pos[i]), r0});
    }
  };
  for (int64_t q = 0; q < p; ++q) {
    for (int dir = 0; dir < 2; ++dir) {
      const int64_t i = dir == 0 ? q : p - 1 - q;
      SolveStep S{};
      S.diag = static_cast<int32_t>(bid[i * p + i]);
      S.off = static_cast<int32_t>(c->pos[i]);
      S.span = static_cast<int32_t>(c->pos[i + 1] - c->pos[i]);
      S.tinv = tinv_off[i];
      S.ext = c->dext_off[bid[i * p + i]];
      const int64_t db = bid[i * p + i];
      S.bl = S.bu = -1;
      S.nseg = 0;
      S.seg_off = 0;
      if (c->band_bl.size() == static_cast<size_t>(nb) && c->band_bl[db] >= 0) {
        S.bl = c->band_bl[db];
        S.bu = c->band_bu[db];
        S.seg_off = c->band_off[db];
        const int64_t next = [&] {  // segments of this block: up to the next block's offset
          int64_t e = static_cast<int64_t>(c->band_seg.size());
          for (int64_t b2 = 0; b2 < nb; ++b2)
            if (c->band_off[b2] > c->band_off[db]) e = std::min(e, c->band_off[b2]);
          return e;
        }();
        S.nseg = static_cast<int32_t>((next - S.seg_off) / 2);
      }
      maxspan = std::max<int64_t>(maxspan, S.span);
      std::vector<SolveUpd>* out = dir == 0 ? &uf : &ub;
      S.upd_off = static_cast<int64_t>(out->size());
      items(i, dir == 0, out);
      S.nupd = static_cast<int32_t>(out->size() - S.upd_off);
      (dir == 0 ? fw : bw).push_back(S);
    }
  }
  const size_t diag_smem = (static_cast<size_t>((maxspan + 1) & ~1LL) + SOLVE_CHUNK * 65) * sizeof(double);
  if (diag_smem > static_cast<size_t>(MAX_SMEM)) return fail(st, LBK_ERR_BAD_ARG, "block span too large for the solve");
  std::vector<int32_t> bstart(c->n);
  std::vector<int64_t> dgrow(c->n);
  for (int64_t i = 0; i < p; ++i) {
    const BlockDev& D = c->hblk[bid[i * p + i]];
    for (int64_t g = c->pos[i]; g < c->pos[i + 1]; ++g) {
      bstart[g] = static_cast<int32_t>(c->pos[i]);
      dgrow[g] = D.dg + (g - c->pos[i]);
    }
  }
  LBK_CUDA(c->sfw.upload(fw), st);
  LBK_CUDA(c->sbw.upload(bw), st);
  LBK_CUDA(c->ufw.upload(uf), st);
  LBK_CUDA(c->ubw.upload(ub), st);
  LBK_CUDA(c->sbstart.upload(bstart), st);
  LBK_CUDA(c->sdgrow.upload(dgrow), st);
  LBK_CUDA(c->sb.alloc(c->n), st);
  LBK_CUDA(c->sv.alloc(c->n), st);
  LBK_CUDA(c->tistep.upload(tistep), st);
  LBK_CUDA(c->sdext.upload(c->dext.empty() ? std::vector<int32_t>(2, 0) : c->dext), st);
  LBK_CUDA(c->titile.upload(titile), st);
  LBK_CUDA(c->sbandseg.upload(c->band_seg.empty() ? std::vector<int32_t>(2, 0) : c->band_seg), st);
  LBK_CUDA(c->stinv.alloc(std::max<int64_t>(ntinv, 1)), st);
  c->n_tinv = static_cast<int64_t>(tistep.size());
  DevPools P = pools(c);
  cudaStream_t s0 = c->stream;
  cudaGraph_t g;
  LBK_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal), st);
  solve_perm_kernel<<<148 * 4, 256, 0, s0>>>(c->sb.p, c->sv.p, c->perm.p, c->sbstart.p, c->sdgrow.p, c->n);
  if (c->n_tinv)
    tile_inverse_kernel<<<static_cast<int>(c->n_tinv), 256, (2 * XREG + XT) * sizeof(double), s0>>>(
        P, c->sfw.p, c->tistep.p, c->titile.p, c->stinv.p);
  for (int dir = 0; dir < 2; ++dir) {
    const std::vector<SolveStep>& steps = dir == 0 ? fw : bw;
    for (size_t q = 0; q < steps.size(); ++q) {
      const SolveStep& S = steps[q];
      const size_t sm = (static_cast<size_t>((S.span + 1) & ~1) + SOLVE_CHUNK * 65) * sizeof(double);
      if (S.bl >= 0 && S.nseg > 0) {
        const int W = std::max(S.bl, S.bu) + 1;
        solve_band_kernel<<<S.nseg, 256, (BAND_SOLVE_ROWS * (W + 1) + BAND_MAX) * sizeof(double), s0>>>(
            P, (dir == 0 ? c->sfw.p : c->sbw.p), static_cast<int>(q), c->sv.p, dir, c->sbandseg.p);
      } else if (S.tinv >= 0) {
        const int nch = (S.span + XT - 1) / XT, rpc = ((nch + SOLVE_CL - 1) / SOLVE_CL) * XT;
        if (LBK_SOLVE_FLAGS)
          solve_diag_flag_kernel<<<SOLVE_CL, 256, (rpc + 5 * XT + (nch + 1) / 2 + 1) * sizeof(double), s0>>>(
              P, (dir == 0 ? c->sfw.p : c->sbw.p), static_cast<int>(q), c->sv.p, dir, c->stinv.p, c->sdext.p);
        else
          solve_diag_cluster_kernel<<<SOLVE_CL, 256, (rpc + 7 * XT) * sizeof(double), s0>>>(
              P, (dir == 0 ? c->sfw.p : c->sbw.p), static_cast<int>(q), c->sv.p, dir, c->stinv.p, c->sdext.p);
      } else {
        solve_diag_kernel<<<1, 256, sm, s0>>>(P, (dir == 0 ? c->sfw.p : c->sbw.p), static_cast<int>(q), c->sv.p, dir);
      }
      if (S.nupd)
        solve_upd_kernel<<<S.nupd, 256, (static_cast<size_t>((S.span + 1) & ~1) + 256) * sizeof(double), s0>>>(
            P, (dir == 0 ? c->ufw.p : c->ubw.p) + S.upd_off, c->sv.p);
    }
  }
  cudaError_t e = cudaStreamEndCapture(s0, &g);
  if (e != cudaSuccess) return cuda_fail(st, e, "solve graph capture");
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaGraphInstantiate(&c->solve_graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(st, e, "solve graph");
  return 0;
}

}  // namespace

extern "C" {

// x = U^-1 L^-1 b[perm_global] on the factors of the last factorization
// (factorize.py:451-457); host vectors of length n in and out.
int lbk_solve(lbk_ctx* c, const double* b, double* x, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (build_solve(c, st)) return st->code;
  LBK_CUDA(cudaMemcpyAsync(c->sb.p, b, c->n * sizeof(double), cudaMemcpyHostToDevice, c->stream), st);
  LBK_CUDA(cudaGraphLaunch(c->solve_graph, c->stream), st);
  LBK_CUDA(cudaMemcpyAsync(x, c->sv.p, c->n * sizeof(double), cudaMemcpyDeviceToHost, c->stream), st);
  LBK_CUDA(cudaStreamSynchronize(c->stream), st);
  ok(st);
  return 0;
}

int lbk_host_alloc(void** ptr, int64_t bytes) {
  return cudaHostAlloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 1)), cudaHostAllocDefault) == cudaSuccess
             ? 0
             : LBK_ERR_OOM;
}

void lbk_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

// Per-level device times: one instrumented replay (external event record
// nodes around every level and every kernel family of the level);
// out_ms[nlevels x 5] = level, DMMA SSSSM, panel solves, tiled GETRF, CSC kernel.
int lbk_level_times(lbk_ctx* c, double pivot_tol, double static_eps, float* out_ms, lbk_status* st) {
  LBK_CUDA(cudaSetDevice(c->device), st);
  if (c->refined && !std::isnan(static_eps))
    return fail(st, LBK_ERR_BAD_ARG, "static pivoting needs a plan without segment-refined levels (lbk_plan flags bit 2)");
  const size_t nl = c->levels.size();
  std::vector<cudaEvent_t> ev(1 + nl * 13);
  for (auto& e : ev) LBK_CUDA(cudaEventCreate(&e), st);
  cudaGraph_t g;
  cudaGraphExec_t ge = nullptr;
  LBK_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), st);
  capture_factorization(c, pivot_tol, static_eps, &ev, 0, nl, true, true);
  LBK_CUDA(cudaStreamEndCapture(c->stream, &g), st);
  cudaError_t e = cudaGraphInstantiate(&ge, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(st, e, "instrumented graph");
  e = cudaGraphLaunch(ge, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  const bool exact = (c->flags & 2) != 0 || !std::isnan(static_eps);
  if (e == cudaSuccess)
    for (size_t l = 0; l < nl; ++l) {
      const Level& L = c->levels[l];
      const size_t b = 1 + l * 13, prev = l ? 1 + (l - 1) * 13 : 0;
      float* o = out_ms + l * 5;
      for (int k = 0; k < 5; ++k) o[k] = 0.f;
      cudaEventElapsedTime(&o[0], ev[prev], ev[b]);
      if (L.ngemm || L.ngemmD || L.ngemmE) cudaEventElapsedTime(&o[1], ev[b + 1], ev[b + 2]);
      if (L.npanel || (exact && L.nexact)) cudaEventElapsedTime(&o[2], ev[b + 3], ev[b + 4]);
      if (!exact && L.ntcol) cudaEventElapsedTime(&o[3], ev[b + 5], ev[b + 6]);
      if (L.nitems) cudaEventElapsedTime(&o[4], ev[b + 7], ev[b + 8]);
    }
  cudaGraphExecDestroy(ge);
  for (auto& x : ev) cudaEventDestroy(x);
  if (e != cudaSuccess) return cuda_fail(st, e, "instrumented replay");
  return finish(c, st);
}

// Executor timeline: one instrumented replay with per-task globaltimer stamps.
// trace[8 x n] = dequeue, ready (dependencies met), done, 4 in-task phase
// stamps (0 if unused), all writes fenced (ns); info[6 x n] =
// type, a, r, c, k, level.  *n = executor tasks (call with NULLs to size).
int lbk_exec_trace(lbk_ctx* c, double pivot_tol, double static_eps, uint64_t* trace, int32_t* info, int64_t* n,
                   lbk_status* st) {
  *n = c->n_exec;
  if (!trace || !info) {
    ok(st);
    return 0;
  }
  LBK_CUDA(cudaSetDevice(c->device), st);
  LBK_CUDA(c->xtrace.alloc(8 * std::max<int64_t>(c->n_exec, 1)), st);
  LBK_CUDA(cudaMemset(c->xtrace.p, 0, 8 * std::max<int64_t>(c->n_exec, 1) * 8), st);
  std::vector<float> lv(c->levels.size() * 5);
  const int rc = lbk_level_times(c, pivot_tol, static_eps, lv.data(), st);
  if (rc == LBK_ERR_CUDA || rc == LBK_ERR_OOM) return rc;
  LBK_CUDA(cudaMemcpy(trace, c->xtrace.p, 8 * c->n_exec * 8, cudaMemcpyDeviceToHost), st);
  std::vector<XTask> ht(c->n_exec);
  LBK_CUDA(cudaMemcpy(ht.data(), c->xtasks.p, c->n_exec * sizeof(XTask), cudaMemcpyDeviceToHost), st);
  for (size_t l = 0; l < c->levels.size(); ++l)
    for (int32_t q = 0; q < c->levels[l].nexec; ++q) {
      const int64_t t = c->levels[l].exec_off + q;
      const XTask& x = ht[t];
      int32_t* o = info + 6 * t;
      o[0] = x.type;
      o[1] = x.a;
      o[2] = x.r;
      o[3] = x.c;
      o[4] = x.k;
      o[5] = static_cast<int32_t>(l);
    }
  c->xtrace.release();
  ok(st);
  return 0;
}

// The executor's per-launch task DAG (analysis tooling): sptr[sum(nexec + 1)] = per launch level,
// local successor offsets; succ[*nsucc] = (local successor << 1) | phase.  NULL buffers: sizes only.
int lbk_exec_graph(lbk_ctx* c, int32_t* sptr, int32_t* succ, int64_t* nsptr, int64_t* nsucc) {
  *nsptr = static_cast<int64_t>(c->xsptr.n);
  *nsucc = static_cast<int64_t>(c->xsucc.n);
  if (!sptr || !succ) return 0;
  if (cudaSetDevice(c->device) != cudaSuccess) return LBK_ERR_CUDA;
  if (c->xsptr.n && cudaMemcpy(sptr, c->xsptr.p, c->xsptr.n * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LBK_ERR_CUDA;
  if (c->xsucc.n && cudaMemcpy(succ, c->xsucc.p, c->xsucc.n * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess)
    return LBK_ERR_CUDA;
  return 0;
}

// levels[4 x nlevels]: generic item offset, generic items, DMMA tiles, panel strips.
int lbk_plan_levels(lbk_ctx* c, int64_t* levels, int32_t* items) {
  const size_t nl = c->levels.size();
  for (size_t l = 0; l < nl; ++l) {
    levels[l] = c->levels[l].item_off;
    levels[nl + l] = c->levels[l].nitems;
    levels[2 * nl + l] = c->levels[l].ngemm;
    levels[3 * nl + l] = c->levels[l].npanel;
  }
  (void)items;
  return 0;
}

int lbk_task_routes(lbk_ctx* c, int8_t* route) {
  if (!c->route.empty()) std::memcpy(route, c->route.data(), c->route.size());
  return 0;
}

// info[0] levels, [1] generic items, [2] diagonal rows, [3] reference entries,
// [4] DMMA SSSSM tiles, [5] panel + exact items, [6] kernel launches per
// factorization (tiled path), [7] working entries, [8..10] SPARSE/RECT/FULL blocks,
// [11] tiled-GETRF items.
int lbk_plan_info(lbk_ctx* c, int64_t* info) {
  info[0] = static_cast<int64_t>(c->levels.size());
  info[1] = c->n_generic;
  info[2] = c->ndiag_rows;
  info[3] = c->nnz;
  info[4] = c->n_gemm;
  info[5] = c->n_panel;
  int64_t launches = 2;  // scatter + gather
  for (const Level& L : c->levels) {
    launches += (L.nitems > 0) + (L.ngemm > 0) + (L.ngemmD > 0) + (L.ngemmE > 0);
    if (c->use_exec) {
      launches += L.nexec > 0;
      continue;
    }
    launches += L.npanel > 0;
    if (L.ntcol) {
      launches += 2;
      for (int k = 0; k < L.nsub; ++k) {
        const SubStep& S = c->subs[L.sub_off + k];
        launches += (S.ngetrf > 0) + (S.ntrsm > 0) + (S.ngemm > 0);
      }
    }
  }
  info[6] = launches;
  info[7] = c->nnz_work;
  info[8] = c->store_count[0];
  info[9] = c->store_count[1];
  info[10] = c->store_count[2];
  info[11] = c->n_tile;
  info[12] = static_cast<int64_t>(c->dmma_flops);
  info[13] = static_cast<int64_t>(c->exec_flops);
  return 0;
}

}  // extern "C"
