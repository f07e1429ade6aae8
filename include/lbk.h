/* lbk.h — C ABI of the B200 block-LU engine (paper_2512_04389_b200).
 *
 * The reference (lublock 0.1.0, pure Python) has no FFI: its boundary is the
 * Python API of module lublock.factorize (pkg/src/lublock/__init__.py:33-42).
 * Every entry point below replaces one reference function; the mapping is
 * given next to each declaration.  Plain pointers and sizes only: no C++ or
 * torch types cross this boundary, no exceptions, no exit().  Every function
 * returns an lbk status code (0 = OK); device functions additionally fill an
 * lbk_status record with the failing block/column.
 *
 * Two shared objects implement it:
 *   liblbk_host.so  — structure path (symbolic, partition, levels), CPU
 *   liblbk.so       — device engine (sm_100a CUDA kernels + scheduler)
 */
#ifndef LBK_H_
#define LBK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map onto pkg/src/lublock/errors.py) ------------------ */
#define LBK_OK 0
#define LBK_ERR_ZERO_PIVOT 1        /* errors.ZeroPivot(block, col)        errors.py:66-75 */
#define LBK_ERR_SUPPORT 2           /* errors.SupportViolation             errors.py:78-82 */
#define LBK_ERR_DIM_MISMATCH 3      /* errors.DimensionMismatch            errors.py:43-44 */
#define LBK_ERR_CUDA 4              /* CUDA runtime failure (msg holds cudaGetErrorString) */
#define LBK_ERR_NCCL 5              /* NCCL failure */
#define LBK_ERR_OOM 6               /* host or device allocation failure */
#define LBK_ERR_PIVOT_SWAP 7        /* a diagonal block needs a row swap while its block row
                                       is stored sparse: the wrapper re-runs in dense mode */
#define LBK_ERR_BAD_ARG 8           /* errors.BadParams */

typedef struct lbk_status {
  int32_t code;
  int32_t block; /* ZeroPivot: diagonal block index (lowest failing one) */
  int32_t col;   /* ZeroPivot: local column inside that block          */
  int32_t pad;
  char msg[256];
} lbk_status;

/* ======================================================================== *
 * Host structure path (liblbk_host.so).  Large outputs: count first, the
 * caller allocates, fill writes straight into the caller's buffers.
 * ======================================================================== */

/* symbolic_factorize(a_sym) -> FilledPattern        symbolic.py:57-108
 * Input: symmetrized CSC (col_ptr[n+1], row_idx[nnz], sorted rows).
 * nnz: *nnz_filled = nnz(L+L^T+I).  fill: col_ptr[n+1], row_idx[nnz_filled]
 * (col,row)-sorted; parent[n] = elimination tree (may be NULL). */
int lbk_symbolic_nnz(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* nnz_filled);
int lbk_symbolic_fill(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* out_col_ptr,
                      int64_t* out_row_idx, int64_t* parent);

/* diag_block_pointer(f).blockptr (Alg. 2)             features.py:44-54
 * blockptr[n+1]; the pattern must be symmetric with a full diagonal. */
int lbk_blockptr(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* blockptr);

/* _require_symmetric_full_diag(col_ptr, row_idx, n)     symbolic.py:46-54
 * 0 = ok, 1 = missing diagonal (*ndiag = count), 2 = not symmetric,
 * 3 = rows not strictly increasing within a column. */
int lbk_check_symmetric(int64_t n, const int64_t* col_ptr, const int64_t* row_idx, int64_t* ndiag);

/* partition(f, a, plan) -> BlockGrid                 grid.py:85-148
 * count: number of stored blocks and pooled col_ptr length.  fill: block
 * table (7 x nblocks, row-major by field: bi, bj, nrows, ncols, nnz,
 * colptr_offset, entry_offset) in column-major block order (the reference
 * dict order), pooled local col_ptr, local row_idx and values (A's values
 * scattered, 0.0 at fill), block_nnz[p*p] row-major.  Returns
 * LBK_ERR_DIM_MISMATCH if A is not covered by the filled pattern. */
int lbk_partition_count(int64_t n, const int64_t* f_col_ptr, const int64_t* f_row_idx, int64_t p,
                        const int64_t* positions, int64_t* nblocks, int64_t* colptr_len);
int lbk_partition_fill(int64_t n, const int64_t* f_col_ptr, const int64_t* f_row_idx,
                       const int64_t* a_col_ptr, const int64_t* a_row_idx, const double* a_values,
                       int64_t p, const int64_t* positions, int64_t nblocks, int64_t* table,
                       int64_t* col_ptr, int64_t* row_idx, double* values, int64_t* block_nnz,
                       int64_t* a_pos /* nullable: int64[nnz(A)], pool position of each entry of A */);

/* dependency_levels(grid) -> DependencyTree            grid.py:223-378 */
int lbk_levels_run(int64_t p, int64_t nblocks, const int64_t* table, const int64_t* col_ptr,
                   const int64_t* row_idx, void** handle, int64_t* ntasks, int64_t* npreds);
int lbk_levels_fetch(void* handle, int8_t* kinds, int32_t* steps, int32_t* rows, int32_t* cols,
                     int64_t* weights, int64_t* costs, int32_t* levels, int64_t* pred_ptr,
                     int32_t* pred_idx);
void lbk_levels_free(void* handle);

/* ======================================================================== *
 * Device engine (liblbk.so).  One lbk_ctx per GPU.  Replaces
 *   lublock.factorize.factorize(grid, tree, workers, pivot_tol,
 *                               static_pivot, dense_blas)   factorize.py:245-384
 * split into plan (structure, once) + numeric (values, every call), the way
 * a refactorization with a fixed pattern is driven.
 * ======================================================================== */
typedef struct lbk_ctx lbk_ctx;

int lbk_create(lbk_ctx** ctx, int device, lbk_status* st);
void lbk_destroy(lbk_ctx* ctx);

/* Upload the block structure (the pooled BlockGrid of lbk_partition_fetch:
 * table[7 x nblocks], local col_ptr pool, local row_idx pool) and the
 * DependencyTree arrays (grid.py:172-181); builds the per-level work lists
 * (items of `chunk` columns/rows) and the CUDA graph lazily.
 * flags bit 0: DMMA storage — diagonal blocks become full dense tiles (tiled
 *   multi-CTA GETRF) and every block whose nonempty-rows x nonempty-columns
 *   rectangle holds >= tau of its entries becomes a compressed dense tile
 *   (SSSSM/GESSM/TSTRF on FP64 tensor cores); other blocks stay CSC;
 * flags bit 1: dense-scratch mode — every block a full tile, true row swaps
 *   (the reference's dense scratch, factorize.py:265);
 * flags bit 2: segment-refined levels — banded diagonal blocks are swept per
 *   independent segment, and updates into them, their sweeps and the panels
 *   reading them wait only for the segments involved (the reference's block
 *   DAG, grid.py:223-378, refined; bitwise the same factors).  Such a plan
 *   rejects static pivoting (LBK_ERR_BAD_ARG): plan without bit 2 for it. */
int lbk_plan(lbk_ctx* ctx, int64_t n, int64_t p, const int64_t* positions, int64_t nblocks,
             const int64_t* table, const int64_t* col_ptr, const int64_t* row_idx, int64_t ntasks,
             const int8_t* kinds, const int32_t* steps, const int32_t* rows, const int32_t* cols,
             const int32_t* levels, const int64_t* costs, int32_t chunk, int32_t flags, double tau,
             lbk_status* st);

/* Pristine A values in pool order, kept resident on the device. */
int lbk_upload_values(lbk_ctx* ctx, const double* values, lbk_status* st);

/* Device-resident factorization of the resident A values (reset + level
 * graph).  static_eps = NaN disables static pivoting (factorize.py:267-269).
 * *ms = device time of the level graph.  ZeroPivot -> LBK_ERR_ZERO_PIVOT
 * with st->block/col = the lowest failing (block, local column). */
int lbk_factorize(lbk_ctx* ctx, double pivot_tol, double static_eps, float* ms, lbk_status* st);

/* End-to-end: host A values in, host factor values (pool order, in place of
 * A's pattern) and per-diagonal-row local permutations out.  With a page-
 * locked lu_values buffer (lbk_host_alloc / cudaHostRegister) every block's
 * factor values are gathered and copied to the host on a copy stream as soon
 * as the level that finishes the block is done, overlapping the rest of the
 * factorization (one cached graph per output buffer). */
int lbk_factorize_host(lbk_ctx* ctx, const double* a_values, double* lu_values, int32_t* perms,
                       double pivot_tol, double static_eps, lbk_status* st);

/* Refactorization input (new values on A's pattern, KLU-style refactor):
 * lbk_bind_matrix gives the reference-pool position of every entry of A in
 * CSC order (grid.pool_positions); lbk_refactor_host then takes A's nnz values
 * instead of the whole pool (fill entries are zero) and is otherwise
 * lbk_factorize_host. */
int lbk_bind_matrix(lbk_ctx* ctx, int64_t nnz_a, const int64_t* pool_pos, lbk_status* st);
int lbk_refactor_host(lbk_ctx* ctx, const double* a_values, double* lu_values, int32_t* perms, double pivot_tol,
                      double static_eps, lbk_status* st);

/* Output layout of the drop-in factorize() (paper_2512_04389_b200/numeric.py):
 * the LUFactors blocks exactly as the reference exports them
 * (pkg/src/lublock/factorize.py:370-384: off-diagonal blocks as stored,
 * diagonal blocks split into triu(d) and tril(d,-1)+I).  nout output entries,
 * block b (pool order) in [xoff[b], xoff[b+1]); xref[x] = reference-pool
 * entry of output entry x, or -1 for a constant 1.0 (unit diagonal).  Every
 * later lbk_factorize_host / lbk_refactor_host / lbk_download writes this
 * layout (nout entries, lbk_num_out). */
int lbk_set_export(lbk_ctx* ctx, int64_t nout, const int64_t* xref, const int64_t* xoff, lbk_status* st);
int64_t lbk_num_out(lbk_ctx* ctx);

/* Exact zeros per block (int64[nblocks]) in the last factorization's output:
 * the reference's export drops exact zeros (factorize.py:179-192); a caller
 * compacts only the blocks that have any. */
int lbk_export_zero_counts(lbk_ctx* ctx, int64_t* counts, lbk_status* st);

/* Copy the last factorization's values / perms to the host. */
int lbk_download(lbk_ctx* ctx, double* lu_values, int32_t* perms, lbk_status* st);

/* Working-layout values of the last factorization (*nwork entries; pass
 * work = NULL to query the size).  In dense-scratch mode every block is a
 * full column-major tile in pool block order: the caller rebuilds blocks
 * whose support moved under row swaps (factorize.py:370-381). */
int lbk_download_work(lbk_ctx* ctx, double* work, int64_t* nwork, lbk_status* st);

/* Overwrite the per-diagonal-row permutations (pool order of the diagonal
 * blocks).  Used by the kernel-level entry points factor_u_panel
 * (factorize.py:150-156), which take an explicit perm_i, when the plan
 * holds no GETRF task to produce it. */
int lbk_set_perms(lbk_ctx* ctx, const int32_t* perms, lbk_status* st);

/* Page-locked host memory for the end-to-end path. */
int lbk_host_alloc(void** ptr, int64_t bytes);
void lbk_host_free(void* ptr);

/* info[14]: [0] launched levels, [1] CSC work items, [2] diagonal rows,
 * [3] reference entries, [4] DMMA SSSSM tiles, [5] panel/exact items,
 * [6] kernel launches per factorization, [7] working entries, [8..10]
 * SPARSE/RECT/FULL blocks, [11] tiled-GETRF items, [12] executed DMMA
 * SSSSM flops (tile rectangles, structural zeros included), [13] executed
 * flops of the tile-DAG executor (64^3-tile equivalents). */
int lbk_plan_info(lbk_ctx* ctx, int64_t* info);

/* Per task of the DependencyTree: the kernel family that executes it
 * (-1 skipped: zero-work update; 0 CSC kernel; 1 DMMA SSSSM; 2 panel solve;
 * 3 tiled GETRF).  route[ntasks]. */
int lbk_task_routes(lbk_ctx* ctx, int8_t* route);

/* FP64 throughput microbenchmark (register-resident DMMA.8x8x4 and DFMA
 * loops on every SM): the dense-block roofline denominator, which
 * MEASURED_PEAKS.json does not carry.  TFLOP/s out. */
int lbk_fp64_peak(int device, double* tflops_dmma, double* tflops_dfma);

/* One instrumented replay: device ms of every launched level and of each
 * kernel family inside it, out_ms[nlevels x 5] = level, DMMA SSSSM, panel
 * solves, tiled GETRF, CSC kernel (load-balance evidence next to
 * metrics.level_work_stats, pkg/src/lublock/metrics.py:63-90). */
int lbk_level_times(lbk_ctx* ctx, double pivot_tol, double static_eps, float* out_ms, lbk_status* st);

/* Persistent-executor timeline of one instrumented replay: trace[8 x n] =
 * dequeue / dependencies-met / done, four in-task phase stamps and the
 * time its phase-2 operands were complete (ns, globaltimer) per tile task,
 * info[6 x n] = type, block, r, c, k, level.  Pass NULL buffers to get *n. */
int lbk_exec_trace(lbk_ctx* ctx, double pivot_tol, double static_eps, uint64_t* trace, int32_t* info,
                   int64_t* n, lbk_status* st);

/* The executor's task DAG behind lbk_exec_trace (analysis tooling): per launch
 * level, nexec + 1 local successor offsets in sptr and (local successor << 1 |
 * phase) entries in succ.  Pass NULL buffers to get *nsptr / *nsucc. */
int lbk_exec_graph(lbk_ctx* ctx, int32_t* sptr, int32_t* succ, int64_t* nsptr, int64_t* nsucc);

/* ---- 2D block-cyclic distribution (north-star subsystem 5; no reference
 * counterpart: SPEC.md:14 scopes multi-process mapping out).  Owner-computes:
 * each rank plans only the tasks whose written block it owns
 * (paper_2512_04389_b200/parallel.py task_owners) and the graph is cut into
 * segments after the tree levels whose finished blocks other ranks read; the
 * host moves those blocks between segments (NCCL point-to-point on the
 * ctx stream) and then launches the next segment.  Both calls precede lbk_plan. */
int lbk_set_task_mask(lbk_ctx* ctx, int64_t ntasks, const int8_t* mask, lbk_status* st);
int lbk_set_cuts(lbk_ctx* ctx, int64_t nlevels, const int8_t* cut_after, lbk_status* st);
int lbk_num_segments(lbk_ctx* ctx);
/* Enqueue segment `seg` on the ctx stream (asynchronous; seg 0 also zeroes and
 * scatters, the last one gathers into the output pool). */
int lbk_run_segment(lbk_ctx* ctx, int32_t seg, double pivot_tol, double static_eps, lbk_status* st);
/* Synchronize; *ms = device time from segment 0 to the last segment;
 * err2 = the raw (block << 32 | col) words of a zero pivot / needed row swap
 * (~0 = none), to be min-reduced across ranks and decoded by lbk_status_from_err. */
int lbk_finish_raw(lbk_ctx* ctx, float* ms, uint64_t* err2, lbk_status* st);
int lbk_status_from_err(const uint64_t* err2, lbk_status* st);
/* The ctx stream (cudaStream_t) and device pointers of the working pool, the
 * per-diagonal-row permutations and the output pool, for the block exchange. */
void* lbk_stream(lbk_ctx* ctx);
int lbk_work_ptrs(lbk_ctx* ctx, void** vals, void** perm, void** vout);
/* layout[3 x nblocks]: working-pool offset, working entries, diagonal-row
 * offset (-1 for off-diagonal blocks), in pool block order. */
int lbk_block_layout(lbk_ctx* ctx, int64_t* layout);

/* Cross-level lookahead: defer[t] = 1 marks a task whose successors all sit
 * >= 2 ASAP levels later (computed from DependencyTree.pred_ptr/pred_idx,
 * grid.py:172-181).  Its DMMA SSSSM tiles run on a side branch concurrently
 * with the next level; the level two later waits for them.  Call before
 * lbk_plan; NULL clears. */
int lbk_set_task_defer(lbk_ctx* ctx, int64_t ntasks, const int8_t* defer, lbk_status* st);

/* Device triangular solve on the factors of the last lbk_factorize /
 * lbk_factorize_host of this ctx: x = U^-1 L^-1 b[perm_global]
 * (factorize.py:451-457; L, U = the blocks LUFactors exports, :370-384).
 * Blocked column-oriented substitution (one launch per diagonal block and
 * one per block column of updates, graph-captured); b, x: host, length n. */
int lbk_solve(lbk_ctx* ctx, const double* b, double* x, lbk_status* st);

/* Launched-level table (4 x nlevels: item offset, items, warps, acc length)
 * and, if items != NULL, the work items (6 x total: kind, a, b, c, begin, end). */
int lbk_plan_levels(lbk_ctx* ctx, int64_t* levels, int32_t* items);

#ifdef __cplusplus
}
#endif

#endif /* LBK_H_ */
