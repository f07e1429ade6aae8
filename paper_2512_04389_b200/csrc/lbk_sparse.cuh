// lbk_sparse.cuh — warp-per-column / warp-per-row kernels on the CSC view.
//
// One warp owns one column (SSSSM, GESSM) or one row (TSTRF) of the output
// block and keeps a dense accumulator of the block's span in shared memory
// (scatter -> update -> gather, SPEC factorize DESIGN DECISIONS).  All
// updates into one accumulator are issued by one warp in the reference's
// order, so results are deterministic; GETRF/GESSM/TSTRF use separately
// rounded mul/sub and true division like the reference's numpy loops
// (factorize.py:38-130) and reproduce its bits on sparse blocks.

#pragma once

#include "lbk_common.cuh"

namespace lbk {

// C(k,j) -= L(k,i) U(i,j); Gustavson by target column (factorize.py:307-325).
// Latency hiding: the U entries of a column are read 32 at a time (lane q holds
// entry e0 + q: its row r, value u and L column bounds Lcp[r], Lcp[r+1], all in
// one round of loads), and the first 32 L entries of the next nonzero U entry
// are loaded before the current one is applied, so the warp no longer waits on
// three dependent global loads per U entry.  Updates into the accumulator are
// still applied one U entry at a time, in the column's order (deterministic).
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
    for (int e0 = u0; e0 < u1; e0 += 32) {
      const int cnt = min(32, u1 - e0);
      double mu = 0.0;
      int ml0 = 0, ml1 = 0;
      if (lane < cnt) {
        mu = Uv[e0 + lane];
        if (mu != 0.0) {  // exact-zero operand: no contribution
          const int r = Ur[e0 + lane];
          ml0 = Lcp[r];
          ml1 = Lcp[r + 1];
        }
      }
      // prefetch registers (pr, pv): the first 32 L entries of the next entry
      int pr = -1;
      double pv = 0.0;
      {
        const int l0 = __shfl_sync(0xffffffffu, ml0, 0), l1 = __shfl_sync(0xffffffffu, ml1, 0);
        if (l0 + lane < l1) {
          pr = Lr[l0 + lane];
          pv = Lv[l0 + lane];
        }
      }
      for (int q = 0; q < cnt; ++q) {
        const double u = __shfl_sync(0xffffffffu, mu, q);
        const int l0 = __shfl_sync(0xffffffffu, ml0, q), l1 = __shfl_sync(0xffffffffu, ml1, q);
        const int cr = pr;
        const double cv = pv;
        // next entry's loads in flight while this one is applied
        const int qn = q + 1 < cnt ? q + 1 : q;
        const int n0 = __shfl_sync(0xffffffffu, ml0, qn), n1 = __shfl_sync(0xffffffffu, ml1, qn);
        pr = -1;
        if (q + 1 < cnt && n0 + lane < n1) {
          pr = Lr[n0 + lane];
          pv = Lv[n0 + lane];
        }
        if (u == 0.0) continue;  // warp-uniform
        if (cr >= 0) acc[cr] = fma(cv, u, acc[cr]);
        for (int f = l0 + 32 + lane; f < l1; f += 32) acc[Lr[f]] = fma(Lv[f], u, acc[Lr[f]]);
        __syncwarp();
      }
    }
    for (int e = c0 + lane; e < c1; e += 32) Cv[e] -= acc[Cr[e]];
    __syncwarp();
  }
}

// X(i,j) <- L_ii^{-1} P_i X(i,j); one warp per column of X (factorize.py:98-109).
__device__ void gessm_item(const Item& it, const DevPools& P, double* acc) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* Dcp = P.colptr + D.cp;
  const int32_t* Dr = P.rows + D.ent;
  const double* Dv = P.vals + D.ent;
  const int32_t* perm = P.perm + D.dg;
  const int32_t* Xcp = P.colptr + X.cp;
  const int32_t* Xr = P.rows + X.ent;
  double* Xv = P.vals + X.ent;
  const bool dfull = D.store == STORE_FULL;
  const int m = D.nrows;
  const bool permute = (it.c != 0) && X.store == STORE_FULL;
  for (int c = it.begin + warp; c < it.end; c += nw) {
    const int x0 = Xcp[c], x1 = Xcp[c + 1];
    if (x0 == x1) continue;
    if (permute) {
      for (int e = x0 + lane; e < x1; e += 32) acc[Xr[e]] = Xv[x0 + perm[Xr[e]]];
    } else {
      for (int e = x0 + lane; e < x1; e += 32) acc[Xr[e]] = Xv[e];
    }
    __syncwarp();
    if (dfull) {
      // dense L_ii: restrict the solve to X's own rows (the result pattern is
      // closed under L, so other rows stay exactly zero)
      for (int e = x0; e < x1; ++e) {
        const int k = Xr[e];
        const double xk = acc[k];
        const double* lk = Dv + static_cast<size_t>(k) * m;
        for (int f = e + 1 + lane; f < x1; f += 32) {
          const int q = Xr[f];
          acc[q] = dsub_mul(acc[q], lk[q], xk);
        }
        __syncwarp();
      }
    } else {
      // sparse L_ii: the column bounds of 32 entries per round of loads, the first 32
      // entries of the next column prefetched while the current one is applied
      const int32_t* dpos = P.diag_csc + D.dg;
      for (int e0 = x0; e0 < x1; e0 += 32) {
        const int cnt = min(32, x1 - e0);
        int mk = 0, mf0 = 0, mf1 = 0;
        if (lane < cnt) {
          mk = Xr[e0 + lane];
          mf0 = dpos[mk] + 1;
          mf1 = Dcp[mk + 1];
        }
        int pq = -1;
        double pd = 0.0;
        {
          const int f0 = __shfl_sync(0xffffffffu, mf0, 0), f1 = __shfl_sync(0xffffffffu, mf1, 0);
          if (f0 + lane < f1) {
            pq = Dr[f0 + lane];
            pd = Dv[f0 + lane];
          }
        }
        for (int q = 0; q < cnt; ++q) {
          const int k = __shfl_sync(0xffffffffu, mk, q);
          const int f0 = __shfl_sync(0xffffffffu, mf0, q), f1 = __shfl_sync(0xffffffffu, mf1, q);
          const int cq = pq;
          const double cd = pd;
          const int qn = q + 1 < cnt ? q + 1 : q;
          const int n0 = __shfl_sync(0xffffffffu, mf0, qn), n1 = __shfl_sync(0xffffffffu, mf1, qn);
          pq = -1;
          if (q + 1 < cnt && n0 + lane < n1) {
            pq = Dr[n0 + lane];
            pd = Dv[n0 + lane];
          }
          const double xk = acc[k];
          if (cq >= 0) acc[cq] = dsub_mul(acc[cq], cd, xk);
          for (int f = f0 + 32 + lane; f < f1; f += 32) {
            const int r = Dr[f];
            acc[r] = dsub_mul(acc[r], Dv[f], xk);
          }
          __syncwarp();
        }
      }
    }
    for (int e = x0 + lane; e < x1; e += 32) Xv[e] = acc[Xr[e]];
    __syncwarp();
  }
}

// X(k,i) <- X(k,i) U_ii^{-1}; one warp per row of X via its CSR index (factorize.py:112-130).
__device__ void tstrf_item(const Item& it, const DevPools& P, double* acc) {
  const BlockDev D = P.blk[it.a], X = P.blk[it.b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Dv = P.vals + D.ent;
  const int32_t* Xrp = P.csr_ptr + X.rp;
  const int32_t* Xcc = P.csr_col + X.csr;
  const int32_t* Xcpos = P.csr_pos + X.csr;
  double* Xv = P.vals + X.ent;
  const bool dfull = D.store == STORE_FULL;
  const int m = D.nrows;
  for (int q = it.begin + warp; q < it.end; q += nw) {
    const int r0 = Xrp[q], r1 = Xrp[q + 1];
    if (r0 == r1) continue;
    for (int e = r0 + lane; e < r1; e += 32) acc[Xcc[e]] = Xv[Xcpos[e]];
    __syncwarp();
    if (dfull) {
      for (int e = r0; e < r1; ++e) {
        const int k = Xcc[e];
        const double xk = __ddiv_rn(acc[k], Dv[static_cast<size_t>(k) * m + k]);
        __syncwarp();
        if (lane == 0) acc[k] = xk;
        for (int f = e + 1 + lane; f < r1; f += 32) {
          const int j = Xcc[f];
          acc[j] = dsub_mul(acc[j], xk, Dv[static_cast<size_t>(j) * m + k]);
        }
        __syncwarp();
      }
    } else {
      const int32_t* Dcsc = P.diag_csc + D.dg;
      const int32_t* Drow = P.diag_csr + D.dg;
      const int32_t* Drp = P.csr_ptr + D.rp;
      const int32_t* Dcc = P.csr_col + D.csr;
      const int32_t* Dcpos = P.csr_pos + D.csr;
      for (int e0 = r0; e0 < r1; e0 += 32) {
        const int cnt = min(32, r1 - e0);
        int mk = 0, mg0 = 0, mg1 = 0;
        double mdiag = 1.0;
        if (lane < cnt) {
          mk = Xcc[e0 + lane];
          mdiag = Dv[Dcsc[mk]];
          mg0 = Drow[mk] + 1;
          mg1 = Drp[mk + 1];
        }
        int pj = -1;
        double pu = 0.0;
        {
          const int g0 = __shfl_sync(0xffffffffu, mg0, 0), g1 = __shfl_sync(0xffffffffu, mg1, 0);
          if (g0 + lane < g1) {
            pj = Dcc[g0 + lane];
            pu = Dv[Dcpos[g0 + lane]];
          }
        }
        for (int q = 0; q < cnt; ++q) {
          const int k = __shfl_sync(0xffffffffu, mk, q);
          const double dkk = __shfl_sync(0xffffffffu, mdiag, q);
          const int g0 = __shfl_sync(0xffffffffu, mg0, q), g1 = __shfl_sync(0xffffffffu, mg1, q);
          const int cj = pj;
          const double cu = pu;
          const int qn = q + 1 < cnt ? q + 1 : q;
          const int n0 = __shfl_sync(0xffffffffu, mg0, qn), n1 = __shfl_sync(0xffffffffu, mg1, qn);
          pj = -1;
          if (q + 1 < cnt && n0 + lane < n1) {
            pj = Dcc[n0 + lane];
            pu = Dv[Dcpos[n0 + lane]];
          }
          const double xk = __ddiv_rn(acc[k], dkk);
          __syncwarp();
          if (lane == 0) acc[k] = xk;
          if (cj >= 0) acc[cj] = dsub_mul(acc[cj], xk, cu);
          for (int g = g0 + 32 + lane; g < g1; g += 32) {
            const int j = Dcc[g];
            acc[j] = dsub_mul(acc[j], xk, Dv[Dcpos[g]]);
          }
          __syncwarp();
        }
      }
    }
    for (int e = r0 + lane; e < r1; e += 32) Xv[Xcpos[e]] = acc[Xcc[e]];
    __syncwarp();
  }
}

// Left-looking LU of a SPARSE diagonal block (all-sparse mode): the CTA
// owns the block, warps take the columns of one intra-block level at a time.
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
      } else if (brow != c && lane == 0) {
        record(&P.err[1], step, c);  // sparse storage cannot represent the swap
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

__global__ void __launch_bounds__(256) level_kernel(const Item* __restrict__ items, DevPools P, int acc_len,
                                                    double pivot_tol, double static_eps) {
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

// I/O between the reference layout (pool order of the filled pattern) and
// the working layout: work[map[e]] = in[e] / out[e] = work[map[e]].
// nonfinite: set when an input value is inf / NaN (its products may reach
// positions outside the pattern: the pool is then zeroed before the next run).
__global__ void scatter_kernel(const double* __restrict__ in, const int64_t* __restrict__ map,
                               double* __restrict__ work, int64_t n, int* nonfinite) {
  bool bad = false;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = in[e];
    bad |= !isfinite(v);
    const int64_t m = map[e];
    if (m >= 0) work[m] = v;  // -2: block without storage on this rank (distributed plans)
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *nonfinite = 1;
}

// work[0, n) = 0 when dirty[0] is set (grid-stride, 16-byte stores); a no-op launch otherwise
__global__ void zero_if_dirty_kernel(double* __restrict__ work, int64_t n, const int* dirty) {
  if (*reinterpret_cast<const volatile int*>(dirty) == 0) return;
  const int64_t n2 = n / 2;
  double2* w2 = reinterpret_cast<double2*>(work);  // cudaMalloc'd: 256-byte aligned
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    w2[e] = make_double2(0.0, 0.0);
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) work[n - 1] = 0.0;
}

// end of a run: the next run zeroes the pool iff this one recorded an error
// (err words start at ~0) or read a non-finite input
__global__ void mark_dirty_kernel(const unsigned long long* err, int* dirty) {
  if (threadIdx.x == 0) {
    dirty[0] = (err[0] != ~0ULL || err[1] != ~0ULL || dirty[1] != 0) ? 1 : 0;
    dirty[1] = 0;
  }
}

// ranges[2 x n] = (offset, length) of reference-pool entries to gather (one CTA
// per range, strided).
__global__ void range_gather_kernel(const double* __restrict__ work, const int64_t* __restrict__ map,
                                    double* __restrict__ out, const int64_t* __restrict__ ranges, int64_t n) {
  for (int64_t q = blockIdx.x; q < n; q += gridDim.x) {
    const int64_t off = ranges[2 * q], len = ranges[2 * q + 1];
    for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
      const int64_t m = map[off + e];
      out[off + e] = m >= 0 ? work[m] : (m == -1 ? 1.0 : 0.0);  // -1: unit diagonal of an exported L block
    }
  }
}

// in[pos[k]] = a[k]: A's entries into the reference pool (refactorization input)
__global__ void expand_kernel(const double* __restrict__ a, const int64_t* __restrict__ pos, double* __restrict__ in,
                              int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    in[pos[k]] = a[k];
}

__global__ void gather_kernel(const double* __restrict__ work, const int64_t* __restrict__ map,
                              double* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = map[e];
    out[e] = m >= 0 ? work[m] : (m == -1 ? 1.0 : 0.0);  // -2: no storage on this rank
  }
}

// omap[x] = xref[x] < 0 ? -1 : map[xref[x]]  (export layout -> working positions)
__global__ void compose_map_kernel(const int64_t* __restrict__ xref, const int64_t* __restrict__ map,
                                   int64_t* __restrict__ omap, int64_t n) {
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < n;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = xref[x];
    omap[x] = r < 0 ? -1 : map[r];  // (map -2 stays -2)
  }
}

// zc[b] = number of exact zeros in out[off[b], off[b+1]) (one CTA per block, strided)
__global__ void zero_count_kernel(const double* __restrict__ out, const int64_t* __restrict__ off, int64_t nb,
                                  int64_t* __restrict__ zc) {
  __shared__ int part[8];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int cnt = 0;
    const int64_t e1 = off[b + 1];
    for (int64_t e = off[b] + threadIdx.x; e < e1; e += blockDim.x) cnt += out[e] == 0.0;
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
      zc[b] = t;
    }
    __syncthreads();
  }
}

}  // namespace lbk
