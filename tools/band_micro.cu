// Band sweep variants on one CTA, timed with clock64: the executor's
// barrier-stepped narrow sweep (band_getrf) vs the single-thread register
// window (band_getrf_reg), same full-band diagonally dominant m x m block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2512_04389_b200/csrc -o tools/band_micro tools/band_micro.cu
#include <cstdio>
#include <vector>
#include <cmath>
#include "lbk_common.cuh"
#include "lbk_exec.cuh"

namespace lbk {
__global__ void __launch_bounds__(256) k_old(BlockDev A, DevPools P, int bw, int m, long long* cyc) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  band_getrf(A, P, sm, bw, bw, 0, m, 0, 0.1);
  if (threadIdx.x == 0) *cyc = clock64() - t0;
}
__global__ void __launch_bounds__(256) k_reg(BlockDev A, DevPools P, int bw, int m, long long* cyc) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  if (bw == 4) band_getrf_reg<4>(A, P, sm, 0, m, 0, 0.1);
  if (threadIdx.x == 0) *cyc = clock64() - t0;
}
}  // namespace lbk

int main() {
  using namespace lbk;
  const int m = 4000;
  for (int bw : {4}) {
    std::vector<double> h(static_cast<size_t>(m) * m, 0.0);
    unsigned s = 12345;
    auto rnd = [&] { s = s * 1664525u + 1013904223u; return (s >> 8) / double(1 << 24) - 0.5; };
    for (int c = 0; c < m; ++c)
      for (int r = std::max(0, c - bw); r <= std::min(m - 1, c + bw); ++r) h[size_t(c) * m + r] = r == c ? 4.0 * (bw + 1) : rnd();
    double *vals, *colmax, *out[2];
    unsigned long long* err;
    long long* cyc;
    cudaMalloc(&vals, h.size() * 8);
    cudaMalloc(&colmax, m * 8);
    cudaMalloc(&err, 16);
    cudaMallocManaged(&cyc, 16);
    for (int v = 0; v < 2; ++v) {
      cudaMemcpy(vals, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      cudaMemset(err, 0xff, 16);
      BlockDev A{};
      A.nrows = A.ncols = m; A.ent = 0; A.dg = 0;
      DevPools P{};
      P.vals = vals; P.colmax = colmax; P.err = err;
      cudaFuncSetAttribute(k_old, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM);
      cudaFuncSetAttribute(k_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, EXEC_SMEM);
      if (v == 0) k_old<<<1, 256, EXEC_SMEM>>>(A, P, bw, m, cyc);
      else k_reg<<<1, 256, EXEC_SMEM>>>(A, P, bw, m, cyc);
      cudaDeviceSynchronize();
      out[v] = new double[h.size()];
      cudaMemcpy(out[v], vals, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long e[2];
      cudaMemcpy(e, err, 16, cudaMemcpyDeviceToHost);
      printf("bw=%d %s: %.1f cycles/column  err %llx %llx  (%s)\n", bw, v ? "reg " : "old ", double(cyc[0]) / m, e[0], e[1],
             cudaGetErrorString(cudaGetLastError()));
    }
    double md = 0;
    for (size_t i = 0; i < h.size(); ++i) md = std::max(md, std::fabs(out[0][i] - out[1][i]));
    printf("bw=%d max |old - reg| = %g\n", bw, md);
    cudaFree(vals); cudaFree(colmax); cudaFree(err);
  }
  return 0;
}
