// Standalone timing of the executor's tile routines (cycles per call, one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2512_04389_b200/csrc/lbk_exec.cuh"
using namespace lbk;

__global__ void k_mma(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* C = sm; double* A = sm + XREG; double* B = sm + 2 * XREG;
  for (int i = threadIdx.x; i < 3 * XREG; i += blockDim.x) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) tile_mma_sub(C, A, B);
  long long t1 = clock64();
  out[blockIdx.x * 4096 + threadIdx.x] = C[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}

__global__ void k_lub(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* T = sm; double* Dd = sm + XREG; double* rinv = sm + 2 * XREG;
  long long tot = 0;
  __shared__ long long prof[4];
  if (threadIdx.x < 4) prof[threadIdx.x] = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) T[i] = (i % 65 == i / 65) ? 100.0 : 1e-3 * ((i * 7) % 13);
    __syncthreads();
    long long t0 = clock64();
    tile_lu64_blocked(T, 64, Dd, rinv, blockIdx.x == 0 ? prof : nullptr);
    tot += clock64() - t0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    printf("lu64_blocked phases per call: panel %lld  U12 %lld  A22 %lld  sync %lld cycles\n", prof[0] / iters,
           prof[1] / iters, prof[2] / iters, prof[3] / iters);
  out[blockIdx.x * 4096 + threadIdx.x] = T[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

__global__ void k_rblk(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* X = sm; double* U = sm + XREG; double* rinv = sm + 3 * XREG; double* Dd = sm + 2 * XREG;
  for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) U[i] = 1.0 + 1e-3 * ((i * 7) % 13);
  if (threadIdx.x < 64) rinv[threadIdx.x] = 0.9;
  long long tot = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) X[i] = 1e-3 * (i % 11);
    __syncthreads();
    long long t0 = clock64();
    tile_right_solve_blk<true>(X, U, rinv, Dd, 64);
    tot += clock64() - t0;
  }
  out[blockIdx.x * 4096 + threadIdx.x] = X[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

__global__ void k_lblk(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* X = sm; double* L = sm + XREG;
  for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) L[i] = 1e-3 * ((i * 7) % 13);
  long long tot = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) X[i] = 1e-3 * (i % 11);
    __syncthreads();
    long long t0 = clock64();
    tile_left_solve_blk(X, L, 64);
    tot += clock64() - t0;
  }
  out[blockIdx.x * 4096 + threadIdx.x] = X[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

int main() {
  double* out; long long* cyc; long long h[148];
  cudaMalloc(&out, 148 * 4096 * 8); cudaMalloc(&cyc, 148 * 8);
  int smem = EXEC_SMEM;
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_lub, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_rblk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_lblk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"tile_mma_sub", "tile_lu64_blocked", "tile_right_solve_blk", "tile_left_solve_blk"};
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      if (k == 0) k_mma<<<148, 256, smem>>>(out, 200, cyc);
      if (k == 1) k_lub<<<148, 256, smem>>>(out, 20, cyc);
      if (k == 2) k_rblk<<<148, 256, smem>>>(out, 20, cyc);
      if (k == 3) k_lblk<<<148, 256, smem>>>(out, 20, cyc);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double o[256], sum = 0.0;
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 256; ++i) sum += o[i] * (1.0 + 1e-3 * i);
    printf("%-22s %8lld cycles/call (%.2f us at 1.965 GHz)  checksum %.15e err=%s\n", names[k], h[0], h[0] / 1965.0,
           sum, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
