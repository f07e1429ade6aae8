// Standalone timing of the executor's tile routines (cycles per call, one CTA per SM).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2512_04389_b200/csrc/lbk_exec.cuh"
using namespace lbk;

__global__ void k_left(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* Lm = sm;
  for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) Lm[i] = 1e-3 * ((i * 7) % 13);
  __syncthreads();
  Line X;
  for (int i = 0; i < 16; ++i) X.x[i] = 1.0 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) line_left_unit_lower(X, 64, Lm);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 16; ++i) s += X.x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}

__global__ void k_right(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* U = sm; double* rinv = sm + XREG; unsigned long long* cm = (unsigned long long*)(sm + XREG + XT);
  double* Dd = sm + 2 * XREG;
  for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) U[i] = 1.0 + 1e-3 * ((i * 7) % 13);
  __syncthreads();
  prep_right(U, 64, rinv, cm);
  __syncthreads();
  Line X;
  for (int i = 0; i < 16; ++i) X.x[i] = 1.0 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) line_right_upper<true>(X, 64, 64, U, rinv, Dd);
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < 16; ++i) s += X.x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}

__global__ void k_lu(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* urow = sm; double* Dd = sm + XREG;
  long long tot = 0;
  Line X;
  for (int it = 0; it < iters; ++it) {
    for (int i = 0; i < 16; ++i) X.x[i] = ((threadIdx.x >> 2) == 4 * i + (threadIdx.x & 3)) ? 100.0 : 1e-3 * i;
    __syncthreads();
    long long t0 = clock64();
    line_lu(X, 64, urow, Dd);
    tot += clock64() - t0;
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += X.x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

__global__ void k_mma(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* C = sm; double* A = sm + XREG; double* B = sm + 2 * XREG;
  for (int i = threadIdx.x; i < 3 * XREG; i += blockDim.x) sm[i] = 1e-3 * (i % 17);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) tile_mma_sub(C, A, B);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = C[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}

int main() {
  double* out; long long* cyc; long long h[148];
  cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 148 * 8);
  int smem = EXEC_SMEM;
  cudaFuncSetAttribute(k_left, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_right, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"line_left_unit_lower", "line_right_upper", "line_lu", "tile_mma_sub"};
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      if (k == 0) k_left<<<148, 256, smem>>>(out, 50, cyc);
      if (k == 1) k_right<<<148, 256, smem>>>(out, 50, cyc);
      if (k == 2) k_lu<<<148, 256, smem>>>(out, 20, cyc);
      if (k == 3) k_mma<<<148, 256, smem>>>(out, 200, cyc);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s %8lld cycles/call (%.2f us at 1.965 GHz)  err=%s\n", names[k], h[0], h[0] / 1965.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
