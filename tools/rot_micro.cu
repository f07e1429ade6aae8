// Cycles per call of the rotated-line tile solvers (tools/rot_tiles.cuh), one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "rot_tiles.cuh"
using namespace lbk;

__global__ void __launch_bounds__(256) k_rright(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* U = sm + XREG; double* rinv = sm + 3 * XREG; double* Dd = sm + 2 * XREG;
  for (int i = threadIdx.x; i < XREG; i += blockDim.x) U[i] = 1.0 + 1e-3 * ((i * 7) % 13);
  if (threadIdx.x < XT) rinv[threadIdx.x] = 0.9;
  __syncthreads();
  long long tot = 0;
  double* G = out + blockIdx.x * 4096;
  for (int it = 0; it < iters; ++it) {
    double x[XT];
    if (threadIdx.x < XT) {
#pragma unroll
      for (int c = 0; c < XT; ++c) x[c] = 1e-3 * (c + threadIdx.x);
      long long t0 = clock64();
      rot_right_upper<true>(x, 64, U, rinv, Dd, G, 64, true);
      tot += clock64() - t0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

__global__ void __launch_bounds__(256) k_rleft(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* X = sm; double* L = sm + XREG;
  for (int i = threadIdx.x; i < XREG; i += blockDim.x) L[i] = 1e-3 * ((i * 7) % 13);
  __syncthreads();
  long long tot = 0;
  for (int it = 0; it < iters; ++it) {
    for (int i = threadIdx.x; i < XT * XTP; i += blockDim.x) X[i] = 1e-3 * (i % 11);
    __syncthreads();
    long long t0 = clock64();
    left_solve_rot(X, L, 64);
    tot += clock64() - t0;
  }
  out[blockIdx.x * 4096 + threadIdx.x] = X[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

__global__ void __launch_bounds__(256) k_rlu(double* out, int iters, long long* cyc) {
  extern __shared__ double sm[];
  double* R = sm; double* Dd = sm + XREG; double* rinv = sm + 3 * XREG;
  long long tot = 0;
  double* G = out + blockIdx.x * 4096;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x < XT) {
      double x[XT];
#pragma unroll
      for (int c = 0; c < XT; ++c) x[c] = (c == threadIdx.x) ? 100.0 : 1e-3 * c;
      long long t0 = clock64();
      rot_lu(x, 64, R, rinv, Dd, G, 64);
      tot += clock64() - t0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / iters;
}

int main() {
  double* out; long long* cyc; long long h[148];
  cudaMalloc(&out, 148 * 4096 * 8); cudaMalloc(&cyc, 148 * 8);
  int smem = EXEC_SMEM;
  cudaFuncSetAttribute(k_rright, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_rleft, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_rlu, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"rot_right_upper", "left_solve_rot", "rot_lu"};
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      if (k == 0) k_rright<<<148, 256, smem>>>(out, 20, cyc);
      if (k == 1) k_rleft<<<148, 256, smem>>>(out, 20, cyc);
      if (k == 2) k_rlu<<<148, 256, smem>>>(out, 20, cyc);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-22s %8lld cycles/call (%.2f us at 1.965 GHz)  err=%s\n", names[k], h[0], h[0] / 1965.0,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
