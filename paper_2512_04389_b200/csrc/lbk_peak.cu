// lbk_peak.cu — FP64 throughput microbenchmark for the roofline denominator.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the dense-block
// roofline of this engine is the FP64 tensor pipe (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4) and, for comparison, plain DFMA.  Both loops keep their
// operands in registers (no memory traffic) with enough independent chains
// per warp to cover the pipe latency.

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/lbk.h"

namespace {

__global__ void __launch_bounds__(256) dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" int lbk_fp64_peak(int device, double* tflops_dmma, double* tflops_dfma) {
  if (cudaSetDevice(device) != cudaSuccess) return LBK_ERR_CUDA;
  (void)cudaGetLastError();  // clear a stale (non-sticky) error left by an earlier call
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return LBK_ERR_OOM;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, iters = 4096;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dmma_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  // per warp per iteration: 8 DMMA of 8x8x4 = 8 * 512 flops
  const double warps = blocks * 8.0;
  *tflops_dmma = warps * iters * 8 * 512.0 / (best * 1e-3) / 1e12;
  best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  *tflops_dfma = blocks * 256.0 * iters * 8 * 2.0 / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : LBK_ERR_CUDA;
}
