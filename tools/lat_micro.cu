// Dependent-chain latencies on one warp (cycles per op): DFMA, DMUL, rcp_fast
// (MUFU.RCP64H + 2 Newton steps + range fixups), LDS.64, SHFL of a double,
// STS->__syncwarp->LDS round trip.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  r = fabs(x) < 1e-300 ? copysign(__longlong_as_double(0x7ff0000000000000LL), x) : r;
  return isinf(x) ? copysign(0.0, x) : r;
}

__global__ void lat(double* out, long long* cyc, int n, double seed) {
  __shared__ double sh[64];
  const int lane = threadIdx.x;
  sh[lane] = seed + lane;
  __syncwarp();
  double x = seed + lane * 1e-9;
  long long t0, t1;
  // DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999999, 1e-7);
  t1 = clock64(); if (lane == 0) cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); if (lane == 0) cyc[1] = t1 - t0;
  // rcp_fast
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rcp_fast(x) + 1e-12;
  t1 = clock64(); if (lane == 0) cyc[2] = t1 - t0;
  // MUFU only
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
  t1 = clock64(); if (lane == 0) cyc[3] = t1 - t0;
  // LDS pointer chase (index from value)
  int idx = lane;
  volatile double* vs = sh;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = vs[idx]; idx = (static_cast<int>(v) + 1) & 31; }
  t1 = clock64(); if (lane == 0) cyc[4] = t1 - t0;
  x += idx;
  // SHFL double
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64(); if (lane == 0) cyc[5] = t1 - t0;
  // STS -> syncwarp -> LDS (value produced by another lane)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (lane == (i & 31)) vs[32] = x + 1.0;
    __syncwarp();
    x = vs[32];
    __syncwarp();
  }
  t1 = clock64(); if (lane == 0) cyc[6] = t1 - t0;
  // DMUL+DFMA+rcp chain typical of one band column (l = d * rcp(u); u' = a - l * b)
  double u = 3.0 + lane * 1e-9;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { const double l = 0.5 * rcp_fast(u); u = fma(-l, 0.25, 3.0 + u * 1e-9); }
  t1 = clock64(); if (lane == 0) cyc[7] = t1 - t0;
  out[lane] = x + u;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8); cudaMallocManaged(&cyc, 16 * 8);
  const int n = 4096;
  lat<<<1, 32>>>(out, cyc, n, 1.5);
  lat<<<1, 32>>>(out, cyc, n, 1.5);
  cudaDeviceSynchronize();
  const char* nm[] = {"DFMA", "DMUL", "rcp_fast", "MUFU.RCP64H", "LDS chase", "SHFL f64", "STS->syncwarp->LDS", "band column chain (rcp,mul,fma)"};
  for (int i = 0; i < 8; ++i) printf("%-34s %7.1f cycles\n", nm[i], double(cyc[i]) / n);
  return 0;
}
