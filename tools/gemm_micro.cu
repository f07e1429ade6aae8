// Standalone throughput of the DMMA SSSSM kernel (gemm_map_kernel) on dense FULL blocks:
// C (M x N) -= L (M x K) * U (K x N), 128 x 64 tiles, every inner chunk active, no gathers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/gemm_micro tools/gemm_micro.cu
//   /tmp/gemm_micro [M N K]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2512_04389_b200/csrc/lbk_dense.cuh"
using namespace lbk;

int main(int argc, char** argv) {
  const int M = argc > 3 ? atoi(argv[1]) : 4096, N = argc > 3 ? atoi(argv[2]) : 4096, K = argc > 3 ? atoi(argv[3]) : 2048;
  std::vector<BlockDev> hb(3);
  const size_t nL = size_t(M) * K, nU = size_t(K) * N, nC = size_t(M) * N;
  auto full = [](int r, int c, int64_t ent) {
    BlockDev b{};
    b.nrows = r; b.ncols = c; b.store = STORE_FULL; b.nR = r; b.nC = c; b.ent = ent;
    b.roff = b.coff = b.rp = b.csr = -1;
    return b;
  };
  hb[0] = full(M, K, 0);
  hb[1] = full(K, N, nL);
  hb[2] = full(M, N, nL + nU);
  GemmTask tk{0, 1, 2, K, -1, -1, -1, -1};
  std::vector<GemmItem> items;
  for (int n0 = 0; n0 < N; n0 += GBN)
    for (int m0 = 0; m0 < M; m0 += GBM) items.push_back(GemmItem{0, m0, n0, -1, 0, 0, (K + GBK - 1) / GBK, -1, 0});
  BlockDev* dblk; GemmTask* dtk; GemmItem* dit; double* vals;
  cudaMalloc(&dblk, 3 * sizeof(BlockDev));
  cudaMalloc(&dtk, sizeof(GemmTask));
  cudaMalloc(&dit, items.size() * sizeof(GemmItem));
  cudaMalloc(&vals, (nL + nU + nC) * sizeof(double));
  std::vector<double> hv(nL + nU + nC);
  for (size_t i = 0; i < hv.size(); ++i) hv[i] = 1e-3 * double((i * 7) % 13);
  cudaMemcpy(vals, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dblk, hb.data(), 3 * sizeof(BlockDev), cudaMemcpyHostToDevice);
  cudaMemcpy(dtk, &tk, sizeof(GemmTask), cudaMemcpyHostToDevice);
  cudaMemcpy(dit, items.data(), items.size() * sizeof(GemmItem), cudaMemcpyHostToDevice);
  DevPools P{};
  P.blk = dblk;
  P.vals = vals;
  cudaFuncSetAttribute(gemm_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) gemm_map_kernel<<<items.size(), 256, GEMM_SMEM>>>(dit, dtk, P);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) gemm_map_kernel<<<items.size(), 256, GEMM_SMEM>>>(dit, dtk, P);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms / reps * 1e-3;
  printf("M=%d N=%d K=%d tiles=%zu: %.3f ms  %.2f TFLOP/s (%s)\n", M, N, K, items.size(), t * 1e3,
         2.0 * M * N * K / t / 1e12, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
