// Dev tool: phase stamps (globaltimer) of K3 combine4<4> (cluster branch sum), B=16, H=24, NB=4.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02188_b200/csrc k3_trace.cu -o k3_trace
#define MLRA_SMALL_TRACE 1
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
#include "aux_kernels.cuh"
using namespace mlra;
template <int SEQS>
int run(int NB) {
  const int B = 16, H = 24, DH = 128, DLAT = 128, nsplit = 9;
  __nv_bfloat16* wuv; float *opart, *lse, *out;
  cudaMalloc(&wuv, size_t(H) * NB * DLAT * DH * 2);
  cudaMalloc(&opart, size_t(B) * nsplit * NB * H * DLAT * 4);
  cudaMalloc(&lse, size_t(B) * nsplit * NB * H * 4);
  cudaMalloc(&out, size_t(B) * H * DH * 4);
  cudaMemset(wuv, 0, size_t(H) * NB * DLAT * DH * 2); cudaMemset(opart, 0, size_t(B) * nsplit * NB * H * DLAT * 4);
  cudaMemset(lse, 0, size_t(B) * nsplit * NB * H * 4);
  auto kern = combine4_kernel<SEQS>;
  const size_t cs = combine4_smem<SEQS>(DLAT, DH, nsplit);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((B + SEQS - 1) / SEQS, H, NB); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = cs;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension; attr[0].val.clusterDim.x = 1; attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = NB; cfg.attrs = attr; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, kern, (const float*)opart, (const float*)lse, (const __nv_bfloat16*)wuv, out, B, H, NB, DLAT, DH, nsplit, 0.5f, 0, TpSum{}, (int*)nullptr, (const int32_t*)nullptr);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern, (const float*)opart, (const float*)lse, (const __nv_bfloat16*)wuv, out, B, H, NB, DLAT, DH, nsplit, 0.5f, 0, TpSum{}, (int*)nullptr, (const int32_t*)nullptr);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const int n = ((B + SEQS - 1) / SEQS) * H * NB;
  std::vector<unsigned long long> t(size_t(n) * 8);
  cudaMemcpyFromSymbol(t.data(), g_small_trace, t.size() * 8);
  unsigned long long t0 = ~0ull, tend = 0;
  for (int c = 0; c < n; ++c) { t0 = std::min(t0, t[c * 8]); tend = std::max(tend, t[c * 8 + 5]); }
  printf("combine4<%d> NB=%d: %.2f us event, first start -> last end %.2f us (%s)\n", SEQS, NB, ms * 1e3, (tend - t0) / 1e3,
         cudaGetErrorString(cudaGetLastError()));
  printf("cta: start  wbar-issued  merge-done  w-landed  gemm+quarters  end   (ns from first CTA start)\n");
  for (int c = 0; c < n; c += n / 12)
    printf("%3d: %6llu %6llu %6llu %6llu %6llu %6llu\n", c, t[c * 8] - t0, t[c * 8 + 1] - t0, t[c * 8 + 2] - t0,
           t[c * 8 + 3] - t0, t[c * 8 + 4] - t0, t[c * 8 + 5] - t0);
  return 0;
}
int main() {
  run<4>(4);  // TP1 (B = 16: four sequences per CTA -- the production variant there)
  run<2>(4);
  run<2>(1);  // TP4 rank
  return 0;
}
