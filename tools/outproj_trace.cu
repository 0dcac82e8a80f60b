// Dev tool: per-CTA phase stamps (clock64) of K4, world 1. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02188_b200/csrc outproj_trace.cu -o outproj_trace
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ long long g_op_trace[4096 * 8];
#define MLRA_OP_STAMP(k)                                                                                  \
  do {                                                                                                    \
    if (threadIdx.x == 0) g_op_trace[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + (k)] = clock64();        \
  } while (0)
#include "outproj_kernel.cuh"
using namespace mlra;

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 16, K = argc > 2 ? atoi(argv[2]) : 3072, D = argc > 3 ? atoi(argv[3]) : 3072;
  const int KS = argc > 4 ? atoi(argv[4]) : 6;
  float *attn, *gate, *y, *resid;
  __nv_bfloat16* w;
  cudaMalloc(&attn, size_t(B) * K * 4); cudaMalloc(&gate, size_t(B) * K * 4);
  cudaMalloc(&y, size_t(B) * D * 4); cudaMalloc(&resid, size_t(B) * D * 4);
  cudaMalloc(&w, size_t(K) * D * 2);
  cudaMemset(attn, 0, size_t(B) * K * 4); cudaMemset(gate, 0, size_t(B) * K * 4); cudaMemset(w, 0, size_t(K) * D * 2);
  __nv_bfloat16* a;
  cudaMalloc(&a, size_t(B) * K * 2);
  cudaMemset(a, 0, size_t(B) * K * 2);
  OutProjParams p = {};
  p.a[0] = a; p.w_o[0] = w; p.y[0] = y; p.resid = resid;
  p.B = B; p.K = K; p.D = D; p.world = 1; p.rank0 = 0; p.nslabs = outproj_nslabs(D); p.ks_count = KS;
  p.k_slice = ((K + KS - 1) / KS + 63) / 64 * 64;
  const size_t smem = outproj_smem();
  cudaFuncSetAttribute(outproj_allreduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(p.nslabs * KS, 1); cfg.blockDim = dim3(kOpThreads); cfg.dynamicSmemBytes = smem;
  attr[0].id = cudaLaunchAttributeClusterDimension; attr[0].val.clusterDim.x = KS; attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1; cfg.attrs = attr; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 5; ++i) cudaLaunchKernelEx(&cfg, outproj_allreduce_kernel, p);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, outproj_allreduce_kernel, p);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("B=%d K=%d D=%d KS=%d grid %d: %.2f us (%s)\n", B, K, D, KS, p.nslabs * KS, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  const int n = p.nslabs * KS;
  std::vector<long long> t(size_t(n) * 8);
  cudaMemcpyFromSymbol(t.data(), g_op_trace, t.size() * 8);
  printf("cta: first-chunk  main-loop  reduce  cluster  epilogue (cycles from stamp 0)\n");
  for (int c = 0; c < n; c += (n > 8 ? n / 8 : 1))
    printf("%3d: %6lld %6lld %6lld %6lld %6lld\n", c, t[c * 8 + 1] - t[c * 8], t[c * 8 + 2] - t[c * 8], t[c * 8 + 3] - t[c * 8],
           t[c * 8 + 4] - t[c * 8], t[c * 8 + 5] - t[c * 8]);
  return 0;
}
