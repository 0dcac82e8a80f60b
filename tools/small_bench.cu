// Dev tool: timing of the small step kernels (K1 absorb4, K3 combine4) in isolation,
// back-to-back launches on one stream, CUDA events; B=16, H=24, DH=128, DLAT=128, nsplit=9.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2603_02188_b200/csrc small_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "aux_kernels.cuh"
using namespace mlra;

__global__ void empty_kernel() {}


int main() {
  const int B = 16, H = 24, DH = 128, DLAT = 128, DR = 64, nsplit = 9;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t cs0;
  cudaStreamCreate(&cs0);
  auto timeit = [&](const char* name, auto&& fn) {
    // graph of 20 launches on a capturing stream (fn launches on the legacy stream -> use
    // global capture mode with the per-thread default redirected: launch fn inside capture)
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(cs0, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 20; ++i) fn();
    cudaStreamEndCapture(cs0, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, cs0);
    cudaStreamSynchronize(cs0);
    cudaEventRecord(e0, cs0);
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, cs0);
    cudaEventRecord(e1, cs0);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.2f us/launch graph-replayed (%s)\n", name, ms * 1e3 / 200, cudaGetErrorString(cudaGetLastError()));
  };
  timeit("empty <<<1,32>>>", [&] { empty_kernel<<<1, 32, 0, cs0>>>(); });
  timeit("empty <<<384,128>>>", [&] { empty_kernel<<<384, 128, 0, cs0>>>(); });
  for (int NB : {1, 4}) {
    const int NCOL = NB * DLAT;
    __nv_bfloat16 *qn, *qr, *wuk, *qabs, *qrs, *wuv;
    float *opart, *lse, *out;
    cudaMalloc(&qn, B * H * DH * 2);
    cudaMalloc(&qr, B * H * DR * 2);
    cudaMalloc(&wuk, size_t(H) * DH * NCOL * 2);
    cudaMalloc(&wuv, size_t(H) * NCOL * DH * 2);
    cudaMalloc(&qabs, size_t(B) * NB * H * DLAT * 2);
    cudaMalloc(&qrs, B * H * DR * 2);
    cudaMalloc(&opart, size_t(B) * nsplit * NB * H * DLAT * 4);
    cudaMalloc(&lse, size_t(B) * nsplit * NB * H * 4);
    cudaMalloc(&out, size_t(B) * NB * H * DH * 4);
    cudaMemset(qn, 0, B * H * DH * 2);
    cudaMemset(wuk, 0, size_t(H) * DH * NCOL * 2);
    cudaMemset(wuv, 0, size_t(H) * NCOL * DH * 2);
    cudaMemset(opart, 0, size_t(B) * nsplit * NB * H * DLAT * 4);
    cudaMemset(lse, 0, size_t(B) * nsplit * NB * H * 4);
    char nm[128];
    snprintf(nm, sizeof nm, "absorb4 NB=%d grid(%d,%d,%d)", NB, (NCOL + 127) / 128, H, (B + 3) / 4);
    timeit(nm, [&] {
      absorb4_kernel<<<dim3((NCOL + 127) / 128, H, (B + 3) / 4), kG4Threads, absorb4_smem(), cs0>>>(qn, wuk, qabs, B, H, DH,
                                                                                                  NB, DLAT, 1.f, qr, qrs, DR);
    });
    for (int seqs : {4, 8}) {
      auto kern = seqs == 4 ? combine4_kernel<4> : combine4_kernel<8>;
      const size_t cs = seqs == 4 ? combine4_smem<4>(DLAT, DH, nsplit) : combine4_smem<8>(DLAT, DH, nsplit);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
      for (int cl : {0, 1}) {
        if (cl && NB == 1) continue;
        snprintf(nm, sizeof nm, "combine4<%d> NB=%d %s", seqs, NB, cl ? "cluster-sum" : "per-branch");
        timeit(nm, [&] {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3((B + seqs - 1) / seqs, H, NB);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = cs;
          cfg.stream = cs0;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeClusterDimension;
          attr[0].val.clusterDim.x = 1;
          attr[0].val.clusterDim.y = 1;
          attr[0].val.clusterDim.z = cl ? NB : 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, kern, (const float*)opart, (const float*)lse, (const __nv_bfloat16*)wuv, out, B, H, NB,
                             DLAT, DH, nsplit, 0.5f, cl ? 0 : 1, TpSum{});
        });
      }
    }
  }
  return 0;
}
