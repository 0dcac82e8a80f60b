// Dev probe: the fused step's absorb unit (fused_step.cuh fused_absorb) alone, 256 threads per
// CTA, one unit per CTA, globaltimer stamps per phase. nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_2603_02188_b200/csrc/fused_step.cuh"
using namespace mlra;
__global__ void __launch_bounds__(256) probe(FuseArgs f, int B, int H, int DR, unsigned long long* ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  fused_absorb(f, B, H, DR, blockIdx.x, gridDim.x, threadIdx.x, sm);
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) { ts[2 * blockIdx.x] = t0; ts[2 * blockIdx.x + 1] = t1; }
}
int main() {
  const int B = 16, H = 24, DH = 128, NB = 1, DLAT = 128, DR = 64;
  __nv_bfloat16 *q, *qr, *w, *qa, *qrs;
  cudaMalloc(&q, B * H * DH * 2); cudaMalloc(&qr, B * H * DR * 2); cudaMalloc(&w, H * DH * NB * DLAT * 2);
  cudaMalloc(&qa, B * NB * H * DLAT * 2); cudaMalloc(&qrs, B * H * DR * 2);
  cudaMemset(q, 0, B * H * DH * 2); cudaMemset(w, 0, H * DH * NB * DLAT * 2); cudaMemset(qr, 0, B * H * DR * 2);
  uint32_t* sync; cudaMalloc(&sync, 4096); cudaMemset(sync, 0, 4096);
  unsigned long long* ts; cudaMalloc(&ts, 8 * 1024);
  FuseArgs f = {};
  f.q_nope = q; f.q_rope = qr; f.w_uk = w; f.q_abs = qa; f.q_rope_s = qrs; f.sync = sync;
  f.score_scale = 1.f; f.DH = DH; f.NB = NB; f.DLAT = DLAT;
  int units = absorb_units(B, H, NB, DLAT);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 5; ++it) {
    cudaMemset(sync, 0, 4096);
    cudaEventRecord(e0);
    probe<<<units, 256, absorb_smem_bytes(DH)>>>(f, B, H, DR, ts);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(2 * units);
    cudaMemcpy(h.data(), ts, 16 * units, cudaMemcpyDeviceToHost);
    unsigned long long mn = ~0ull, mx = 0;
    for (int i = 0; i < units; ++i) { mn = std::min(mn, h[2 * i]); mx = std::max(mx, h[2 * i + 1]); }
    printf("units %d: event %.2f us, first start -> last end %.2f us, cta0 %.2f us\n", units, ms * 1e3,
           (mx - mn) / 1e3, (h[1] - h[0]) / 1e3);
  }
  return 0;
}
