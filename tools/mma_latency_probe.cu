// Microbenchmark + layout probe (dev tool):
//  1. latency of a chain of N dependent tcgen05.mma (M=128/64, N=32, K=16, bf16) into one
//     accumulator vs N independent accumulators (issue -> commit -> mbarrier observed);
//  2. whether a K-major no-swizzle A operand with LBO = SBO = 0 (one 128-byte core matrix
//     of ones re-read everywhere) yields D = column sums of B.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "ptx.cuh"
using namespace mlra;

__global__ void lat_kernel(long long* out, float* colsum_out, const __nv_bfloat16* P) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* a_buf = dsm;            // 16 KB
  uint8_t* b_buf = dsm + 16384;    // 32 KB (N up to 256 rows of 128 B)
  __shared__ __align__(128) uint8_t ones[128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_sh;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(a_buf)[i] = 0x3c003c00u * 0;
  for (int i = tid; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(b_buf)[i] = 0;
  if (tid < 64) reinterpret_cast<__nv_bfloat16*>(ones)[tid] = __float2bfloat16(1.f);
  // P [128 tok x 32 heads] -> MN-major interleave (as in the decode kernel), SBO = 16*128
  for (int idx = tid; idx < 128 * 4; idx += blockDim.x) {
    int t = idx / 4, g = idx % 4;
    *reinterpret_cast<uint4*>(b_buf + g * 2048 + (t / 8) * 128 + (t % 8) * 16) =
        *reinterpret_cast<const uint4*>(P + t * 32 + g * 8);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase_sh);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_sh;
  uint32_t phase = 0;
  if (tid == 0) {
    const uint64_t adesc = make_sdesc(smem_u32(a_buf), 16, 1024, kSw128);
    const uint64_t bdesc_k = make_sdesc(smem_u32(b_buf), 16, 1024, kSw128);
    int k = 0;
    for (int M : {128, 64}) {
      const uint32_t idesc = make_idesc_bf16(M, 32, false, false);
      for (int n : {1, 2, 4, 8, 12, 16, 32}) {
        for (int indep = 0; indep < 2; ++indep) {
          long long t0 = clock64();
          for (int i = 0; i < n; ++i) mma_bf16_ss(tb + (indep ? (i % 8) * 32 : 0), adesc, bdesc_k, idesc, i > 0);
          mma_commit(&bar);
          mbar_wait(&bar, phase);
          phase ^= 1;
          long long t1 = clock64();
          out[k++] = t1 - t0;
        }
      }
    }
    // N sweep: chain of 8 dependent MMAs, M=128, A/B from smem (B rows beyond 32 read garbage)
    for (int N : {16, 32, 64, 128, 256}) {
      const uint32_t idesc = make_idesc_bf16(128, N, false, false);
      long long t0 = clock64();
      for (int i = 0; i < 8; ++i) mma_bf16_ss(tb, adesc, bdesc_k, idesc, i > 0);
      mma_commit(&bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
      out[k++] = clock64() - t0;
    }
    // A from TMEM (ts): A tile [128 x 16] bf16 lives in TMEM cols [384, 392)
    for (int N : {32, 128, 256}) {
      const uint32_t idesc = make_idesc_bf16(128, N, false, false);
      long long t0 = clock64();
      for (int i = 0; i < 8; ++i)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     :: "r"(tb), "r"(tb + 384), "l"(bdesc_k), "r"(idesc), "r"(i > 0 ? 1 : 0) : "memory");
      mma_commit(&bar);
      mbar_wait(&bar, phase);
      phase ^= 1;
      out[k++] = clock64() - t0;
    }
    // ones-A column sums: M=64, K = 128 tokens (8 x K16), B = P MN-major interleave
    const uint64_t a1 = make_sdesc(smem_u32(ones), 0, 0, kSwNone);
    const uint32_t idesc64 = make_idesc_bf16(64, 32, false, true);
    for (int i = 0; i < 8; ++i)
      mma_bf16_ss(tb + 256, a1, make_sdesc(smem_u32(b_buf) + i * 256, 128, 2048, kSwNone), idesc64, i > 0);
    mma_commit(&bar);
    mbar_wait(&bar, phase);
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t r[32];
    tmem_ld16(tb + 256, r);
    tmem_ld16(tb + 256 + 16, r + 16);
    tmem_ld_wait();
    for (int c = 0; c < 32; ++c) colsum_out[lane_id() * 32 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  long long* d_out;
  float* d_cs;
  __nv_bfloat16* d_p;
  std::vector<__nv_bfloat16> hp(128 * 32);
  std::vector<float> pf(128 * 32);
  for (int i = 0; i < 128 * 32; ++i) {
    pf[i] = float((i * 37) % 11) * 0.125f;
    hp[i] = __float2bfloat16(pf[i]);
  }
  cudaMalloc(&d_out, 64 * 8);
  cudaMalloc(&d_cs, 32 * 32 * 4);
  cudaMalloc(&d_p, hp.size() * 2);
  cudaMemcpy(d_p, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 60000);
  lat_kernel<<<1, 128, 49152 + 1024>>>(d_out, d_cs, d_p);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  long long h[64];
  cudaMemcpy(h, d_out, 64 * 8, cudaMemcpyDeviceToHost);
  int k = 0;
  for (int M : {128, 64})
    for (int n : {1, 2, 4, 8, 12, 16, 32}) {
      printf("M=%d N=32 chain=%2d dependent %6lld cyc   independent %6lld cyc\n", M, n, h[k], h[k + 1]);
      k += 2;
    }
  for (int N : {16, 32, 64, 128, 256}) printf("SS M=128 N=%3d chain=8: %6lld cyc\n", N, h[k++]);
  for (int N : {32, 128, 256}) printf("TS M=128 N=%3d chain=8: %6lld cyc\n", N, h[k++]);
  std::vector<float> cs(32 * 32);
  cudaMemcpy(cs.data(), d_cs, cs.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int c = 0; c < 32; ++c) {
    double s = 0;
    for (int t = 0; t < 128; ++t) s += pf[t * 32 + c];
    for (int lane = 0; lane < 16; ++lane) err = fmax(err, fabs(s - cs[lane * 32 + c]));
  }
  printf("ones-A (LBO=SBO=0) column-sum max err %.3e (%s)\n", err, err < 1e-3 ? "OK" : "FAIL");
  return 0;
}
