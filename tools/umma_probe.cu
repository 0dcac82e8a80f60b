// Layout probe for the tcgen05 operand encodings the decode kernel relies on.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2603_02188_b200/csrc tools/umma_probe.cu -o probe
// Checks, against a CPU fp32 product on the same bf16 data:
//   QK  : D[tok, head] = KV[tok, 0:192] . Q[head, 0:192]       A K-major SW128 (TMA), B K-major SW128 (manual)
//         for M = 128 and M = 64 (TMEM lane map m0 + 32*m1)
//   PV  : D[lat, head] = sum_tok KV[tok, lat] . P[tok, head]    A MN-major SW128 (TMA), B MN-major no-swizzle
//         for M = 128 (two 64-col chunks via LBO) and M = 64
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "ptx.cuh"

using namespace mlra;

constexpr int ROWS = 128, W = 192, NP = 32;

__global__ void __launch_bounds__(128, 1)
probe_kernel(const __grid_constant__ CUtensorMap kv_map, const __nv_bfloat16* __restrict__ Q,
             const __nv_bfloat16* __restrict__ P, float* out_qk128, float* out_qk64, float* out_pv128,
             float* out_pv64) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kv = smem;                      // 3 chunks x [128 rows x 128 B] = 48 KB
  uint8_t* qs = smem + 3 * 16384;          // 3 chunks x [32 rows x 128 B] = 12 KB
  uint8_t* ps = qs + 3 * 4096;             // P [128 tok x 32 heads] MN-major interleave = 8 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;

  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  // Q: K-major SW128 rows of 128 B; 16-byte unit j of row r stored at unit j ^ (r & 7)
  for (int idx = tid; idx < NP * W / 8; idx += blockDim.x) {
    int r = idx / (W / 8), u = idx % (W / 8);  // u-th 16B unit across the full row
    int chunk = u / 8, j = u % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(Q + r * W + u * 8);
    *reinterpret_cast<uint4*>(qs + chunk * 4096 + r * 128 + ((j ^ (r & 7)) * 16)) = v;
  }
  // P: MN-major interleave: (tok t, head n) at (n/8)*SBO + (t/8)*128 + (t%8)*16 + (n%8)*2, SBO = 16*128
  for (int idx = tid; idx < ROWS * NP / 8; idx += blockDim.x) {
    int t = idx / (NP / 8), g = idx % (NP / 8);
    const uint4 v = *reinterpret_cast<const uint4*>(P + t * NP + g * 8);
    *reinterpret_cast<uint4*>(ps + g * (ROWS / 8) * 128 + (t / 8) * 128 + (t % 8) * 16) = v;
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;

  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_tma, 3 * 16384);
    for (int c = 0; c < 3; ++c)
      for (int h = 0; h < 2; ++h) tma_load_2d(&kv_map, &bar_tma, kv + c * 16384 + h * 8192, c * 64, h * 64);
  }
  mbar_wait(&bar_tma, 0);
  tc_fence_after();
  if (tid == 0) {
    // QK, M = 128 -> cols [0,32); M = 64 -> cols [32,64)
    for (int c = 0; c < 3; ++c)
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t a = make_sdesc(smem_u32(kv + c * 16384) + kk * 32, 16, 1024, kSw128);
        uint64_t b = make_sdesc(smem_u32(qs + c * 4096) + kk * 32, 16, 1024, kSw128);
        mma_bf16_ss(tbase + 0, a, b, make_idesc_bf16(128, NP, false, false), (c | kk) != 0);
        mma_bf16_ss(tbase + 32, a, b, make_idesc_bf16(64, NP, false, false), (c | kk) != 0);
      }
    // PV, M = 128 over latent cols [0,128) (chunks 0,1 via LBO) -> cols [64,96)
    // PV, M = 64 over latent cols [0,64) (chunk 0) -> cols [96,128)
    for (int i = 0; i < ROWS / 16; ++i) {
      uint64_t a = make_sdesc(smem_u32(kv) + i * 2048, 16384, 1024, kSw128);
      uint64_t b = make_sdesc(smem_u32(ps) + i * 256, 128, (ROWS / 8) * 128, kSwNone);
      mma_bf16_ss(tbase + 64, a, b, make_idesc_bf16(128, NP, true, true), i != 0);
      mma_bf16_ss(tbase + 96, a, b, make_idesc_bf16(64, NP, true, true), i != 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const int lane_base = (warp & 3) * 32;
  const uint32_t trow = tbase + (uint32_t(lane_base) << 16);
  uint32_t r[32];
  for (int blk = 0; blk < 4; ++blk) {
    for (int q = 0; q < 4; ++q) tmem_ld8(trow + blk * 32 + q * 8, r + q * 8);
    tmem_ld_wait();
    const int L = lane_base + lane_id();
    for (int n = 0; n < NP; ++n) {
      float v = __uint_as_float(r[n]);
      if (blk == 0) out_qk128[L * NP + n] = v;
      if (blk == 2) out_pv128[L * NP + n] = v;
      // M = 64: row m lives at lane (m % 16) + 32 * (m / 16)
      if ((blk == 1 || blk == 3) && (L % 32) < 16) {
        int m = (L % 32) + 16 * (L / 32);
        (blk == 1 ? out_qk64 : out_pv64)[m * NP + n] = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

static float bf(float x) {  // round to bf16 and back
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  std::vector<float> kvf(ROWS * W), qf(NP * W), pf(ROWS * NP);
  srand(1);
  auto rnd = [] { return bf((rand() / float(RAND_MAX)) * 2.f - 1.f); };
  for (auto& x : kvf) x = rnd();
  for (auto& x : qf) x = rnd();
  for (auto& x : pf) x = rnd();
  std::vector<__nv_bfloat16> kvb(kvf.size()), qb(qf.size()), pb(pf.size());
  for (size_t i = 0; i < kvf.size(); ++i) kvb[i] = __float2bfloat16(kvf[i]);
  for (size_t i = 0; i < qf.size(); ++i) qb[i] = __float2bfloat16(qf[i]);
  for (size_t i = 0; i < pf.size(); ++i) pb[i] = __float2bfloat16(pf[i]);
  __nv_bfloat16 *dkv, *dq, *dp;
  float* dout;
  cudaMalloc(&dkv, kvb.size() * 2);
  cudaMalloc(&dq, qb.size() * 2);
  cudaMalloc(&dp, pb.size() * 2);
  cudaMalloc(&dout, 4 * ROWS * NP * 4);
  cudaMemset(dout, 0, 4 * ROWS * NP * 4);
  cudaMemcpy(dkv, kvb.data(), kvb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, qb.data(), qb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pb.data(), pb.size() * 2, cudaMemcpyHostToDevice);

  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qres;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &qres);
  CUtensorMap map;
  cuuint64_t dims[2] = {W, ROWS};
  cuuint64_t strides[1] = {W * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dkv, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    printf("encode failed %d\n", int(cr));
    return 1;
  }
  int smem = 3 * 16384 + 3 * 4096 + 8192 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(map, dq, dp, dout, dout + ROWS * NP, dout + 2 * ROWS * NP, dout + 3 * ROWS * NP);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> out(4 * ROWS * NP);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  double err[4] = {0, 0, 0, 0};
  for (int t = 0; t < ROWS; ++t)
    for (int n = 0; n < NP; ++n) {
      double s = 0;
      for (int k = 0; k < W; ++k) s += double(kvf[t * W + k]) * qf[n * W + k];
      err[0] = fmax(err[0], fabs(s - out[t * NP + n]));
      if (t < 64) err[1] = fmax(err[1], fabs(s - out[ROWS * NP + t * NP + n]));
    }
  for (int c = 0; c < 128; ++c)
    for (int n = 0; n < NP; ++n) {
      double s = 0;
      for (int t = 0; t < ROWS; ++t) s += double(kvf[t * W + c]) * pf[t * NP + n];
      err[2] = fmax(err[2], fabs(s - out[2 * ROWS * NP + c * NP + n]));
      if (c < 64) err[3] = fmax(err[3], fabs(s - out[3 * ROWS * NP + c * NP + n]));
    }
  printf("QK M128 maxerr %.3e\nQK M64 maxerr %.3e\nPV M128 maxerr %.3e\nPV M64 maxerr %.3e\n", err[0], err[1],
         err[2], err[3]);
  bool ok = err[0] < 1e-2 && err[1] < 1e-2 && err[2] < 1e-2 && err[3] < 1e-2;
  printf(ok ? "PROBE OK\n" : "PROBE FAIL\n");
  return ok ? 0 : 2;
}
