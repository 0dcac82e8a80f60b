// Read-bandwidth ceiling probe (dev tool): what does HBM deliver for a pure streaming READ
// on this B200 — (1) plain 16-byte LDG at full occupancy, (2) TMA boxes into an smem ring
// with an immediate consumer, over the TP1 decode pool geometry (1152-byte rows, 604 MB).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2603_02188_b200/csrc -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <algorithm>
#include "ptx.cuh"
using namespace mlra;

__global__ void ldg_kernel(const uint4* __restrict__ src, size_t n, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
          d = __ldcs(src + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldcs(src + i).x;
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, int rows_per_cta, int box_rows, int nchunks,
                           int slots, int slot_bytes, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + slots * slot_bytes);
  uint64_t* empty = full + 32;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int n = rows_per_cta / box_rows;
  const int row0 = blockIdx.x * rows_per_cta;
  if (tid == 0) {
    const uint64_t pol = l2_policy_evict_first();
    for (int i = 0; i < n; ++i) {
      const int s = i % slots;
      mbar_wait(&empty[s], ((i / slots) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], slot_bytes);
      tma_load_3d_hint(&map, &full[s], smem + s * slot_bytes, 0, row0 + i * box_rows, 0, pol);
    }
  } else if (tid == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % slots;
      mbar_wait(&full[s], (i / slots) & 1);
      acc += smem[s * slot_bytes + (i & 127)];
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345678) *sink = acc;
  }
}

// K2's access pattern: per tile, NB boxes of `cpb` chunks (one per branch, columns b*cpb*64)
// then a rope box of 1 chunk, each into its own ring slot.
__global__ void tma_branchy_kernel(const __grid_constant__ CUtensorMap map_b, const __grid_constant__ CUtensorMap map_r,
                                   int rows_per_cta, int box_rows, int nb, int cpb, int slots, int slot_bytes,
                                   unsigned long long* sink, int hold, long long* lat) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + slots * slot_bytes);
  uint64_t* empty = full + 32;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int ntile = rows_per_cta / box_rows;
  const int n = ntile * (nb + 1);
  const int row0 = blockIdx.x * rows_per_cta;
  const int rope_bytes = box_rows * 128;
  if (tid == 0) {
    const uint64_t pol = l2_policy_evict_first();
    for (int i = 0; i < n; ++i) {
      const int s = i % slots, t = i / (nb + 1), b = i % (nb + 1);
      mbar_wait(&empty[s], ((i / slots) & 1) ^ 1);
      if (blockIdx.x == 0 && i < 512) lat[i] = clock64();
      if (b < nb) {
        mbar_arrive_expect_tx(&full[s], slot_bytes);
        tma_load_3d_hint(&map_b, &full[s], smem + s * slot_bytes, 0, row0 + t * box_rows, b * cpb, pol);
      } else {
        mbar_arrive_expect_tx(&full[s], rope_bytes);
        tma_load_2d_hint(&map_r, &full[s], smem + s * slot_bytes, nb * cpb * 64, row0 + t * box_rows, pol);
      }
    }
  } else if (tid == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % slots;
      mbar_wait(&full[s], (i / slots) & 1);
      const long long ta = clock64();
      if (blockIdx.x == 0 && i < 512) lat[512 + i] = ta;
      acc += smem[s * slot_bytes + (i & 127)];
      while (clock64() - ta < hold) {
      }
      mbar_arrive(&empty[s]);
    }
    if (acc == 12345678) *sink = acc;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int W = 576;  // TP1 MLRA-4 row: 4 x 128 latent + 64 rope, bf16 = 1152 B
  const long long rows = 16LL * 32768;
  const size_t bytes = size_t(rows) * W * 2;
  void* pool;
  cudaMalloc(&pool, bytes);
  cudaMemset(pool, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto&& launch) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(flush, it, 512 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it > 0 && ms < best) best = ms;
    }
    return best;
  };
  for (int per_sm : {1, 2, 4, 8}) {
    for (int threads : {256, 512, 1024}) {
      if (per_sm * threads > 2048) continue;
      const float ms = timeit([&] {
        ldg_kernel<<<sms * per_sm, threads>>>(static_cast<const uint4*>(pool), bytes / 16, reinterpret_cast<unsigned*>(sink));
      });
      printf("LDG  grid=%4d x %4d: %7.1f us %6.0f GB/s %s\n", sms * per_sm, threads, ms * 1e3, bytes / ms / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  for (int box_rows : {32, 64, 128}) {
    CUtensorMap map;
    const int nchunks = W / 64;
    cuuint64_t dims[3] = {64, cuuint64_t(rows), cuuint64_t(nchunks)};
    cuuint64_t str[2] = {cuuint64_t(W) * 2, 128};
    cuuint32_t box[3] = {64, cuuint32_t(box_rows), cuuint32_t(nchunks > 8 ? 8 : nchunks)};
    cuuint32_t es[3] = {1, 1, 1};
    // box covers 8 of the 9 chunks at most (box dims <= 256); stream those
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      continue;
    }
    const int slot_bytes = box_rows * 128 * (nchunks > 8 ? 8 : nchunks);
    for (int ctas : {144, 148, 296}) {
      for (int slots : {2, 3, 4, 6, 8, 12, 16}) {
        const int smem = slots * slot_bytes + 64 * 8 + 64;
        if (smem > 232448 / (ctas > 148 ? 2 : 1) || slots > 32) continue;
        const int rows_per_cta = int(rows / ctas) / box_rows * box_rows;
        const float ms = timeit([&] {
          tma_kernel<<<ctas, 64, smem>>>(map, rows_per_cta, box_rows, nchunks, slots, slot_bytes, sink);
        });
        const double moved = double(rows_per_cta) * ctas * slot_bytes / box_rows;
        printf("TMA  box_rows=%3d ctas=%3d slot=%6d B slots=%2d in-flight/SM=%7d B: %7.1f us %6.0f GB/s %s\n", box_rows,
               ctas, slot_bytes, slots, slots * slot_bytes * (ctas > 148 ? 2 : 1), ms * 1e3, moved / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  cudaFuncSetAttribute(tma_branchy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  long long* lat;
  cudaMalloc(&lat, 1024 * 8);
  for (int box_rows : {128}) {
    const int nchunks = W / 64, cpb = 2, nb = 4;
    CUtensorMap mb, mr;
    cuuint64_t dims[3] = {64, cuuint64_t(rows), cuuint64_t(nchunks)};
    cuuint64_t str[2] = {cuuint64_t(W) * 2, 128};
    cuuint32_t box[3] = {64, cuuint32_t(box_rows), cuuint32_t(cpb)};
    cuuint32_t es[3] = {1, 1, 1};
    encode(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint64_t d2[2] = {cuuint64_t(W), cuuint64_t(rows)};
    cuuint64_t s2[1] = {cuuint64_t(W) * 2};
    cuuint32_t b2[2] = {64, cuuint32_t(box_rows)};
    encode(&mr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int slot_bytes = box_rows * 128 * cpb;
    for (int slots : {4, 5, 6}) {
      for (int hold : {0, 500, 1000, 2000, 3000}) {
        const int smem = slots * slot_bytes + 64 * 8 + 64;
        if (smem > 232448) continue;
        const int ctas = 144;
        const int rows_per_cta = int(rows / ctas) / box_rows * box_rows;
        const float ms = timeit([&] {
          tma_branchy_kernel<<<ctas, 64, smem>>>(mb, mr, rows_per_cta, box_rows, nb, cpb, slots, slot_bytes, sink, hold, lat);
        });
        long long h[1024];
        cudaMemcpy(h, lat, sizeof(h), cudaMemcpyDeviceToHost);
        long long l[400];
        for (int i = 0; i < 400; ++i) l[i] = h[512 + 50 + i] - h[50 + i];
        std::sort(l, l + 400);
        const double moved = double(rows_per_cta) * ctas * W * 2;
        printf("TMA-branchy slots=%d hold=%4d: %7.1f us %6.0f GB/s  median load latency %lld cycles\n", slots, hold,
               ms * 1e3, moved / ms / 1e6, l[200]);
      }
    }
  }
  return 0;
}
