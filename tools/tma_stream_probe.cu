// TMA streaming microbenchmark (dev tool): how much HBM bandwidth do 2-D/3-D TMA boxes
// deliver as a function of ring depth and box size, with a consumer that frees slots
// immediately. Pool rows of W bf16; each CTA streams `rows_per_cta` consecutive rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "ptx.cuh"
using namespace mlra;

__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, int rows_per_cta, int box_rows, int nchunks,
                              int slots, int slot_bytes, int use3d, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + slots * slot_bytes);
  uint64_t* empty = full + 16;
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
      if (use3d) {
        tma_load_3d_hint(&map, &full[s], smem + s * slot_bytes, 0, row0 + i * box_rows, 0, pol);
      } else {
        for (int c = 0; c < nchunks; ++c)
          tma_load_2d_hint(&map, &full[s], smem + s * slot_bytes + c * box_rows * 128, c * 64, row0 + i * box_rows, pol);
      }
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

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int W = 192;  // TP4 row: 384 B
  const long long rows = 16LL * 32768;
  void* pool;
  cudaMalloc(&pool, rows * W * 2);
  cudaMemset(pool, 1, rows * W * 2);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  const int ctas = 144;
  const int rows_per_cta = int(rows / ctas) / 128 * 128;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  for (int use3d = 0; use3d < 2; ++use3d)
    for (int box_rows : {64, 128, 256}) {
      const int nchunks = 3;  // all 192 columns per box (3 x 64)
      CUtensorMap map;
      CUresult cr;
      if (use3d) {
        cuuint64_t dims[3] = {64, cuuint64_t(rows), 3};
        cuuint64_t str[2] = {cuuint64_t(W) * 2, 128};
        cuuint32_t box[3] = {64, cuuint32_t(box_rows), 3};
        cuuint32_t es[3] = {1, 1, 1};
        cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[2] = {cuuint64_t(W), cuuint64_t(rows)};
        cuuint64_t str[1] = {cuuint64_t(W) * 2};
        cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
        cuuint32_t es[2] = {1, 1};
        cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", int(cr)); continue; }
      const int slot_bytes = box_rows * 128 * nchunks;
      for (int slots : {2, 3, 4, 6, 8, 12}) {
        const int smem = slots * slot_bytes + 16 * 16 + 64;
        if (smem > 232448 || slots > 16) continue;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9;
        for (int it = 0; it < 4; ++it) {
          cudaMemsetAsync(flush, it, 512 << 20);
          cudaEventRecord(e0);
          stream_kernel<<<ctas, 64, smem>>>(map, rows_per_cta, box_rows, nchunks, slots, slot_bytes, use3d, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (it > 0 && ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        const double bytes = double(rows_per_cta) * ctas * W * 2;
        printf("%s box_rows=%3d slot=%6d B slots=%2d in-flight/SM=%7d B: %7.1f us %6.0f GB/s %s\n", use3d ? "3D" : "2D",
               box_rows, slot_bytes, slots, slots * slot_bytes, best * 1e3, bytes / best / 1e6,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  return 0;
}
