// K4 -- attention output side: sigmoid output gate, W^O projection,
// residual, and the tensor-parallel sum over ranks, fused in one kernel.
//
// Reference semantics (attnkit/zoo.py:125-127 gated_output, :146-149 block_forward):
//   y = hidden + (attn_flat * sigmoid(hidden @ W_g)) @ W_o
// Under tensor parallelism a rank holds the attention output of its heads (or, for MLRA-4
// sharded by branch, a per-head partial of every head); both the gate and the projection are
// linear in that output, so rank r computes  y_r = (attn_r * sigmoid(gate_pre_r)) @ W_o[rows_r]
// and y = hidden + sum_r y_r  (attnkit/decode.py:264-285 sums contributions in device order).
//
// One CTA owns a slab of NC = 32 output columns for all sequences:
//   1. GEMM: W_o[:, slab] streamed in KC = 64-row chunks by cp.async (4-stage ring, XOR-swizzled
//      so ldmatrix.trans is conflict-free) together with the fp32 attn / gate chunks; the gated
//      A operand is formed in registers (fp32 -> bf16) and multiplied on mma.sync m16n8k16
//      (8 warps = 4 k-steps x 2 column halves, reduced through smem).
//   2. world == 1: y = resid + partial.
//      world > 1 (one-shot all-reduce over peer memory, NVLink P2P / IPC mappings): the slab
//      partial is stored into EVERY rank's receive buffer (slot [parity][my rank]), then a
//      release store of the call's epoch to that rank's flag for (parity, my rank, slab);
//      the CTA waits (acquire, bounded) for the world flags of its slab, and sums the world
//      partials in ascending rank order -- every rank computes bit-identical y.
//   The receive buffers are double-buffered by epoch parity: a rank reaches call e+2 only after
//   each peer has pushed call e+1, which that peer does after finishing call e's reads.
//
// Communication region of a rank (mlra_outproj_comm_bytes): fp32 recv [2][world][B][D], then
// uint32 flags [2][world][nslabs]; zero-initialised once, epochs start at 1 and increase by 1.
// Sim mode (tests on one GPU): gridDim.y = world CTAs-rows act as the ranks on one device,
// launched cooperatively so every CTA is resident (flag waits cannot starve).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

namespace mlra {

constexpr int kOpThreads = 256, kOpNC = 32, kOpKC = 64, kOpStages = 4, kOpM = 16, kOpMaxRanks = 8;
constexpr int kOpAStride = kOpKC + 8;  // fp32 row stride of the A / gate chunks (conflict-free float2 reads)
constexpr int kOpWBytes = kOpKC * kOpNC * 2;                // 4 KB
constexpr int kOpABytes = kOpM * kOpAStride * 4;            // 4.5 KB
constexpr int kOpStageBytes = kOpWBytes + 2 * kOpABytes;    // W, attn, gate
constexpr int kOpMaxB = 64;

struct OutProjParams {
  // per local rank (index blockIdx.y): one entry in real mode, `world` in sim mode
  const float* attn[kOpMaxRanks];            // [B, K] fp32
  const float* gate_pre[kOpMaxRanks];        // [B, K] fp32 pre-activation or null
  const __nv_bfloat16* w_o[kOpMaxRanks];     // [K, D] bf16
  float* y[kOpMaxRanks];                     // [B, D] fp32
  const float* resid;                        // [B, D] fp32 or null (shared by the ranks)
  float* comm[kOpMaxRanks];                  // communication region of every GLOBAL rank
  int B, K, D, world, rank0, nslabs;
  uint32_t epoch;
};

inline size_t outproj_smem() {
  return size_t(kOpStages) * kOpStageBytes + size_t(4) * kOpM * kOpNC * 4 + size_t(kOpMaxB) * kOpNC * 4;
}

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long op_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

__global__ void __launch_bounds__(kOpThreads)
outproj_allreduce_kernel(const __grid_constant__ OutProjParams p) {
  extern __shared__ __align__(128) uint8_t op_smem[];
  float* red = reinterpret_cast<float*>(op_smem + size_t(kOpStages) * kOpStageBytes);  // [4 ks][16][32]
  float* part = red + 4 * kOpM * kOpNC;                                                 // [B][32]
  const int li = blockIdx.y, rank = p.rank0 + li, slab = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int B = p.B, K = p.K, D = p.D, n0 = slab * kOpNC;
  const float* attn = p.attn[li];
  const float* gate = p.gate_pre[li];
  const __nv_bfloat16* w = p.w_o[li];
  const int nchunks = (K + kOpKC - 1) / kOpKC;
  const int ks = warp & 3, nh = warp >> 2;  // this warp: k16 step ks of a chunk, n-tiles 2nh, 2nh+1
  const uint32_t smem_base = smem_u32(op_smem);

  for (int m0 = 0; m0 < B; m0 += kOpM) {
    // ---- stage loader: chunk c -> ring slot c % S (one 16-byte cp.async per thread per operand)
    auto load_chunk = [&](int c) {
      const int k0 = c * kOpKC;
      const uint32_t st = smem_base + (c % kOpStages) * kOpStageBytes;
      {  // W rows k0.., columns n0..n0+31: row r = tid / 4, 16-byte part q = tid % 4
        const int r = tid >> 2, q = tid & 3, k = k0 + r, n = n0 + q * 8;
        const bool ok = k < K && n < D;
        const void* src = ok ? static_cast<const void*>(w + size_t(k) * D + n) : static_cast<const void*>(w);
        cp_async16(st + r * (kOpNC * 2) + ((q ^ ((r >> 1) & 3)) * 16), src, ok ? 16u : 0u);
      }
      {  // attn / gate rows m0.. (16), columns k0..k0+63: row = tid / 16, float4 part = tid % 16
        const int r = tid >> 4, q = tid & 15, m = m0 + r, k = k0 + q * 4;
        const bool ok = m < B && k < K;
        const size_t off = size_t(m) * K + k;
        const uint32_t dst = st + kOpWBytes + (r * kOpAStride + q * 4) * 4;
        cp_async16(dst, ok ? static_cast<const void*>(attn + off) : static_cast<const void*>(attn), ok ? 16u : 0u);
        if (gate != nullptr)
          cp_async16(dst + kOpABytes, ok ? static_cast<const void*>(gate + off) : static_cast<const void*>(gate),
                     ok ? 16u : 0u);
      }
    };
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int c = 0; c < kOpStages - 1; ++c) {
      if (c < nchunks) load_chunk(c);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int c = 0; c < nchunks; ++c) {
      asm volatile("cp.async.wait_group %0;" ::"n"(kOpStages - 2) : "memory");
      __syncthreads();  // chunk c landed for every thread; slot (c-1) % S is free
      if (c + kOpStages - 1 < nchunks) load_chunk(c + kOpStages - 1);
      asm volatile("cp.async.commit_group;" ::: "memory");
      const uint8_t* st = op_smem + (c % kOpStages) * kOpStageBytes;
      const float* As = reinterpret_cast<const float*>(st + kOpWBytes);
      const float* Gs = reinterpret_cast<const float*>(st + kOpWBytes + kOpABytes);
      // A fragment (rows g, g+8; columns ks*16 + 2*t4 (+1), +8 (+9)) gated in fp32, then bf16
      uint32_t a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int row = g + (i & 1) * 8, col = ks * 16 + 2 * t4 + (i >> 1) * 8;
        float2 v = *reinterpret_cast<const float2*>(As + row * kOpAStride + col);
        if (gate != nullptr) {
          const float2 z = *reinterpret_cast<const float2*>(Gs + row * kOpAStride + col);
          v.x *= 1.f / (1.f + __expf(-z.x));
          v.y *= 1.f / (1.f + __expf(-z.y));
        }
        a[i] = pack_bf16(v.x, v.y);
      }
      // B fragments of n-tiles 2nh, 2nh+1: ldmatrix.x4.trans over the [k][n] W chunk
      uint32_t b[4];
      {
        const int q = lane >> 3, k = ks * 16 + (q & 1) * 8 + (lane & 7), part16 = nh * 2 + (q >> 1);
        ldmatrix_x4_trans(b, smem_u32(st) + k * (kOpNC * 2) + ((part16 ^ ((k >> 1) & 3)) * 16));
      }
      mma_m16n8k16_bf16(acc[0], a, b[0], b[1]);
      mma_m16n8k16_bf16(acc[1], a, b[2], b[3]);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // ---- reduce the 4 k-step warps of each column half: red[ks][row][col]
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = (nh * 2 + j) * 8 + 2 * t4;
      red[(ks * kOpM + g) * kOpNC + col] = acc[j][0];
      red[(ks * kOpM + g) * kOpNC + col + 1] = acc[j][1];
      red[(ks * kOpM + g + 8) * kOpNC + col] = acc[j][2];
      red[(ks * kOpM + g + 8) * kOpNC + col + 1] = acc[j][3];
    }
    __syncthreads();
    for (int i = tid; i < kOpM * kOpNC; i += kOpThreads) {
      const int row = i / kOpNC;
      const float v = red[i] + red[kOpM * kOpNC + i] + red[2 * kOpM * kOpNC + i] + red[3 * kOpM * kOpNC + i];
      if (m0 + row < B) part[(m0 + row) * kOpNC + (i % kOpNC)] = v;
    }
    __syncthreads();  // red and the ring are reused by the next row group
  }

  // ---- epilogue: local write or one-shot all-reduce across ranks
  const int ncol = min(kOpNC, D - n0);
  if (p.world == 1) {
    for (int i = tid; i < B * kOpNC; i += kOpThreads) {
      const int m = i / kOpNC, c = i % kOpNC;
      if (c < ncol) {
        const size_t o = size_t(m) * D + n0 + c;
        p.y[li][o] = (p.resid != nullptr ? p.resid[o] : 0.f) + part[i];
      }
    }
    return;
  }
  const int W = p.world, par = int(p.epoch & 1u);
  const size_t recv_floats = size_t(2) * W * B * D;
  // push: my slab partial -> recv[par][rank] of every rank (float4 stores, peers over NVLink)
  for (int r = 0; r < W; ++r) {
    float* dst = p.comm[r] + (size_t(par) * W + rank) * size_t(B) * D;
    for (int i = tid; i < B * (kOpNC / 4); i += kOpThreads) {
      const int m = i / (kOpNC / 4), c = (i % (kOpNC / 4)) * 4;
      if (c < ncol) {
        const float4 v = *reinterpret_cast<const float4*>(part + m * kOpNC + c);
        *reinterpret_cast<float4*>(dst + size_t(m) * D + n0 + c) = v;  // D % 8 == 0: whole float4s
      }
    }
  }
  __syncthreads();
  if (tid < W) {
    __threadfence_system();
    uint32_t* flags = reinterpret_cast<uint32_t*>(p.comm[tid] + recv_floats);
    st_release_sys_u32(flags + (size_t(par) * W + rank) * p.nslabs + slab, p.epoch);
  }
  // wait for the W partials of this slab (bounded: a peer that never arrives traps instead of hanging)
  if (tid < W) {
    const uint32_t* flags = reinterpret_cast<const uint32_t*>(p.comm[rank] + recv_floats);
    const uint32_t* f = flags + (size_t(par) * W + tid) * p.nslabs + slab;
    const unsigned long long t_start = op_globaltimer();
    while (ld_acquire_sys_u32(f) != p.epoch) {
      if (op_globaltimer() - t_start > 4000000000ull) __trap();
      __nanosleep(64);
    }
  }
  __syncthreads();
  const float* recv = p.comm[rank] + size_t(par) * W * size_t(B) * D;
  for (int i = tid; i < B * kOpNC; i += kOpThreads) {
    const int m = i / kOpNC, c = i % kOpNC;
    if (c >= ncol) continue;
    const size_t o = size_t(m) * D + n0 + c;
    float s = 0.f;
    for (int r = 0; r < W; ++r) s += __ldcv(recv + size_t(r) * B * D + o);  // ascending rank order
    p.y[li][o] = (p.resid != nullptr ? p.resid[o] : 0.f) + s;
  }
}

}  // namespace mlra
