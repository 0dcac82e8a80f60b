// K4 -- attention output side: sigmoid output gate, W^O projection,
// residual, and the tensor-parallel sum over ranks, fused into one GEMM + collective kernel.
//
// Reference semantics (attnkit/zoo.py:125-127 gated_output, :146-149 block_forward):
//   y = hidden + (attn_flat * sigmoid(hidden @ W_g)) @ W_o
// Under tensor parallelism a rank holds the attention output of its heads (or, for MLRA-4
// sharded by branch, a per-head partial of every head); both the gate and the projection are
// linear in that output, so rank r computes  y_r = (attn_r * sigmoid(gate_pre_r)) @ W_o[rows_r]
// and y = hidden + sum_r y_r  (attnkit/decode.py:264-285 sums contributions in device order).
//
// K4a (outproj_gate_kernel): a = bf16(attn * sigmoid(gate_pre)) [B, K] -- tiny, elementwise.
// K4  (outproj_allreduce_kernel), launched as a programmatic dependent of K4a, streams W_o
// (K x D bf16, the only large operand) from HBM exactly once. Grid: slabs of NC = 128 output
// columns x KS slices of K; the KS CTAs of a slab form a thread-block cluster.
//   1. GEMM: the CTA's W_o slice goes through a 4-stage ring of 32 KB chunks (128 rows x 128
//      columns, cp.async, 16-byte units XOR-swizzled by row so ldmatrix.trans is conflict-free);
//      the ring is primed BEFORE griddepcontrol.wait (W_o does not depend on K4a). The bf16 A
//      slice ([16 rows][<= 1024], one cp.async group) is loaded after the wait. Warp w owns
//      output columns [16w, 16w+16) of the slab: per 128-row chunk 8 x (ldmatrix A, ldmatrix.trans
//      W, 2 mma.sync m16n8k16), fp32 accumulators in registers, no cross-warp reduction.
//   2. Cluster: row m of the slab belongs to CTA m % KS. Every CTA stores its slice partial of
//      each row into the owner's slot [my slice][row] through DSMEM (st.shared::cluster); after one
//      cluster barrier the owner adds the KS slots in ascending slice order.
//   3. world == 1: y = resid + partial.
//      world > 1 (one-shot all-reduce over peer memory: NVLink P2P through IPC mappings): the
//      owner stores its rows into EVERY rank's receive buffer (slot [parity][my rank]), then a
//      release store of the call's epoch to that rank's flag (parity, my rank, slab, ks); it waits
//      (acquire, bounded) for the world flags of its (slab, ks) and sums the world partials in
//      ascending rank order -- every rank computes bit-identical y.
//   The receive buffers are double-buffered by epoch parity: a rank reaches call e+2 only after
//   every peer has pushed call e+1, which the peer does after finishing call e's reads.
//
// Communication region of a rank (mlra_outproj_comm_bytes): fp32 recv [2][world][B][D], then
// uint32 flags [2][world][nslabs * kOpMaxKS], then uint32 {epoch counter, done counter};
// zero-filled once. The call epoch lives there (read at kernel start, advanced by the last CTA
// to finish), so the call can be captured in a CUDA graph and replayed.
// Sim mode (tests on one GPU): gridDim.y = world CTA rows act as the ranks on one device, KS = 1,
// one cooperative launch so every CTA is resident (flag waits cannot starve).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

#ifndef MLRA_OP_STAMP  // dev phase stamps (tools/outproj_trace.cu)
#define MLRA_OP_STAMP(k) \
  do {                   \
  } while (0)
#endif

namespace mlra {

constexpr int kOpThreads = 256, kOpNC = 128, kOpKC = 128, kOpStages = 4, kOpM = 16, kOpMaxRanks = 8;
constexpr int kOpMaxKS = 8, kOpMaxB = 64, kOpAK = 1024;   // A slice: at most 1024 K per pass
constexpr int kOpWBytes = kOpKC * kOpNC * 2;               // 32 KB ring stage
constexpr int kOpARow = (kOpAK + 8) * 2;                   // A row stride (bytes): 16 mod 128, conflict-free
constexpr int kOpABytes = kOpM * kOpARow;
constexpr int kOpSlotRows = 72;                            // >= KS * ceil(B / KS) for B <= 64, KS <= 8
constexpr int kOpSlotBytes = kOpSlotRows * kOpNC * 4;

struct OutProjParams {
  // per local rank (index blockIdx.y): one entry in real mode, `world` in sim mode
  const __nv_bfloat16* a[kOpMaxRanks];       // [B, K] bf16 gated attention output (K4a)
  const __nv_bfloat16* w_o[kOpMaxRanks];     // [K, D] bf16
  float* y[kOpMaxRanks];                     // [B, D] fp32
  const float* resid;                        // [B, D] fp32 or null (shared by the ranks)
  float* comm[kOpMaxRanks];                  // communication region of every GLOBAL rank
  int B, K, D, world, rank0, nslabs, ks_count, k_slice;
};

inline size_t outproj_smem() { return size_t(kOpStages) * kOpWBytes + kOpABytes + kOpSlotBytes; }
inline int outproj_nslabs(int D) { return (D + kOpNC - 1) / kOpNC; }

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
__device__ __forceinline__ void st_shared_cluster_f32x2(uint32_t addr, float x, float y) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(x), "f"(y) : "memory");
}

// K4a: a[i] = bf16(attn[i] * sigmoid(gate[i])) (gate may be null), 8 elements per thread.
__global__ void __launch_bounds__(256) outproj_gate_kernel(const float* __restrict__ attn,
                                                           const float* __restrict__ gate,
                                                           __nv_bfloat16* __restrict__ a, int n) {
  griddep_launch_dependents();
  const int i = (blockIdx.x * 256 + threadIdx.x) * 8;
  if (i >= n) return;
  float v[8];
  *reinterpret_cast<float4*>(v) = __ldg(reinterpret_cast<const float4*>(attn + i));
  *reinterpret_cast<float4*>(v + 4) = __ldg(reinterpret_cast<const float4*>(attn + i + 4));
  if (gate != nullptr) {
    float z[8];
    *reinterpret_cast<float4*>(z) = __ldg(reinterpret_cast<const float4*>(gate + i));
    *reinterpret_cast<float4*>(z + 4) = __ldg(reinterpret_cast<const float4*>(gate + i + 4));
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= 1.f / (1.f + __expf(-z[j]));
  }
  uint4 o;
  o.x = pack_bf16(v[0], v[1]);
  o.y = pack_bf16(v[2], v[3]);
  o.z = pack_bf16(v[4], v[5]);
  o.w = pack_bf16(v[6], v[7]);
  *reinterpret_cast<uint4*>(a + i) = o;
}

__global__ void __launch_bounds__(kOpThreads, 1)
outproj_allreduce_kernel(const __grid_constant__ OutProjParams p) {
  extern __shared__ __align__(128) uint8_t op_smem[];
  uint8_t* ring = op_smem;                                                       // [S][128 rows][256 B]
  uint8_t* a_tile = op_smem + kOpStages * kOpWBytes;                              // [16][kOpARow]
  float* slots = reinterpret_cast<float*>(a_tile + kOpABytes);                   // [KS][rpo][128]
  float* fin = reinterpret_cast<float*>(ring);                                   // [rpo][128] after the GEMM
  const int KS = p.ks_count;
  const int li = blockIdx.y, rank = p.rank0 + li, slab = blockIdx.x / KS, ks = blockIdx.x % KS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int B = p.B, K = p.K, D = p.D, n0 = slab * kOpNC;
  const int rpo = (B + KS - 1) / KS;  // rows per owner
  const int kbeg = ks * p.k_slice, kend = min(K, kbeg + p.k_slice);
  const __nv_bfloat16* a_g = p.a[li];
  const __nv_bfloat16* w = p.w_o[li];
  const uint32_t ring_u32 = smem_u32(ring), a_u32 = smem_u32(a_tile), slots_u32 = smem_u32(slots);
  MLRA_OP_STAMP(0);
  cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store (peers started)
  bool waited = false, cl_started = false;

  for (int m0 = 0; m0 < B; m0 += kOpM) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int sb = kbeg; sb < kend; sb += kOpAK) {  // pass: 16 rows x <= 1024 of K
      const int se = min(kend, sb + kOpAK);
      const int nch = (se - sb + kOpKC - 1) / kOpKC;
      auto load_w = [&](int c) {
        const int k0 = sb + c * kOpKC;
        const uint32_t st = ring_u32 + (c % kOpStages) * kOpWBytes;
#pragma unroll
        for (int j = 0; j < kOpKC * (kOpNC / 8) / kOpThreads; ++j) {  // 128 rows x 16 units of 16 B
          const int i = tid + j * kOpThreads, r = i >> 4, q = i & 15, k = k0 + r, n = n0 + q * 8;
          const bool ok = k < se && n < D;
          const void* src = ok ? static_cast<const void*>(w + size_t(k) * D + n) : static_cast<const void*>(w);
          cp_async16(st + r * (kOpNC * 2) + ((q ^ (r & 7)) * 16), src, ok ? 16u : 0u);
        }
      };
      for (int c = 0; c < kOpStages - 1; ++c) {
        if (c < nch) load_w(c);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      if (!waited) {
        griddep_wait();  // a comes from K4a (W_o above does not)
        waited = true;
      }
      for (int i = tid; i < kOpM * (kOpAK / 8); i += kOpThreads) {  // A: 16 rows x (se - sb) bf16
        const int r = i / (kOpAK / 8), q = i % (kOpAK / 8), m = m0 + r, k = sb + q * 8;
        if (k >= sb + ((se - sb + kOpKC - 1) / kOpKC) * kOpKC) continue;  // beyond the last chunk
        const bool ok = m < B && k < se;
        cp_async16(a_u32 + r * kOpARow + q * 16,
                   ok ? static_cast<const void*>(a_g + size_t(m) * K + k) : static_cast<const void*>(a_g),
                   ok ? 16u : 0u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      MLRA_OP_STAMP(1);
      for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kOpStages - 2) : "memory");
        __syncthreads();  // chunk c landed for every thread; slot (c-1) % S is free again
        if (c + kOpStages - 1 < nch) load_w(c + kOpStages - 1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const uint32_t st = ring_u32 + (c % kOpStages) * kOpWBytes;
        const int q = lane >> 3;
#pragma unroll
        for (int kk = 0; kk < kOpKC / 16; ++kk) {
          uint32_t a[4], b[4];
          const int ka = c * kOpKC + kk * 16;  // within the A tile
          ldmatrix_x4(a, a_u32 + ((lane & 7) + (q & 1) * 8) * kOpARow + (ka + (q >> 1) * 8) * 2);
          const int kw = kk * 16 + (q & 1) * 8 + (lane & 7);  // within the W chunk
          ldmatrix_x4_trans(b, st + kw * (kOpNC * 2) + (((warp * 2 + (q >> 1)) ^ (kw & 7)) * 16));
          mma_m16n8k16_bf16(acc[0], a, b[0], b[1]);
          mma_m16n8k16_bf16(acc[1], a, b[2], b[3]);
        }
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // ring and A tile are reused by the next pass
    }
    MLRA_OP_STAMP(2);
    if (!cl_started) {  // every CTA of the cluster runs: its shared memory may be written
      cluster_wait_acquire();
      cl_started = true;
    }
    // slice partial of rows m0+g, m0+g+8 -> owner (m % KS) slot [ks][m / KS] through DSMEM
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = m0 + g + 8 * h;
      if (m >= B) continue;
      const uint32_t remote_row = mapa_shared(slots_u32 + ((ks * rpo + m / KS) * kOpNC) * 4, m % KS);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = warp * 16 + j * 8 + 2 * t4;
        st_shared_cluster_f32x2(remote_row + col * 4, acc[j][2 * h], acc[j][2 * h + 1]);
      }
    }
  }
  if (!waited) griddep_wait();  // (empty K slice) keep the dependency on K4a
  if (!cl_started) cluster_wait_acquire();
  cluster_arrive_release();
  cluster_wait_acquire();
  MLRA_OP_STAMP(3);
  // ---- my rows (m = lr * KS + ks): add the KS slice slots in ascending slice order
  const int nrows = ks < B ? (B - ks + KS - 1) / KS : 0;
  for (int i = tid; i < nrows * kOpNC; i += kOpThreads) {
    const int lr = i / kOpNC, c = i % kOpNC;
    float s = 0.f;
    for (int j = 0; j < KS; ++j) s += slots[(j * rpo + lr) * kOpNC + c];
    fin[i] = s;
  }
  __syncthreads();
  MLRA_OP_STAMP(4);
  const int ncol = min(kOpNC, D - n0);
  if (p.world == 1) {
    for (int i = tid; i < nrows * kOpNC; i += kOpThreads) {
      const int lr = i / kOpNC, c = i % kOpNC;
      if (c >= ncol) continue;
      const size_t o = size_t(lr * KS + ks) * D + n0 + c;
      p.y[li][o] = (p.resid != nullptr ? p.resid[o] : 0.f) + fin[i];
    }
    MLRA_OP_STAMP(5);
    return;
  }
  // ---- one-shot all-reduce of my rows across ranks
  const int W = p.world;
  const size_t recv_floats = size_t(2) * W * B * D;
  const size_t flag_idx = size_t(slab) * kOpMaxKS + ks;
  const size_t flags_per_rank = size_t(p.nslabs) * kOpMaxKS;
  uint32_t* ctr = reinterpret_cast<uint32_t*>(p.comm[rank] + recv_floats) + size_t(2) * W * flags_per_rank;
  __shared__ uint32_t s_epoch;
  if (tid == 0) s_epoch = *reinterpret_cast<volatile uint32_t*>(ctr) + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int par = int(epoch & 1u);
  for (int r = 0; r < W; ++r) {
    float* dst = p.comm[r] + (size_t(par) * W + rank) * size_t(B) * D;
    for (int i = tid; i < nrows * (kOpNC / 4); i += kOpThreads) {
      const int lr = i / (kOpNC / 4), c4 = (i % (kOpNC / 4)) * 4;
      if (c4 < ncol)  // D % 8 == 0: whole float4s
        *reinterpret_cast<float4*>(dst + size_t(lr * KS + ks) * D + n0 + c4) =
            *reinterpret_cast<const float4*>(fin + lr * kOpNC + c4);
    }
  }
  __syncthreads();
  if (tid < W) {
    __threadfence_system();
    uint32_t* flags = reinterpret_cast<uint32_t*>(p.comm[tid] + recv_floats);
    st_release_sys_u32(flags + (size_t(par) * W + rank) * flags_per_rank + flag_idx, epoch);
  }
  if (tid < W) {  // wait for the world partials of my rows (a peer missing for 4 s traps)
    const uint32_t* flags = reinterpret_cast<const uint32_t*>(p.comm[rank] + recv_floats);
    const uint32_t* f = flags + (size_t(par) * W + tid) * flags_per_rank + flag_idx;
    const unsigned long long t_start = op_globaltimer();
    while (ld_acquire_sys_u32(f) != epoch) {
      if (op_globaltimer() - t_start > 4000000000ull) __trap();
      __nanosleep(64);
    }
  }
  __syncthreads();
  const float* recv = p.comm[rank] + size_t(par) * W * size_t(B) * D;
  for (int i = tid; i < nrows * kOpNC; i += kOpThreads) {
    const int lr = i / kOpNC, c = i % kOpNC;
    if (c >= ncol) continue;
    const size_t o = size_t(lr * KS + ks) * D + n0 + c;
    float s = 0.f;
    for (int r = 0; r < W; ++r) s += __ldcv(recv + size_t(r) * B * D + o);  // ascending rank order
    p.y[li][o] = (p.resid != nullptr ? p.resid[o] : 0.f) + s;
  }
  if (tid == 0) {  // advance this rank's epoch once every CTA of the call has read it
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1u) {
      ctr[1] = 0u;
      atomicExch(ctr, epoch);
    }
  }
  MLRA_OP_STAMP(5);
}

}  // namespace mlra
