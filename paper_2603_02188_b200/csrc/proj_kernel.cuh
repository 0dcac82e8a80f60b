// K-1 -- pre-attention projections (attnkit/latent.py:129-159
// latent_projections, attnkit/decode.py:108-126 token_cache_rows / token_queries).
//
// One weight-streaming GEMM kernel, two epilogues:
//   down  (proj_down):  [c_q_raw | kv_raw | kr_raw] = h . [W^DQ | W^DKV | W^KR]          (fp32 out)
//         + per-64-column partial sums of squares of c_q_raw (the query rmsnorm's input)
//   query (proj_query): c_q = alpha_q * rmsnorm(c_q_raw)                    (tensors.py:83-87)
//                       [q_x | q_r] = c_q . [W^Q | W^QR]
//                       q_x -> bf16 * q_scale (W^Q = W^UQ: q_nope for K1; or W^UQ.W^UK_b
//                              pre-multiplied at pack time: the absorbed query, K1 skipped)
//                       q_r -> rope(pos) (rope.py:37-60, pairs (2l, 2l+1)) * r_scale -> bf16
// The decode batch is M <= 16 rows, so the GEMMs are weight streams (HBM-bound): every CTA
// requests its whole W slice with TMA at once (boxes of 64 rows x 64 columns, 128-byte
// swizzle, one mbarrier per box) and consumes the boxes in arrival order. The weight is
// SLAB-PACKED once at load time -- [ceil(N/64)][K_pad][64]: a slab's 64 columns contiguous
// over all K rows -- so a CTA's slice is one contiguous run of HBM (k_slice x 128 B); with the
// plain row-major [K, N] layout every box row is a 128-byte piece of a different weight row
// and the grid's interleaved reads ran at ~10% of the DRAM bandwidth.
//
// Grid: slabs of 64 output columns x KS slices of K; the KS CTAs of a slab are one cluster.
//   1. W slice: k_slice x 64 bf16 (<= 48 KB) by TMA, issued first (before griddepcontrol.wait:
//      the weights do not depend on the previous kernel).
//   2. X slice: the M rows of X[:, kbeg:kend) (fp32) -> (rmsnorm scale) -> bf16 hi + lo planes
//      (two MMAs per step: ~16-bit mantissa for the activations; the weights are bf16).
//   3. mma.sync m16n8k16: warp w owns columns [16 (w%4), +16) and half (w/4) of the slice's
//      boxes; the two halves are added in a fixed order, then every CTA stores its slab
//      partial into the cluster rank 0's slot (DSMEM) and rank 0 adds the KS slots in
//      ascending slice order (deterministic) and runs the epilogue.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include "ptx.cuh"

namespace mlra {

// kPjMaxRows bounds a CTA's weight slice (48 KB) so that a CTA needs ~105 KB of shared memory:
// two fit an SM, and the query launch (a programmatic dependent) prefetches its weights into
// SMs the down launch leaves free while the down projection still runs.
constexpr int kPjThreads = 256, kPjNC = 64, kPjBox = 64, kPjM = 16, kPjMaxRows = 384, kPjMaxKS = 8;
constexpr int kPjMaxBoxes = kPjMaxRows / kPjBox;
constexpr int kPjXRow = (kPjMaxRows + 8) * 2;  // bytes per X plane row: 16 mod 128 (conflict-free ldmatrix)
constexpr int kPjWBytes = kPjMaxRows * kPjNC * 2;
constexpr int kPjXBytes = 2 * kPjM * kPjXRow;
constexpr int kPjRedBytes = 2 * kPjM * kPjNC * 4;
constexpr int kPjSlotBytes = kPjMaxKS * kPjM * kPjNC * 4;

struct ProjParams {
  const float* x;        // [M, ldx] fp32 input rows
  int ldx;
  const float* ssq_in;   // query: [norm_parts][M] partial sums of squares of x's rows (or null)
  int norm_parts;
  float norm_alpha, eps;
  int M, K, N, KS, k_slice, mode;  // mode 0: down (fp32 segments), 1: query
  int K_pad;                       // rows per slab in the slab-packed weight (K rounded up to 64)
  // down
  float* seg_out[3];     // [M, width_i] fp32
  int seg_end[3];        // cumulative column ends
  float* ssq_out;        // [ceil(ssq_cols / 64)][M]
  int ssq_cols;
  // query
  __nv_bfloat16* q_out;  // [M, nq]
  __nv_bfloat16* r_out;  // [M, H, drp]
  int nq, H, dr, drp;
  const int32_t* pos;    // [M] rope positions (+ pos_delta)
  int pos_delta;
  float rope_base, q_scale, r_scale;
  double theta[32];      // rope frequencies rope_base^(-2l/dr), l < dr/2 (host-computed)
  unsigned long long* trace;  // dev: per-CTA globaltimer stamps [grid][8] (MLRA_DEBUG_PROJ_TRACE), or null
};

__device__ __forceinline__ void pj_stamp(const ProjParams& p, int k) {
  if (p.trace != nullptr && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    p.trace[blockIdx.x * 8 + k] = t;
  }
}

static_assert(kPjRedBytes <= kPjXBytes, "the warp partials alias the (dead) X planes");
inline size_t proj_smem() { return size_t(kPjWBytes) + kPjXBytes + kPjSlotBytes + 256; }

__device__ __forceinline__ void st_shared_cluster_f32(uint32_t addr, float x) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(x) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(kPjThreads, 1) proj_gemm_kernel(const __grid_constant__ CUtensorMap w_map,
                                                                  const ProjParams p) {
  extern __shared__ __align__(1024) uint8_t pj_smem[];
  uint8_t* wt = pj_smem;                                               // [rows][64] bf16, SW128 boxes
  uint8_t* xt = wt + kPjWBytes;                                        // [2][16][kPjXRow] hi, lo
  float* red = reinterpret_cast<float*>(xt);                           // [2][16][64] (aliases X after the GEMM)
  float* slots = reinterpret_cast<float*>(xt + kPjXBytes);             // [KS][16][64] (rank 0)
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + kPjMaxKS * kPjM * kPjNC);
  float* rscale = reinterpret_cast<float*>(bars + kPjMaxBoxes);        // [16]
  const int KS = p.KS, slab = blockIdx.x / KS, ks = blockIdx.x % KS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = slab * kPjNC;
  const int kbeg = ks * p.k_slice, kend = min(p.K, kbeg + p.k_slice);
  const int rows = max(0, kend - kbeg);
  const int nbox = (rows + kPjBox - 1) / kPjBox;
  const uint32_t wt_u32 = smem_u32(wt), xt_u32 = smem_u32(xt);

  pj_stamp(p, 0);
  cluster_arrive_relaxed();  // paired with the wait before the first DSMEM store (peers started)
  if (tid == 0) {
    tma_prefetch_desc(&w_map);
    for (int b = 0; b < nbox; ++b) mbar_init(&bars[b], 1);
    fence_barrier_init();
    for (int b = 0; b < nbox; ++b) {  // every box in flight at once (OOB rows / columns zero-fill)
      mbar_arrive_expect_tx(&bars[b], kPjBox * kPjNC * 2);
      tma_load_2d(&w_map, &bars[b], wt + b * kPjBox * kPjNC * 2, 0, slab * p.K_pad + kbeg + b * kPjBox);
    }
  }
  griddep_wait();  // x (and ssq_in) come from the previous kernel on the stream
  // Dependents may start only now: a kernel launched after this one may then rely on every
  // kernel before this one being complete (K2 streams cache rows K0 wrote before this launch).
  griddep_launch_dependents();
  pj_stamp(p, 1);
  // X slice: every load in flight at once (registers), then the rmsnorm statistics, then the
  // bf16 hi / lo planes (rows >= M and columns >= rows are zero). A load loop with one
  // outstanding load per thread would pay the L2 latency ~12 times in a row.
  const int kpad = nbox * kPjBox;
  const int q4 = kpad / 4;  // float4 units per row
  constexpr int kXIter = kPjM * (kPjMaxRows / 4) / kPjThreads;
  float4 xv[kXIter];
#pragma unroll
  for (int it = 0; it < kXIter; ++it) {
    const int i = tid + it * kPjThreads, r = i / max(q4, 1), c4 = (i % max(q4, 1)) * 4;
    xv[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < kPjM * q4 && r < p.M) {
      const float* src = p.x + size_t(r) * p.ldx + kbeg + c4;
      if (c4 + 4 <= rows && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        xv[it] = __ldg(reinterpret_cast<const float4*>(src));
      } else {
        xv[it].x = c4 + 0 < rows ? __ldg(src + 0) : 0.f;
        xv[it].y = c4 + 1 < rows ? __ldg(src + 1) : 0.f;
        xv[it].z = c4 + 2 < rows ? __ldg(src + 2) : 0.f;
        xv[it].w = c4 + 3 < rows ? __ldg(src + 3) : 0.f;
      }
    }
  }
  // rmsnorm scale per row (query): alpha / sqrt(sum_j ssq[j][m] / K + eps), the partials staged
  // by all threads at once and added in order by thread m
  float* ssq_sm = red;  // [parts][16] (red is free until the GEMM)
  const bool norm = p.ssq_in != nullptr;
  if (norm)
    for (int i = tid; i < p.norm_parts * kPjM; i += kPjThreads) {
      const int j = i / kPjM, m = i % kPjM;
      ssq_sm[i] = m < p.M ? __ldg(p.ssq_in + size_t(j) * p.M + m) : 0.f;
    }
  __syncthreads();
  if (tid < kPjM) {
    float sc = 1.f;
    if (norm && tid < p.M) {
      float t = 0.f;
      for (int j = 0; j < p.norm_parts; ++j) t += ssq_sm[j * kPjM + tid];
      sc = p.norm_alpha * rsqrtf(t / float(p.K) + p.eps);
    }
    rscale[tid] = sc;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kXIter; ++it) {
    const int i = tid + it * kPjThreads;
    if (i >= kPjM * q4) break;
    const int r = i / q4, c4 = (i % q4) * 4;
    const float sc = rscale[r];
    float v[4] = {xv[it].x * sc, xv[it].y * sc, xv[it].z * sc, xv[it].w * sc};
    __nv_bfloat16 h[4];
    float lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      h[j] = __float2bfloat16_rn(v[j]);
      lo[j] = v[j] - __bfloat162float(h[j]);
    }
    uint2 hv, lv;
    hv.x = pack_bf16_raw(h[0], h[1]);
    hv.y = pack_bf16_raw(h[2], h[3]);
    lv.x = pack_bf16(lo[0], lo[1]);
    lv.y = pack_bf16(lo[2], lo[3]);
    *reinterpret_cast<uint2*>(xt + r * kPjXRow + c4 * 2) = hv;
    *reinterpret_cast<uint2*>(xt + kPjM * kPjXRow + r * kPjXRow + c4 * 2) = lv;
  }
  __syncthreads();
  pj_stamp(p, 2);
  // ---- GEMM: warp (column group cg, box half kh)
  const int cg = warp & 3, kh = warp >> 2, q = lane >> 3, g = lane >> 2, t4 = lane & 3;
  const int half = (nbox + 1) / 2;
  const int b_lo = kh == 0 ? 0 : half, b_hi = kh == 0 ? half : nbox;
  // hi and lo planes into separate accumulators (summed at the end): independent mma.sync chains
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}}, acl[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  for (int b = b_lo; b < b_hi; ++b) {
    mbar_wait(&bars[b], 0);
    if (b == 0) pj_stamp(p, 3);
    const uint32_t wb = wt_u32 + b * kPjBox * kPjNC * 2;
#pragma unroll
    for (int kk = 0; kk < kPjBox / 16; ++kk) {
      const int ka = b * kPjBox + kk * 16;  // within the X planes
      uint32_t ahi[4], alo[4], bf[4];
      const uint32_t aoff = ((lane & 7) + (q & 1) * 8) * kPjXRow + (ka + (q >> 1) * 8) * 2;
      ldmatrix_x4(ahi, xt_u32 + aoff);
      ldmatrix_x4(alo, xt_u32 + kPjM * kPjXRow + aoff);
      const int kr = kk * 16 + (q & 1) * 8 + (lane & 7);  // row within the box
      ldmatrix_x4_trans(bf, wb + kr * 128 + (((cg * 2 + (q >> 1)) ^ (kr & 7)) * 16));
      mma_m16n8k16_bf16(acc[0], ahi, bf[0], bf[1]);
      mma_m16n8k16_bf16(acl[0], alo, bf[0], bf[1]);
      mma_m16n8k16_bf16(acc[1], ahi, bf[2], bf[3]);
      mma_m16n8k16_bf16(acl[1], alo, bf[2], bf[3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[j][e] += acl[j][e];
  __syncthreads();  // every warp is done with the X planes: the partials reuse them
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int col = cg * 16 + j * 8 + 2 * t4;
    red[(kh * kPjM + g) * kPjNC + col] = acc[j][0];
    red[(kh * kPjM + g) * kPjNC + col + 1] = acc[j][1];
    red[(kh * kPjM + g + 8) * kPjNC + col] = acc[j][2];
    red[(kh * kPjM + g + 8) * kPjNC + col + 1] = acc[j][3];
  }
  __syncthreads();
  pj_stamp(p, 4);
  // slab partial of this slice -> cluster rank 0's slot [ks] (DSMEM; rank 0 stores locally),
  // once every CTA of the cluster is known to run (its shared memory exists)
  cluster_wait_acquire();
  const uint32_t slot_u32 = mapa_shared(smem_u32(slots + ks * kPjM * kPjNC), 0);
  for (int i = tid; i < kPjM * kPjNC; i += kPjThreads) st_shared_cluster_f32(slot_u32 + i * 4, red[i] + red[kPjM * kPjNC + i]);
  cluster_arrive_release();
  cluster_wait_acquire();
  pj_stamp(p, 5);
  if (ks != 0) return;  // rank 0 of the cluster (ks == cluster rank: the cluster spans x)
  for (int i = tid; i < kPjM * kPjNC; i += kPjThreads) {
    float s = 0.f;
    for (int j = 0; j < KS; ++j) s += slots[j * kPjM * kPjNC + i];
    red[i] = s;  // final slab tile [16][64]
  }
  __syncthreads();
  if (p.mode == 0) {
    for (int i = tid; i < p.M * kPjNC; i += kPjThreads) {
      const int r = i / kPjNC, c = i % kPjNC, n = n0 + c;
      if (n >= p.seg_end[2]) continue;  // (zero pad columns of the packed weight)
      const int sgi = n < p.seg_end[0] ? 0 : (n < p.seg_end[1] ? 1 : 2);
      const int sb = sgi == 0 ? 0 : p.seg_end[sgi - 1];
      float* o = p.seg_out[sgi];
      if (o != nullptr) o[size_t(r) * (p.seg_end[sgi] - sb) + (n - sb)] = red[i];
    }
    if (p.ssq_out != nullptr && n0 < p.ssq_cols && tid < p.M) {  // this slab's partial sum of squares
      float s = 0.f;
      const int ce = min(kPjNC, p.ssq_cols - n0);
      for (int c = 0; c < ce; ++c) s = fmaf(red[tid * kPjNC + c], red[tid * kPjNC + c], s);
      p.ssq_out[size_t(slab) * p.M + tid] = s;
    }
    return;
  }
  // query epilogue: pairs of columns (c, c+1), c even
  for (int i = tid; i < p.M * (kPjNC / 2); i += kPjThreads) {
    const int r = i / (kPjNC / 2), c = 2 * (i % (kPjNC / 2)), n = n0 + c;
    if (n >= p.nq + p.H * p.dr) continue;  // (zero pad columns of the packed weight)
    const float y0 = red[r * kPjNC + c], y1 = red[r * kPjNC + c + 1];
    if (n < p.nq) {
      __nv_bfloat16* o = p.q_out + size_t(r) * p.nq + n;
      o[0] = __float2bfloat16_rn(y0 * p.q_scale);
      if (n + 1 < p.nq) o[1] = __float2bfloat16_rn(y1 * p.q_scale);
      continue;
    }
    const int j = n - p.nq, h = j / p.dr, l = (j % p.dr) / 2;
    const double a = double(p.pos[r] + p.pos_delta) * p.theta[l];
    const double two_pi = 6.283185307179586476925286766559;
    float sn, cs;
    sincosf(float(a - two_pi * floor(a * (1.0 / two_pi))), &sn, &cs);
    const float e = (y0 * cs - y1 * sn) * p.r_scale, o = (y0 * sn + y1 * cs) * p.r_scale;
    reinterpret_cast<__nv_bfloat162*>(p.r_out + (size_t(r) * p.H + h) * p.drp)[l] = __floats2bfloat162_rn(e, o);
  }
}

}  // namespace mlra
