// K0 (paged append), K1 (query absorption) and K3 (split merge + W^UV up-projection +
// branch sum), the small kernels around the K2 decode kernel.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include <cmath>

namespace mlra {

// ----------------------------------------------------------------------------- K0
// attnkit/decode.py:129-150 (append_owned) + cache.py:44-57: write one token row per
// sequence into its page. rows [B, W] bf16; positions [B] = slot index of the new token.
__global__ void cache_append_kernel(const __nv_bfloat16* __restrict__ rows, const int32_t* __restrict__ block_table,
                                    const int32_t* __restrict__ positions, int W, int page_size, int max_pages,
                                    __nv_bfloat16* __restrict__ pool) {
  const int s = blockIdx.x;
  const int pos = positions[s];
  const int page = block_table[size_t(s) * max_pages + pos / page_size];
  __nv_bfloat16* dst = pool + (size_t(page) * page_size + pos % page_size) * W;
  const __nv_bfloat16* src = rows + size_t(s) * W;
  for (int i = threadIdx.x; i < W / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
}

// ----------------------------------------------------------------------------- per-head GEMM
// Y[s, h, n] = scale * sum_k X[s, h, k] * W[h][k][n] for a batch of sequences, one weight
// matrix per head. Used twice:
//   K1 (query absorption, decode.py:155-167 / :224): X = q_nope [B, H, DH] (bf16),
//      W = W^UK packed [H][DH][NB*DLAT], Y = q~ written bf16 to [B, NB, H, DLAT]; the CTAs of
//      column block 0 also scale q_rope into its output buffer;
//   K3b (value up-projection, decode.py:228): X = merged latent Z [B, H, NB*DLAT] (fp32),
//      W = W^UV packed [H][NB*DLAT][DH], Y = out fp32 [B, H, DH] (branches summed over K in
//      ascending order), or per branch [B, NB, H, DH] when the K range is partitioned.
// CTA tile: one head, NT output columns, 8 sequences, the whole K extent resident in smem
// (one round trip of independent 16-byte loads). Warp = sequence, lane = NT/32 columns.
constexpr int kHG_S = 8, kHG_THREADS = 256;

template <typename Tx, bool kOutBf16, int NT>
__global__ void __launch_bounds__(kHG_THREADS)
head_gemm_kernel(const Tx* __restrict__ X, const __nv_bfloat16* __restrict__ W, void* __restrict__ Y, int B, int H,
                 int K, int N, int kparts, float scale, int out_nb, int out_dlat,
                 const __nv_bfloat16* __restrict__ rope_in, __nv_bfloat16* __restrict__ rope_out, int DR) {
  constexpr int CPL = NT / 32;  // columns per lane
  extern __shared__ __align__(16) uint8_t hg_smem[];
  const int nblk = blockIdx.x, h = blockIdx.y;
  const int sblk = blockIdx.z / kparts, part = blockIdx.z % kparts;
  const int kp = K / kparts, k_begin = part * kp;
  __nv_bfloat16* ws = reinterpret_cast<__nv_bfloat16*>(hg_smem);                       // [kp][NT]
  float* xs = reinterpret_cast<float*>(hg_smem + ((size_t(kp) * NT * 2 + 15) / 16) * 16);  // [kHG_S][kp]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = nblk * NT;
  for (int i = threadIdx.x; i < kp * NT / 8; i += kHG_THREADS) {
    const int r = i / (NT / 8), c8 = i % (NT / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n0 + c8 * 8 < N) v = *reinterpret_cast<const uint4*>(W + (size_t(h) * K + k_begin + r) * N + n0 + c8 * 8);
    *reinterpret_cast<uint4*>(ws + size_t(r) * NT + c8 * 8) = v;
  }
  for (int i = threadIdx.x; i < kHG_S * kp; i += kHG_THREADS) {
    const int ss = i / kp, kk = i % kp;
    const int sg = sblk * kHG_S + ss;
    float v = 0.f;
    if (sg < B) {
      if constexpr (sizeof(Tx) == 2)
        v = __bfloat162float(X[(size_t(sg) * H + h) * K + k_begin + kk]);
      else
        v = X[(size_t(sg) * H + h) * K + k_begin + kk];
    }
    xs[ss * kp + kk] = v;
  }
  if (rope_out != nullptr && nblk == 0) {
    for (int i = threadIdx.x; i < kHG_S * DR; i += kHG_THREADS) {
      const int sg = sblk * kHG_S + i / DR;
      if (sg < B) {
        const size_t off = (size_t(sg) * H + h) * DR + i % DR;
        rope_out[off] = __float2bfloat16(__bfloat162float(rope_in[off]) * scale);
      }
    }
  }
  __syncthreads();
  const int s = sblk * kHG_S + warp;
  if (s >= B) return;
  float acc[CPL];
#pragma unroll
  for (int j = 0; j < CPL; ++j) acc[j] = 0.f;
  const float* xr = xs + warp * kp;
#pragma unroll 4
  for (int kk = 0; kk < kp; ++kk) {
    const float xv = xr[kk];
    if constexpr (CPL == 4) {
      const uint2 wv = *reinterpret_cast<const uint2*>(ws + size_t(kk) * NT + lane * 4);
      const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
      const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
      acc[0] = fmaf(xv, w01.x, acc[0]);
      acc[1] = fmaf(xv, w01.y, acc[1]);
      acc[2] = fmaf(xv, w23.x, acc[2]);
      acc[3] = fmaf(xv, w23.y, acc[3]);
    } else {
#pragma unroll
      for (int j = 0; j < CPL; ++j) acc[j] = fmaf(xv, __bfloat162float(ws[size_t(kk) * NT + lane * CPL + j]), acc[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < CPL; ++j) {
    const int n = n0 + lane * CPL + j;
    if (n >= N) continue;
    const float v = acc[j] * scale;
    if constexpr (kOutBf16) {
      // K1 output layout [B, NB, H, DLAT]: column n -> (branch n / DLAT, latent n % DLAT)
      const int b = n / out_dlat, c = n % out_dlat;
      reinterpret_cast<__nv_bfloat16*>(Y)[((size_t(s) * out_nb + b) * H + h) * out_dlat + c] = __float2bfloat16(v);
    } else {
      // K3b output layout [B, kparts, H, N]
      reinterpret_cast<float*>(Y)[((size_t(s) * kparts + part) * H + h) * N + n] = v;
    }
  }
}

template <int NT>
inline size_t head_gemm_smem(int kp) {
  return ((size_t(kp) * NT * 2 + 15) / 16) * 16 + size_t(kHG_S) * kp * 4;
}

// ----------------------------------------------------------------------------- K3a
// Flash-decoding merge of the K2 split partials: for every (sequence, branch, head) row,
//   Z = sum_k w_k O_k with w_k = 2^(lse_k - max) / sum_j 2^(lse_j - max).
// One warp per row: lane k < nsplit computes split k's weight once (shuffled to all
// lanes), then every lane sums its latent columns over the splits with independent loads.
// Output [B, H, NB*DLAT] (the K3b input) or, with zout_bnh, [B, NB, H, DLAT] * alpha.
constexpr int kMergeMaxSplits = 64;
__global__ void merge_splits_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part,
                                    float* __restrict__ z, int B, int NB, int H, int DLAT, int nsplit, float alpha,
                                    int zout_bnh) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= B * NB * H) return;
  const int h = row % H, b = (row / H) % NB, s = row / (H * NB);
  const float* l = lse_part + (size_t(s) * nsplit * NB + b) * H + h;  // split stride NB*H
  float lk[2];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int k = lane + 32 * j;
    lk[j] = k < nsplit ? l[size_t(k) * NB * H] : -INFINITY;
    m = fmaxf(m, lk[j]);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float wk[2], tot = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    wk[j] = (m == -INFINITY || lk[j] == -INFINITY) ? 0.f : exp2f(lk[j] - m);
    tot += wk[j];
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
  const float inv = tot > 0.f ? 1.f / tot : 0.f;
  const float* o = o_part + ((size_t(s) * nsplit * NB + b) * H + h) * DLAT;  // split stride NB*H*DLAT
  float* dst = zout_bnh ? z + ((size_t(s) * NB + b) * H + h) * DLAT : z + (size_t(s) * H + h) * (NB * DLAT) + b * DLAT;
  const float sc = (zout_bnh ? alpha : 1.f) * inv;
  const size_t sstride = size_t(NB) * H * DLAT;
  for (int c0 = 0; c0 < DLAT; c0 += 32 * 4) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < nsplit; ++k) {
      const float w = __shfl_sync(0xffffffffu, wk[k >> 5], k & 31);
      if (w == 0.f) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + lane + 32 * j;
        if (c < DLAT) acc[j] = fmaf(w, o[k * sstride + c], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + lane + 32 * j;
      if (c < DLAT) dst[c] = acc[j] * sc;
    }
  }
}

}  // namespace mlra
