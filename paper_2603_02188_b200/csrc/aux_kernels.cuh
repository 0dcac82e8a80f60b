// K0 (paged append), K1 (query absorption) and K3 (split merge + W^UV up-projection +
// branch sum), the small kernels around the K2 decode kernel.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include <cmath>
#include "ptx.cuh"

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


// acc[0..8) += x * (8 bf16 of w)
__device__ __forceinline__ void fma8(float (&acc)[8], float x, const uint4& w) {
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(w2[j]);
    acc[2 * j] = fmaf(x, f.x, acc[2 * j]);
    acc[2 * j + 1] = fmaf(x, f.y, acc[2 * j + 1]);
  }
}

// ----------------------------------------------------------------------------- K1
// Query absorption (attnkit/decode.py:155-167, used per branch at :224):
//   q_abs[s, b, h, c] = scale * sum_p q_nope[s, h, p] * W^UK_b[c, h, p]
// with W^UK packed [H][DH][NB*DLAT] (column n -> branch n / DLAT, latent n % DLAT) and
// scale = tau * log2(e) folded in for K2's log2-domain softmax; CTAs of column block 0
// also write q_rope * scale. One CTA per (32-column block, head), 16 sequences per pass:
// the W^UK tile [DH x 32] and the queries are staged in smem with one round trip of
// independent 16-byte loads; thread = (sequence, 8-column octet, quarter of DH) runs
// DH/4 x 8 FMAs and the quarters are summed with two shuffles.
// Triggers the dependent launch at entry so K2 (PDL) can start streaming the cache.
constexpr int kAbsCols = 32, kAbsThreads = 256, kAbsSeqs = 16;
__global__ void __launch_bounds__(kAbsThreads)
absorb_kernel(const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ w_uk,
              __nv_bfloat16* __restrict__ q_abs, int B, int H, int DH, int NB, int DLAT, float scale,
              const __nv_bfloat16* __restrict__ rope_in, __nv_bfloat16* __restrict__ rope_out, int DR) {
  griddep_launch_dependents();
  griddep_wait();  // q_nope comes from the previous kernel on the stream
  extern __shared__ __align__(16) uint4 abs_smem[];
  uint4* ws = abs_smem;            // [DH][4]: W^UK[h][p][c0 .. c0+32)
  uint4* xs = abs_smem + DH * 4;   // [kAbsSeqs][DH/8]: q_nope rows of this pass
  const int NCOL = NB * DLAT;
  const int h = blockIdx.y, c0 = blockIdx.x * kAbsCols, tid = threadIdx.x;
  const int o = tid & 3, qk = (tid >> 2) & 3, sl = tid >> 4;
  const int col = c0 + o * 8;
  for (int i = tid; i < DH * 4; i += kAbsThreads) {
    const int k = i >> 2, oo = i & 3;
    ws[i] = (c0 + oo * 8 < NCOL) ? __ldg(reinterpret_cast<const uint4*>(w_uk + (size_t(h) * DH + k) * NCOL + c0 + oo * 8))
                                  : make_uint4(0, 0, 0, 0);
  }
  if (blockIdx.x == 0 && rope_out != nullptr) {
    for (int i = tid; i < B * DR; i += kAbsThreads) {
      const size_t off = (size_t(i / DR) * H + h) * DR + i % DR;
      rope_out[off] = __float2bfloat16(__bfloat162float(rope_in[off]) * scale);
    }
  }
  const int xw = DH / 8, kq = xw / 4;  // 16-byte words per row, per quarter (DH % 32 == 0)
  for (int s0 = 0; s0 < B; s0 += kAbsSeqs) {
    const int ns = min(kAbsSeqs, B - s0);
    if (s0 > 0) __syncthreads();
    for (int i = tid; i < ns * xw; i += kAbsThreads)
      xs[i] = __ldg(reinterpret_cast<const uint4*>(q_nope + (size_t(s0 + i / xw) * H + h) * DH) + i % xw);
    __syncthreads();
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (sl < ns) {
      const uint4* xr = xs + sl * xw + qk * kq;
      const uint4* wq = ws + qk * kq * 8 * 4;
      for (int k8 = 0; k8 < kq; ++k8) {
        const uint4 xv = xr[k8];
        const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 xf = __bfloat1622float2(x2[j]);
          fma8(acc, xf.x, wq[(k8 * 8 + 2 * j) * 4 + o]);
          fma8(acc, xf.y, wq[(k8 * 8 + 2 * j + 1) * 4 + o]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 4);
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 8);
    }
    if (qk == 0 && sl < ns && col < NCOL) {
      const int b = col / DLAT, cc = col % DLAT;
      uint4 v;
      v.x = pack_bf16(acc[0] * scale, acc[1] * scale);
      v.y = pack_bf16(acc[2] * scale, acc[3] * scale);
      v.z = pack_bf16(acc[4] * scale, acc[5] * scale);
      v.w = pack_bf16(acc[6] * scale, acc[7] * scale);
      *reinterpret_cast<uint4*>(q_abs + ((size_t(s0 + sl) * NB + b) * H + h) * DLAT + cc) = v;
    }
  }
}

inline size_t absorb_smem(int DH) { return size_t(DH) * 4 * 16 + size_t(kAbsSeqs) * (DH / 8) * 16; }

// ----------------------------------------------------------------------------- K3
// Split merge + value up-projection in one kernel (attnkit/decode.py:228 per branch, then
// reduce_contributions :264-285 summing the branches in ascending order):
//   w_k = 2^(lse_k - max) / sum_j 2^(lse_j - max)         (per sequence, branch, head)
//   Z_b = sum_k w_k O_k                                      (merged latent, fp32)
//   out[s, h, :] = alpha * sum_b Z_b . W^UV_b[h]            (per_branch = 0)
//   out[s, b, h, :] = alpha * Z_b . W^UV_b[h]               (per_branch = 1)
// One CTA per (head, 4 sequences). W^UV[h] ([NB*DLAT][DH] bf16, <= 128 KB) does not depend
// on K2, so its bulk copy into smem is issued before griddepcontrol.wait; then the split
// weights and merged latents (smem), then thread (sequence, 4-column quad of d, half of the
// latent rows) accumulates per branch and the two halves are added through smem.
constexpr int kCmbSeqs = 4, kCmbThreads = 256;
// smem: W^UV [NCOL][DH] bf16 | Z [4][NCOL] | weights [4][NB][nsplit] | red [4][4][DH] | mbarriers
//       | (staged = 1) partials [4][nsplit][NB][DLAT] fp32
inline size_t combine_smem(int NB, int DLAT, int DH, int nsplit, int staged) {
  const size_t w = size_t(NB) * DLAT * DH * 2;
  const size_t z = size_t(kCmbSeqs) * NB * DLAT * 4;
  const size_t wt = size_t(kCmbSeqs) * NB * nsplit * 4;
  const size_t red = size_t(kCmbSeqs) * 4 * DH * 4;
  const size_t parts = staged ? size_t(kCmbSeqs) * nsplit * NB * DLAT * 4 : 0;
  return ((w + z + wt + red + 15) / 16) * 16 + 16 + parts;
}

__global__ void __launch_bounds__(kCmbThreads)
combine_upproj_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part,
                      const __nv_bfloat16* __restrict__ w_uv, float* __restrict__ out, int B, int H, int NB, int DLAT,
                      int DH, int nsplit, float alpha, int per_branch, int staged) {
  extern __shared__ __align__(128) uint8_t cmb_smem[];
  const int NCOL = NB * DLAT;
  const __nv_bfloat16* wsm = reinterpret_cast<const __nv_bfloat16*>(cmb_smem);      // [NCOL][DH]
  float* zs = reinterpret_cast<float*>(cmb_smem + size_t(NCOL) * DH * 2);          // [kCmbSeqs][NCOL]
  float* wts = zs + kCmbSeqs * NCOL;                                               // [kCmbSeqs][NB][nsplit]
  float* red = wts + kCmbSeqs * NB * nsplit;                                       // [kCmbSeqs][4][DH]
  const size_t head_bytes =
      ((size_t(NCOL) * DH * 2 + (kCmbSeqs * NCOL + kCmbSeqs * NB * nsplit + kCmbSeqs * 4 * DH) * 4 + 15) / 16) * 16;
  uint64_t* bar = reinterpret_cast<uint64_t*>(cmb_smem + head_bytes);  // [0] W^UV, [1] partials
  float* parts = reinterpret_cast<float*>(cmb_smem + head_bytes + 16);  // [4][nsplit][NB][DLAT]
  const int h = blockIdx.x, s0 = blockIdx.y * kCmbSeqs, tid = threadIdx.x;
  const int ns = min(kCmbSeqs, B - s0);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint32_t wbytes = uint32_t(NCOL) * DH * 2;
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], wbytes);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(w_uv + size_t(h) * NCOL * DH);
    for (uint32_t off = 0; off < wbytes; off += 65536)
      bulk_copy_g2s(cmb_smem + off, src + off, min(65536u, wbytes - off), &bar[0]);
  }
  griddep_wait();  // partials of K2
  if (staged && tid < 32) {
    // every (sequence, split, branch) row of this head: DLAT contiguous floats
    const int nrows = ns * nsplit * NB;
    if (tid == 0) mbar_arrive_expect_tx(&bar[1], uint32_t(nrows) * DLAT * 4);
    __syncwarp();
    for (int i = tid; i < nrows; i += 32) {
      const int s = i / (nsplit * NB), kb = i % (nsplit * NB);  // kb = k * NB + b
      bulk_copy_g2s(parts + size_t(i) * DLAT, o_part + ((size_t(s0 + s) * nsplit * NB + kb) * H + h) * DLAT,
                    uint32_t(DLAT) * 4, &bar[1]);
    }
  }
  // split weights, one thread per (sequence, branch)
  for (int i = tid; i < ns * NB; i += kCmbThreads) {
    const int s = i / NB, b = i % NB;
    const float* l = lse_part + (size_t(s0 + s) * nsplit * NB + b) * H + h;  // split stride NB*H
    float m = -INFINITY;
    for (int k = 0; k < nsplit; ++k) m = fmaxf(m, l[size_t(k) * NB * H]);
    float tot = 0.f;
    float* wr = wts + i * nsplit;
    for (int k = 0; k < nsplit; ++k) {
      const float lk = l[size_t(k) * NB * H];
      const float w = (m == -INFINITY || lk == -INFINITY) ? 0.f : ex2(lk - m);
      wr[k] = w;
      tot += w;
    }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
    for (int k = 0; k < nsplit; ++k) wr[k] *= inv;
  }
  __syncthreads();
  // merged latents
  if (staged) {
    mbar_wait(&bar[1], 0);
    for (int i = tid; i < ns * NCOL; i += kCmbThreads) {
      const int s = i / NCOL, col = i % NCOL, b = col / DLAT, c = col % DLAT;
      const float* wr = wts + (s * NB + b) * nsplit;
      const float* pr = parts + (size_t(s) * nsplit * NB + b) * DLAT + c;
      float acc = 0.f;
      for (int k = 0; k < nsplit; ++k) acc = fmaf(wr[k], pr[size_t(k) * NB * DLAT], acc);
      zs[i] = acc;
    }
  }
  const size_t kstride = size_t(NB) * H * DLAT;
  for (int i = staged ? ns * NCOL : tid; i < ns * NCOL; i += kCmbThreads) {
    const int s = i / NCOL, col = i % NCOL, b = col / DLAT, c = col % DLAT;
    const float* o = o_part + ((size_t(s0 + s) * nsplit * NB + b) * H + h) * DLAT + c;
    const float* wr = wts + (s * NB + b) * nsplit;
    // up to 16 split loads in flight per pass (independent addresses, one round trip)
    float acc = 0.f;
    for (int k0 = 0; k0 < nsplit; k0 += 16) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = (k0 + j < nsplit) ? __ldcg(o + size_t(k0 + j) * kstride) : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j < nsplit) acc = fmaf(wr[k0 + j], v[j], acc);
    }
    zs[i] = acc;
  }
  __syncthreads();
  mbar_wait(&bar[0], 0);
  // up-projection: thread = (half of the latent rows, sequence, quad of d); 2 * 4 * DH/4 <= 256
  // items for DH <= 128 (host-checked), so one uniform pass around the __syncthreads below
  const int nq = DH / 4;
  {
    const int item = tid;
    const bool valid = item < 2 * kCmbSeqs * nq;
    const int half = valid ? item / (kCmbSeqs * nq) : 2, s = (item / nq) % kCmbSeqs, dq = item % nq;
    float acc[4][4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[b][j] = 0.f;
    if (valid && s < ns) {
      const int rows = (DLAT + 1) / 2;
      const int r0 = half * rows, r1 = min(DLAT, r0 + rows);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (b >= NB) break;
        const float* z = zs + s * NCOL + b * DLAT;
        const __nv_bfloat16* wb = wsm + size_t(b) * DLAT * DH + dq * 4;
#pragma unroll 4
        for (int r = r0; r < r1; ++r) {
          const float zv = z[r];
          const uint2 wv = *reinterpret_cast<const uint2*>(wb + size_t(r) * DH);
          const float2 w01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.x));
          const float2 w23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv.y));
          acc[b][0] = fmaf(zv, w01.x, acc[b][0]);
          acc[b][1] = fmaf(zv, w01.y, acc[b][1]);
          acc[b][2] = fmaf(zv, w23.x, acc[b][2]);
          acc[b][3] = fmaf(zv, w23.y, acc[b][3]);
        }
      }
    }
    if (half == 1) {
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (b < NB) *reinterpret_cast<float4*>(red + (s * 4 + b) * DH + dq * 4) = make_float4(acc[b][0], acc[b][1], acc[b][2], acc[b][3]);
    }
    __syncthreads();
    if (half == 0 && s < ns) {
      float tot[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (b >= NB) break;
        const float4 o1 = *reinterpret_cast<const float4*>(red + (s * 4 + b) * DH + dq * 4);
        const float v0 = (acc[b][0] + o1.x) * alpha, v1 = (acc[b][1] + o1.y) * alpha;
        const float v2 = (acc[b][2] + o1.z) * alpha, v3 = (acc[b][3] + o1.w) * alpha;
        if (per_branch) {
          *reinterpret_cast<float4*>(out + ((size_t(s0 + s) * NB + b) * H + h) * DH + dq * 4) = make_float4(v0, v1, v2, v3);
        } else {
          tot[0] += v0; tot[1] += v1; tot[2] += v2; tot[3] += v3;
        }
      }
      if (!per_branch)
        *reinterpret_cast<float4*>(out + (size_t(s0 + s) * H + h) * DH + dq * 4) = make_float4(tot[0], tot[1], tot[2], tot[3]);
    }
  }
}

}  // namespace mlra
