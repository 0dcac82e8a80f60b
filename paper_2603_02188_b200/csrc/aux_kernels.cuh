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

// ----------------------------------------------------------------------------- K1
// attnkit/decode.py:155-167 (absorb_query), used per branch at decode.py:224:
//   q~[s, b, h, c] = scale * sum_p q_nope[s, h, p] * W^UK[b*DLAT + c, h*DH + p]
// w_uk is pre-packed per head as [H][DH][NCOL] (NCOL = NB*DLAT, latent contiguous), so a
// thread owns two adjacent latent columns and streams its column of the head's matrix.
// Also writes q_rope * scale. scale = tau * log2(e) (scores are consumed in the log2 domain).
template <int SEQ>
__global__ void absorb_query_kernel(const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ q_rope,
                                    const __nv_bfloat16* __restrict__ w_uk, __nv_bfloat16* __restrict__ q_abs,
                                    __nv_bfloat16* __restrict__ q_rope_out, int B, int H, int DH, int NCOL, int DLAT,
                                    int DR, float scale) {
  extern __shared__ float qs[];  // [SEQ][DH]
  const int h = blockIdx.x, s0 = blockIdx.y * SEQ;
  const int nseq = min(SEQ, B - s0);
  for (int i = threadIdx.x; i < SEQ * DH; i += blockDim.x) {
    const int j = i / DH, pp = i % DH;
    qs[i] = j < nseq ? __bfloat162float(q_nope[(size_t(s0 + j) * H + h) * DH + pp]) : 0.f;
  }
  __syncthreads();
  const __nv_bfloat162* w = reinterpret_cast<const __nv_bfloat162*>(w_uk + size_t(h) * DH * NCOL);
  for (int c2 = threadIdx.x; c2 < NCOL / 2; c2 += blockDim.x) {
    float acc[SEQ][2];
#pragma unroll
    for (int j = 0; j < SEQ; ++j) acc[j][0] = acc[j][1] = 0.f;
    for (int pp = 0; pp < DH; ++pp) {
      const float2 wv = __bfloat1622float2(w[size_t(pp) * (NCOL / 2) + c2]);
#pragma unroll
      for (int j = 0; j < SEQ; ++j) {
        acc[j][0] = fmaf(qs[j * DH + pp], wv.x, acc[j][0]);
        acc[j][1] = fmaf(qs[j * DH + pp], wv.y, acc[j][1]);
      }
    }
    // output [B, NB, H, DLAT] with NCOL = NB*DLAT: column c -> (b = c / DLAT, c % DLAT)
    const int c = 2 * c2, b = c / DLAT, cc = c % DLAT;
    const int NB = NCOL / DLAT;
    for (int j = 0; j < nseq; ++j) {
      __nv_bfloat162 v = __floats2bfloat162_rn(acc[j][0] * scale, acc[j][1] * scale);
      *reinterpret_cast<__nv_bfloat162*>(q_abs + ((size_t(s0 + j) * NB + b) * H + h) * DLAT + cc) = v;
    }
  }
  for (int i = threadIdx.x; i < nseq * DR; i += blockDim.x) {
    const int j = i / DR, rr = i % DR;
    const size_t off = (size_t(s0 + j) * H + h) * DR + rr;
    q_rope_out[off] = __float2bfloat16(__bfloat162float(q_rope[off]) * scale);
  }
}

// ----------------------------------------------------------------------------- K3
// Merge the split partials of K2 (flash-decoding LSE merge), then
//   out[s, h, :] = alpha * sum_b Z_b[s, h, :] . W^UV_b[:, h]      (decode.py:228 + :274-285)
// w_uv packed per head as [H][NCOL][DH] (NCOL = NB*DLAT, DH contiguous).
// Branches are summed in ascending order inside one fp32 accumulator (the reference's
// reduce_contributions order, decode.py:276-278, up to fp reassociation).
// upproj == 0: no up-projection (GQA / raw latent output): out[s, b, h, :DLAT] = Z_b.
template <int SEQ>
__global__ void combine_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part,
                               const __nv_bfloat16* __restrict__ w_uv, float* __restrict__ out, int B, int H, int NB,
                               int DLAT, int DH, int nsplit, float alpha, int upproj) {
  extern __shared__ float z[];  // [SEQ][NB*DLAT]
  const int h = blockIdx.x, s0 = blockIdx.y * SEQ;
  const int nseq = min(SEQ, B - s0);
  const int NCOL = NB * DLAT;
  __shared__ float wsh[SEQ * 4][64];  // per (seq, branch) split weights (nsplit <= 64)
  for (int i = threadIdx.x; i < nseq * NB; i += blockDim.x) {
    const int j = i / NB, b = i % NB;
    float m = -INFINITY;
    for (int k = 0; k < nsplit; ++k) m = fmaxf(m, lse_part[((size_t(s0 + j) * nsplit + k) * NB + b) * H + h]);
    float tot = 0.f;
    for (int k = 0; k < nsplit; ++k) {
      const float l = lse_part[((size_t(s0 + j) * nsplit + k) * NB + b) * H + h];
      const float w = (m == -INFINITY) ? 0.f : exp2f(l - m);
      wsh[i][k] = w;
      tot += w;
    }
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
    for (int k = 0; k < nsplit; ++k) wsh[i][k] *= inv;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nseq * NCOL; i += blockDim.x) {
    const int j = i / NCOL, col = i % NCOL, b = col / DLAT, c = col % DLAT;
    float acc = 0.f;
    for (int k = 0; k < nsplit; ++k) {
      const float w = wsh[j * NB + b][k];
      if (w != 0.f) acc += w * o_part[(((size_t(s0 + j) * nsplit + k) * NB + b) * H + h) * DLAT + c];
    }
    z[j * NCOL + col] = acc;
  }
  __syncthreads();
  if (!upproj) {
    for (int i = threadIdx.x; i < nseq * NCOL; i += blockDim.x) {
      const int j = i / NCOL, col = i % NCOL, b = col / DLAT, c = col % DLAT;
      out[((size_t(s0 + j) * NB + b) * H + h) * DLAT + c] = alpha * z[j * NCOL + col];
    }
    return;
  }
  // thread -> (d pair, k slice); partial sums over k slices reduced through smem.
  // upproj == 1: one accumulation over all NB*DLAT latent columns (ascending branch order)
  //              -> out[s, h, :];  upproj == 2: per branch -> out[s, b, h, :] (no branch sum).
  const int DH2 = DH / 2;
  const int kslices = blockDim.x / DH2;
  const int d2 = threadIdx.x % DH2, ks = threadIdx.x / DH2;
  const __nv_bfloat162* w = reinterpret_cast<const __nv_bfloat162*>(w_uv + size_t(h) * NCOL * DH);
  const int nout = (upproj == 2) ? NB : 1;
  const int kspan = (upproj == 2) ? DLAT : NCOL;
  float* red = z + SEQ * NCOL;  // [kslices][SEQ][DH] (host sizes the smem for both regions)
  for (int ob = 0; ob < nout; ++ob) {
    float acc[SEQ][2];
#pragma unroll
    for (int j = 0; j < SEQ; ++j) acc[j][0] = acc[j][1] = 0.f;
    if (ks < kslices) {
      for (int k = ob * kspan + ks; k < (ob + 1) * kspan; k += kslices) {
        const float2 wv = __bfloat1622float2(w[size_t(k) * DH2 + d2]);
#pragma unroll
        for (int j = 0; j < SEQ; ++j) {
          const float zz = z[j * NCOL + k];
          acc[j][0] = fmaf(zz, wv.x, acc[j][0]);
          acc[j][1] = fmaf(zz, wv.y, acc[j][1]);
        }
      }
#pragma unroll
      for (int j = 0; j < SEQ; ++j) {
        red[(ks * SEQ + j) * DH + 2 * d2] = acc[j][0];
        red[(ks * SEQ + j) * DH + 2 * d2 + 1] = acc[j][1];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nseq * DH; i += blockDim.x) {
      const int j = i / DH, d = i % DH;
      float v = 0.f;
      for (int k = 0; k < kslices; ++k) v += red[(k * SEQ + j) * DH + d];
      if (upproj == 2) out[((size_t(s0 + j) * NB + ob) * H + h) * DH + d] = alpha * v;
      else out[(size_t(s0 + j) * H + h) * DH + d] = alpha * v;
    }
    __syncthreads();
  }
}

}  // namespace mlra
