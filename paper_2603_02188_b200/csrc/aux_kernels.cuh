// K0 (paged append), K1 (query absorption) and K3 (split merge + W^UV up-projection +
// branch sum), the small kernels around the K2 decode kernel.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>
#include <cmath>
#include "ptx.cuh"
#include "allreduce_kernel.cuh"
#include "fused_step.cuh"

namespace mlra {

// Dev-only phase stamps for the small kernels (tools/small_trace.cu defines MLRA_SMALL_TRACE).
#ifdef MLRA_SMALL_TRACE
__device__ unsigned long long g_small_trace[4096 * 8];
#define MLRA_STAMP(k)                                                                                   \
  do {                                                                                                  \
    if (threadIdx.x == 0) {                                                                             \
      unsigned long long t_;                                                                            \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)::"memory");                                  \
      g_small_trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 8 + (k)] = t_;   \
    }                                                                                                   \
  } while (0)
#else
#define MLRA_STAMP(k) \
  do {                \
  } while (0)
#endif

// ----------------------------------------------------------------------------- K0
// attnkit/decode.py:129-150 (append_owned) + cache.py:44-57: write one token row per
// sequence into its page. rows [B, W] bf16; positions [B] = slot index of the new token.
// advance != 0: positions[s] += 1 once the slot is read (the reference append grows the
// cache length, cache.py:44-57), saving the separate length-update launch.
__global__ void cache_append_kernel(const __nv_bfloat16* __restrict__ rows, const int32_t* __restrict__ block_table,
                                    int32_t* __restrict__ positions, int W, int page_size, int max_pages, int advance,
                                    __nv_bfloat16* __restrict__ pool) {
  const int s = blockIdx.x;
  const int pos = positions[s];
  if (advance) {
    __syncthreads();
    if (threadIdx.x == 0) positions[s] = pos + 1;
  }
  const int page = block_table[size_t(s) * max_pages + pos / page_size];
  __nv_bfloat16* dst = pool + (size_t(page) * page_size + pos % page_size) * W;
  const __nv_bfloat16* src = rows + size_t(s) * W;
  for (int i = threadIdx.x; i < W / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
}

// ----------------------------------------------------------------------------- K0 (fused write side)
// attnkit/latent.py:129-159 (the cache half of latent_projections) + decode.py:129-150
// (append_owned): from the token's raw down-projections
//   c_kv = alpha_kv * rmsnorm(h W^DKV)            (latent.py:149, tensors.py:83-87, eps 1e-6)
//   k_rope = rope(h W^KR, pos)                     (latent.py:140, rope.py:37-60: pairs (2l, 2l+1),
//                                                   theta_l = base^(-2l/dr))
// write the device's owned latent blocks (each zero-padded to dlp) and the rotary key (padded
// to drp) as one bf16 pool row at the sequence's next slot. One CTA per sequence. The RMS needs
// the whole c_kv row even when the device owns one block (TP4), so kv_raw is the full row.
// Angles are formed in fp64 and reduced mod 2*pi before the fp32 sincos: at 128K positions an
// fp32 angle would be off by ~1e-2 rad.
constexpr int kK0Threads = 128;
__global__ void __launch_bounds__(kK0Threads)
cache_append_latent_kernel(const float* __restrict__ kv_raw, const float* __restrict__ kr_raw,
                           const int32_t* __restrict__ rope_pos, int32_t* __restrict__ slots,
                           const int32_t* __restrict__ block_table, int d_c, int bs, int block0, int nblocks, int dlp,
                           int dr, int drp, float alpha_kv, float rope_base, float eps, int page_size, int max_pages,
                           int norm_groups, int advance, __nv_bfloat16* __restrict__ pool) {
  // RMS per latent group: the row is norm_groups consecutive groups of d_c/norm_groups
  // columns (1 for MLA / MLRA-4; one per group for GLA / MLRA-2, latent.py:145-158)
  constexpr int kMaxGroups = 4;
  __shared__ float red[kMaxGroups][kK0Threads / 32];
  __shared__ float gscale[kMaxGroups];
  const int s = blockIdx.x, tid = threadIdx.x;
  // advance bit 1: a programmatic dependent that releases its own dependent at once (the next
  // kernel waits for this one's completion before it reads the pool: decode_layer's K-1 query)
  if (advance & 2) griddep_launch_dependents();
  griddep_wait();  // kv_raw / kr_raw come from the previous kernel
  // slots == NULL: ONE sequence's n rows (prefill): row s -> slot s of block_table row 0
  const int slot = slots != nullptr ? slots[s] : s;  // read before the barriers below; advanced after them
  const float* kv = kv_raw + size_t(s) * d_c;
  const int gw = d_c / norm_groups;
  for (int g = 0; g < norm_groups; ++g) {
    float ss = 0.f;
    for (int c = tid; c < gw; c += kK0Threads) ss = fmaf(kv[g * gw + c], kv[g * gw + c], ss);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if ((tid & 31) == 0) red[g][tid >> 5] = ss;
  }
  __syncthreads();
  if (tid < norm_groups) {
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kK0Threads / 32; ++w) tot += red[tid][w];
    gscale[tid] = alpha_kv * rsqrtf(tot / float(gw) + eps);
  }
  __syncthreads();
  if ((advance & 1) && slots != nullptr && tid == 0) slots[s] = slot + 1;
  const int page = block_table[size_t(slots != nullptr ? s : 0) * max_pages + slot / page_size];
  const int W = nblocks * dlp + drp;
  __nv_bfloat16* dst = pool + (size_t(page) * page_size + slot % page_size) * W;
  for (int i = tid; i < nblocks * dlp; i += kK0Threads) {
    const int u = i / dlp, c = i % dlp;
    const int col = (block0 + u) * bs + c;
    const float v = c < bs ? kv[col] * gscale[col / gw] : 0.f;
    dst[i] = __float2bfloat16(v);
  }
  const double pos = double(rope_pos != nullptr ? rope_pos[s] : slot);  // NULL: the slot written
  const float* kr = kr_raw + size_t(s) * dr;
  for (int l = tid; l < drp / 2; l += kK0Threads) {
    float e = 0.f, o = 0.f;
    if (2 * l + 1 < dr) {
      const double theta = pow(double(rope_base), -2.0 * l / dr);
      const double a = pos * theta, two_pi = 6.283185307179586476925286766559;
      float sn, cs;
      sincosf(float(a - two_pi * floor(a * (1.0 / two_pi))), &sn, &cs);  // reduced mod 2 pi in fp64
      const float x0 = kr[2 * l], x1 = kr[2 * l + 1];
      e = x0 * cs - x1 * sn;
      o = x0 * sn + x1 * cs;
    }
    reinterpret_cast<__nv_bfloat162*>(dst + nblocks * dlp)[l] = __floats2bfloat162_rn(e, o);
  }
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
  griddep_wait();  // X is the previous kernel's output (PDL launch: the weights above overlap it)
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

// ----------------------------------------------------------------------------- K2 plan
// Ragged-batch split scheduler (mlra_decode_plan): a deterministic work table for K2 that
// balances the token tiles of B sequences of any lengths over `ctas` CTAs (one wave per head
// group). The smallest per-CTA tile budget c >= ceil(total / ctas) is searched such that the
// per-sequence split counts ns_s = max(1, ceil(tiles_s / c)) (<= nsplit_max) fit the CTAs;
// sequence s gets ns_s consecutive splits of ceil(tiles_s / ns_s) tiles (items in ascending
// (sequence, split) order: the merge adds the splits in that order). seq_splits[s] = ns_s: the
// merge reads only those slots. One CTA.
constexpr int kPlanThreads = 32;  // one warp: warp reductions only (the plan sits on the step's critical path)
__global__ void __launch_bounds__(kPlanThreads)
decode_plan_kernel(const int32_t* __restrict__ seqlens, int B, int T, int ctas, int nsplit_max,
                   int32_t* __restrict__ plan, int32_t* __restrict__ seq_splits) {
  extern __shared__ int pl_smem[];
  int* tiles = pl_smem;  // [B]
  int* offs = pl_smem + B;  // [B]
  const int lane = threadIdx.x;
  auto wsum = [](int v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  auto wmax = [](int v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  };
  int loc = 0, mx = 0;
  for (int s = lane; s < B; s += 32) {
    const int t = (max(seqlens[s], 0) + T - 1) / T;
    tiles[s] = t;
    loc += t;
    mx = max(mx, t);
  }
  const int total = wsum(loc);
  mx = wmax(mx);
  __syncwarp();
  // binary search of the tile budget c: feasible(c) <=> sum_s max(1, ceil(tiles_s / c)) <= ctas and
  // every ceil(tiles_s / c) <= nsplit_max (monotone in c)
  int lo = max(1, (total + ctas - 1) / ctas), hi = max(lo, mx);
  while (lo < hi) {
    const int c = (lo + hi) / 2;
    int cnt = 0, bad = 0;
    for (int s = lane; s < B; s += 32) {
      const int k = max(1, (tiles[s] + c - 1) / c);
      cnt += k;
      bad |= k > nsplit_max;
    }
    cnt = wsum(cnt);
    bad = wsum(bad);
    if (cnt <= ctas && bad == 0) hi = c; else lo = c + 1;
  }
  const int c = lo;
  // item offsets: exclusive prefix sum of the split counts (lane-chunked scan)
  int run = 0;
  for (int s0 = 0; s0 < B; s0 += 32) {
    const int s = s0 + lane;
    const int k = s < B ? min(nsplit_max, max(1, (tiles[s] + c - 1) / c)) : 0;
    int incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (s < B) {
      offs[s] = run + incl - k;
      seq_splits[s] = k;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  __syncwarp();
  for (int s = lane; s < B; s += 32) {
    const int t = tiles[s], k = seq_splits[s], off = offs[s];
    const int per = (t + k - 1) / max(k, 1);
    for (int j = 0; j < k; ++j)
      reinterpret_cast<int4*>(plan)[off + j] = make_int4(s, j, j * per, max(0, min(per, t - j * per)));
  }
  for (int i = run + lane; i < ctas; i += 32) reinterpret_cast<int4*>(plan)[i] = make_int4(-1, 0, 0, 0);
}

// ----------------------------------------------------------------------------- K3a
// Flash-decoding merge of the K2 split partials: for every (sequence, branch, head) row,
//   Z = sum_k w_k O_k with w_k = 2^(lse_k - max) / sum_j 2^(lse_j - max).
// CTA = (row, CW latent columns), CW x Q threads: warp 0 forms the split weights once (lane k <
// nsplit, shuffled max / sum) into smem; thread (q, c) merges column c over the splits k = q,
// q+Q, ... and the Q partial sums are added in ascending q through smem (deterministic).
// Q = 4 with 128 columns (8 loads in flight per round); Q = 16 with 32 columns when the rows are
// few and the splits many (batch-1 decode runs up to 148): a thread's <= 10 split values are all
// loaded at once, issued before the weights are known, so the merge costs one round trip.
// Output [B, H, NB*DLAT] (the K3b input) or, with zout_bnh, [B, NB, H, DLAT] * alpha (the latent
// mixture itself: the paper's decode scope).
constexpr int kMergeMaxSplits = 160;  // 5 per lane
constexpr int kMergeQ = 4;            // split groups with 128 columns per CTA
constexpr int kMergeQWide = 16;       // split groups with 32 columns per CTA
template <int Q>
__global__ void __launch_bounds__(512)
merge_splits_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part, float* __restrict__ z, int B,
                    int NB, int H, int DLAT, int nsplit, float alpha, int zout_bnh, int* __restrict__ status,
                    const int32_t* __restrict__ seq_splits) {
  __shared__ float wsh[kMergeMaxSplits];
  __shared__ float part[512];  // [Q][CW]
  const int CW = blockDim.x / Q;
  const int row = blockIdx.x, cl = threadIdx.x % CW, qk = threadIdx.x / CW, c = blockIdx.y * CW + cl;
  const int lane = threadIdx.x % 32;
  const int h = row % H, b = (row / H) % NB, s = row / (H * NB);
  const int ns = seq_splits != nullptr ? min(seq_splits[s], nsplit) : nsplit;  // splits of this sequence
  const float* o = o_part + ((size_t(s) * nsplit * NB + b) * H + h) * DLAT + c;  // split stride NB*H*DLAT
  const size_t sstride = size_t(NB) * H * DLAT;
  griddep_launch_dependents();  // the up-projection (K3b) may stage its weights meanwhile
  griddep_wait();
  constexpr int kPre = Q == kMergeQWide ? (kMergeMaxSplits + Q - 1) / Q : 1;
  float pre[kPre];
  if (Q == kMergeQWide) {  // every split value of this thread in flight before the weights
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const int k = qk + j * Q;
      pre[j] = (c < DLAT && k < ns) ? __ldcg(o + size_t(k) * sstride) : 0.f;
    }
  }
  if (threadIdx.x < 32) {
    const float* l = lse_part + (size_t(s) * nsplit * NB + b) * H + h;  // split stride NB*H
    float lk[kMergeMaxSplits / 32];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMergeMaxSplits / 32; ++j) {
      const int k = lane + 32 * j;
      lk[j] = k < ns ? __ldcg(l + size_t(k) * NB * H) : -INFINITY;
      m = fmaxf(m, lk[j]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    {  // numeric status (attnkit/tensors.py:74-78): a NaN logit, or no finite logit in the row
      bool nan = false;
#pragma unroll
      for (int j = 0; j < kMergeMaxSplits / 32; ++j) nan |= lk[j] != lk[j];
      const bool any_nan = __any_sync(0xffffffffu, nan);
      if (status != nullptr && lane == 0 && blockIdx.y == 0 && (any_nan || m == -INFINITY))
        atomicOr(status, (any_nan ? kStatusNaN : 0) | (m == -INFINITY ? kStatusNoFinite : 0));
    }
    float tot = 0.f;
#pragma unroll
    for (int j = 0; j < kMergeMaxSplits / 32; ++j) {
      lk[j] = (m == -INFINITY || lk[j] == -INFINITY) ? 0.f : exp2f(lk[j] - m);
      tot += lk[j];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
    const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
    for (int j = 0; j < kMergeMaxSplits / 32; ++j)
      if (lane + 32 * j < ns) wsh[lane + 32 * j] = lk[j] * inv;
  }
  __syncthreads();
  float acc = 0.f;
  if (Q == kMergeQWide) {
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const int k = qk + j * Q;
      if (k < ns) acc = fmaf(wsh[k], pre[j], acc);
    }
  } else if (c < DLAT) {
    for (int k0 = qk; k0 < ns; k0 += 8 * Q) {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j * Q;
        v[j] = k < ns ? __ldcg(o + size_t(k) * sstride) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0 + j * Q;
        if (k < ns) acc = fmaf(wsh[k], v[j], acc);
      }
    }
  }
  part[qk * CW + cl] = acc;
  __syncthreads();
  if (qk != 0 || c >= DLAT) return;
  float t = part[cl];
#pragma unroll
  for (int q = 1; q < Q; ++q) t += part[q * CW + cl];
  float* dst = zout_bnh ? z + ((size_t(s) * NB + b) * H + h) * DLAT : z + (size_t(s) * H + h) * (NB * DLAT) + b * DLAT;
  dst[c] = t * (zout_bnh ? alpha : 1.f);
}


// ----------------------------------------------------------------------------- K1 / K3 (v2)
// Both small GEMMs of the step are "4 sequences x 128 output columns per CTA" kernels with
// the weight tile staged in smem. 512 threads = 128 columns x 4 quarters of the
// contraction: a thread's loop reads a conflict-free bf16 of the weight row and a
// broadcast float4 of the 4 sequences (4 FMAs per 2 shared loads), 16 warps per SM hide
// the shared-load latency, and the 4 quarters are added through smem at the end.
// Spreading a head's columns x sequence groups (x branches) over 100s of CTAs keeps every
// SM's share of the weights at 32 KB: the kernels cost about one round trip to L2/HBM.
constexpr int kG4Seqs = 4, kG4Threads = 512, kG4Cols = 128, kG4KChunk = 128, kG4Q = kG4Threads / kG4Cols;

// K1: q_abs[s, b, h, c] = scale * sum_p q_nope[s, h, p] * W^UK[h][p][b*DLAT + c]
// (attnkit/decode.py:155-167, per branch at :224). Grid (ceil(NCOL/128), H, ceil(B/4)).
// The W^UK tile does not depend on the previous kernel: its loads are issued before
// griddepcontrol.wait. CTAs of column block 0 also write q_rope * scale.
inline size_t absorb4_smem() {
  return size_t(kG4KChunk) * kG4Cols * 2 + size_t(kG4KChunk) * kG4Seqs * 4 + size_t(kG4Q) * kG4Seqs * kG4Cols * 4;
}

__global__ void __launch_bounds__(kG4Threads)
absorb4_kernel(const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ w_uk,
               __nv_bfloat16* __restrict__ q_abs, int B, int H, int DH, int NB, int DLAT, float scale,
               const __nv_bfloat16* __restrict__ rope_in, __nv_bfloat16* __restrict__ rope_out, int DR) {
  griddep_launch_dependents();
  extern __shared__ __align__(16) uint8_t g4_smem[];
  __nv_bfloat16* ws = reinterpret_cast<__nv_bfloat16*>(g4_smem);                      // [KC][128]
  float4* xs = reinterpret_cast<float4*>(g4_smem + size_t(kG4KChunk) * kG4Cols * 2);  // [KC] x 4 seqs
  float* red = reinterpret_cast<float*>(xs + kG4KChunk);                              // [Q][4][128]
  const int NCOL = NB * DLAT;
  const int c0 = blockIdx.x * kG4Cols, h = blockIdx.y, s0 = blockIdx.z * kG4Seqs, tid = threadIdx.x;
  const int ncols = min(kG4Cols, NCOL - c0);
  const int oct = ncols / 8;  // 16-byte chunks per weight row (NCOL % 8 == 0, host-checked)
  const int col = tid % kG4Cols, kq = tid / kG4Cols;
  MLRA_STAMP(0);
  float acc[kG4Seqs] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < DH; k0 += kG4KChunk) {
    const int kc = min(kG4KChunk, DH - k0);
    if (k0 > 0) __syncthreads();
    {
      // weight tile: kc rows x ncols in 16-byte chunks, and this thread's query element;
      // every load is in flight before the first store
      constexpr int kPer = kG4KChunk * kG4Cols / 8 / kG4Threads;  // 4
      uint4 v[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int i = tid + j * kG4Threads;
        const int r = i / (kG4Cols / 8), c8 = i % (kG4Cols / 8);
        v[j] = (r < kc && c8 < oct) ? __ldg(reinterpret_cast<const uint4*>(w_uk + (size_t(h) * DH + k0 + r) * NCOL + c0) + c8)
                                   : make_uint4(0, 0, 0, 0);
      }
      if (k0 == 0) griddep_wait();  // q_nope comes from the previous kernel on the stream
      // x: thread (row r = tid / 4, sequence tid % 4)
      const int xr = tid / kG4Seqs, xsq = tid % kG4Seqs;
      float xv = 0.f;
      if (xr < kc && s0 + xsq < B) xv = __bfloat162float(q_nope[(size_t(s0 + xsq) * H + h) * DH + k0 + xr]);
#pragma unroll
      for (int j = 0; j < kPer; ++j) reinterpret_cast<uint4*>(ws)[tid + j * kG4Threads] = v[j];
      if (xr < kG4KChunk) reinterpret_cast<float*>(xs)[tid] = xv;
    }
    __syncthreads();
    MLRA_STAMP(1);
    const int q_len = (kc + kG4Q - 1) / kG4Q, r0 = kq * q_len, r1 = min(kc, r0 + q_len);
    const __nv_bfloat16* wc = ws + col;
#pragma unroll 8
    for (int r = r0; r < r1; ++r) {
      const float w = __bfloat162float(wc[r * kG4Cols]);
      const float4 x = xs[r];
      acc[0] = fmaf(x.x, w, acc[0]);
      acc[1] = fmaf(x.y, w, acc[1]);
      acc[2] = fmaf(x.z, w, acc[2]);
      acc[3] = fmaf(x.w, w, acc[3]);
    }
  }
  MLRA_STAMP(2);
  if (kq > 0) {
#pragma unroll
    for (int s = 0; s < kG4Seqs; ++s) red[((kq - 1) * kG4Seqs + s) * kG4Cols + col] = acc[s];
  }
  __syncthreads();
  if (kq == 0 && col < ncols) {
    const int cc = c0 + col, b = cc / DLAT, c = cc % DLAT;
#pragma unroll
    for (int s = 0; s < kG4Seqs; ++s) {
      float v = acc[s];
#pragma unroll
      for (int q = 1; q < kG4Q; ++q) v += red[((q - 1) * kG4Seqs + s) * kG4Cols + col];
      if (s0 + s < B) q_abs[((size_t(s0 + s) * NB + b) * H + h) * DLAT + c] = __float2bfloat16(v * scale);
    }
  }
  if (blockIdx.x == 0 && rope_out != nullptr) {
    for (int i = tid; i < kG4Seqs * DR; i += kG4Threads) {
      const int s = s0 + i / DR;
      if (s < B) {
        const size_t off = (size_t(s) * H + h) * DR + i % DR;
        rope_out[off] = __float2bfloat16(__bfloat162float(rope_in[off]) * scale);
      }
    }
  }
  MLRA_STAMP(3);
}

// K1 on tensor cores (d_h % 16 == 0, d_h <= 256): CTA = (128 output columns, head, 16
// sequences); the W^UK tile [d_h][128] (cp.async, row-XOR swizzled, issued before
// griddepcontrol.wait) and the bf16 queries [16][d_h] (exact operands) meet in mma.sync
// m16n8k16 with fp32 accumulation; warp w owns columns [16w, 16w+16). Grid (ceil(NCOL/128),
// H, ceil(B/16)): W^UK is read once per 16 sequences.
constexpr int kAmThreads = 256, kAmMaxDH = 256;
inline size_t absorb_mma_smem(int DH) { return size_t(DH) * 256 + size_t(16) * (DH + 8) * 2; }

__global__ void __launch_bounds__(kAmThreads)
absorb_mma_kernel(const __nv_bfloat16* __restrict__ q_nope, const __nv_bfloat16* __restrict__ w_uk,
                  __nv_bfloat16* __restrict__ q_abs, int B, int H, int DH, int NB, int DLAT, float scale,
                  const __nv_bfloat16* __restrict__ rope_in, __nv_bfloat16* __restrict__ rope_out, int DR) {
  griddep_launch_dependents();
  extern __shared__ __align__(128) uint8_t am_smem[];
  const int NCOL = NB * DLAT, arow = (DH + 8) * 2;
  const int c0 = blockIdx.x * 128, h = blockIdx.y, m0 = blockIdx.z * 16, tid = threadIdx.x;
  const uint32_t wbase = smem_u32(am_smem), abase = wbase + uint32_t(DH) * 256;
  for (int i = tid; i < DH * 16; i += kAmThreads) {  // W^UK[h][k][c0 + 8q ..] -> row k, unit q ^ (k & 7)
    const int r = i >> 4, q = i & 15;
    const bool ok = c0 + q * 8 < NCOL;
    cp_async16(wbase + r * 256 + ((q ^ (r & 7)) * 16),
               ok ? static_cast<const void*>(w_uk + (size_t(h) * DH + r) * NCOL + c0 + q * 8) : static_cast<const void*>(w_uk),
               ok ? 16u : 0u);
  }
  griddep_wait();  // q_nope comes from the previous kernel on the stream
  const int units = DH / 8;
  for (int i = tid; i < 16 * units; i += kAmThreads) {
    const int r = i / units, q = i % units, m = m0 + r;
    const bool ok = m < B;
    cp_async16(abase + r * arow + q * 16,
               ok ? static_cast<const void*>(q_nope + (size_t(m) * H + h) * DH + q * 8) : static_cast<const void*>(q_nope),
               ok ? 16u : 0u);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  cp_async_wait_all();
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3, q = lane >> 3;
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  for (int kb = 0; kb < DH; kb += 16) {
    uint32_t a[4], bfr[4];
    ldmatrix_x4(a, abase + ((lane & 7) + (q & 1) * 8) * arow + (kb + (q >> 1) * 8) * 2);
    const int k = kb + (q & 1) * 8 + (lane & 7);
    ldmatrix_x4_trans(bfr, wbase + k * 256 + (((warp * 2 + (q >> 1)) ^ (k & 7)) * 16));
    mma_m16n8k16_bf16(acc[0], a, bfr[0], bfr[1]);
    mma_m16n8k16_bf16(acc[1], a, bfr[2], bfr[3]);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int col = c0 + warp * 16 + j * 8 + 2 * t4;
    if (col >= NCOL) continue;
    const int bb = col / DLAT, cc = col % DLAT;  // DLAT even: the pair stays in one branch
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const int m = m0 + g + 8 * hf;
      if (m < B)
        *reinterpret_cast<uint32_t*>(q_abs + ((size_t(m) * NB + bb) * H + h) * DLAT + cc) =
            pack_bf16(acc[j][2 * hf] * scale, acc[j][2 * hf + 1] * scale);
    }
  }
  if (blockIdx.x == 0 && rope_out != nullptr) {
    for (int i = tid; i < 16 * DR; i += kAmThreads) {
      const int m = m0 + i / DR;
      if (m < B) {
        const size_t off = (size_t(m) * H + h) * DR + i % DR;
        rope_out[off] = __float2bfloat16(__bfloat162float(rope_in[off]) * scale);
      }
    }
  }
}

// K3: split merge + W^UV up-projection + ascending branch sum + alpha
// (attnkit/decode.py:228 per branch, then reduce_contributions :264-285).
// Grid (ceil(B/SEQS), H, NB), SEQS (4) sequences per CTA; with NB > 1 and a summed output the NB CTAs of a (sequence group, head)
// form a cluster: each up-projects its branch, rank 0 adds the NB results through
// distributed shared memory in ascending branch order (deterministic, the reference's
// order) and writes the head. Per CTA:
//   W^UV_b[h]  [DLAT][DH] bf16 bulk-copied into smem before griddepcontrol.wait (PDL);
//   w_k  = 2^(lse_k - max) / sum_j 2^(lse_j - max)  per (sequence, split);
//   Z[c] = sum_k w_k O_k[c], thread = (latent c, sequence), all split loads in flight;
//   y[d] = alpha * sum_c Z[c] W[c][d], thread = (column d, quarter of c), quarters added in smem.
template <int SEQS, int THREADS = 256>
inline size_t combine4_smem(int DLAT, int DH, int nsplit) {
  return ((size_t(DLAT) * DH * 2 + 15) / 16) * 16 + size_t(DLAT) * SEQS * 4 + size_t(THREADS / kG4Cols) * SEQS * DH * 4 +
         16 + size_t(SEQS) * kMergeMaxSplits * 4;
}

// Non-volatile DSMEM load: independent loads after a cluster barrier may be issued together.
__device__ __forceinline__ float ld_shared_cluster_f32_batched(uint32_t addr) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

constexpr int kMergeChunk = 12;  // split loads in flight per thread (B = 16 -> 9 splits: one pass)

// 256 threads = 128 columns x 2 halves of the contraction: small enough that every CTA of
// the TP1 grid (384) is resident at once (4 per SM).
template <int SEQS, int THREADS = 256>
__global__ void __launch_bounds__(THREADS, 512 / THREADS * 2)
combine4_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part,
                const __nv_bfloat16* __restrict__ w_uv, float* __restrict__ out, int B, int H, int NB, int DLAT, int DH,
                int nsplit, float alpha, int per_branch, const TpSum tp, int* __restrict__ status,
                const int32_t* __restrict__ seq_splits) {
  static_assert(SEQS == 2 || SEQS == 4 || SEQS == 8, "2, 4 or 8 sequences per CTA");
  constexpr int kQ = THREADS / kG4Cols;  // parts of the contraction per output column
  extern __shared__ __align__(128) uint8_t c4_smem[];
  const size_t wbytes = size_t(DLAT) * DH * 2;
  const __nv_bfloat16* wsm = reinterpret_cast<const __nv_bfloat16*>(c4_smem);  // [DLAT][DH]
  float* zs = reinterpret_cast<float*>(c4_smem + ((wbytes + 15) / 16) * 16);    // [DLAT][SEQS]
  float* ys = zs + DLAT * SEQS;                                                 // [Q][SEQS][DH]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ys + kQ * SEQS * DH);
  float* wts = reinterpret_cast<float*>(bar + 2);                                // [SEQS][kMergeMaxSplits]
  const int s0 = blockIdx.x * SEQS, h = blockIdx.y, b = blockIdx.z, tid = threadIdx.x;
  MLRA_STAMP(0);
  // fused TP sum (tp.world > 1, summed output): this call's epoch from the rank's region
  uint32_t& s_tp_epoch = *reinterpret_cast<uint32_t*>(bar + 1);  // (dynamic smem: no static carve-out)
  const size_t tp_n = size_t(B) * H * DH, tp_ns = ar_stride(int(tp_n));
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    if (tp.world > 1)
      s_tp_epoch = *reinterpret_cast<volatile uint32_t*>(
                       reinterpret_cast<uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), tp.world)) +
                       ar_flag_words(tp.world)) + 1u;
  }
  __syncthreads();
  // DH = 128 and >= 4 sequences: the up-projection runs on mma.sync and W^UV_b[h] is staged with
  // cp.async, its 16-byte units XOR-swizzled by row (conflict-free ldmatrix.trans); otherwise
  // (2 sequences would fill 2 of the MMA's 16 rows) FMAs on one bulk copy of W^UV_b[h].
  const bool use_mma = DH == 128 && DLAT % 16 == 0 && SEQS > 2;
  const uint8_t* w_src = reinterpret_cast<const uint8_t*>(w_uv + (size_t(h) * NB + b) * DLAT * DH);
  if (use_mma) {
    const uint32_t wbase = smem_u32(c4_smem);
    for (int i = tid; i < DLAT * 16; i += THREADS) {
      const int r = i >> 4, q = i & 15;
      cp_async16(wbase + r * 256 + ((q ^ (r & 7)) * 16), w_src + size_t(r) * 256 + q * 16, 16u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else if (tid == 0) {
    mbar_arrive_expect_tx(bar, uint32_t(wbytes));
    for (size_t off = 0; off < wbytes; off += 32768)
      bulk_copy_g2s(c4_smem + off, w_src + off, uint32_t(wbytes - off < 32768 ? wbytes - off : 32768), bar);
  }
  griddep_wait();  // partials of K2 (a no-op in plain stream order)
  MLRA_STAMP(1);
  const size_t kstride = size_t(NB) * H * DLAT;  // split stride of o_part
  // merge: thread = (latent column c, sequence), two items at a time with every split load of
  // both in flight: Z[c] = sum_k w_k O_k[c]. The first pair's partial loads are issued before
  // the split weights are formed, so the two L2 round trips overlap.
  auto load_pair = [&](int i0, int k0, float (&v)[2][kMergeChunk]) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = i0 + u * THREADS, c = i / SEQS, sq = i % SEQS, s = s0 + sq;
      const bool ok = i < DLAT * SEQS && s < B;
      const float* o = o_part + ((size_t(s) * nsplit * NB + b) * H + h) * DLAT + c;
      const int ns = (ok && seq_splits != nullptr) ? min(seq_splits[s], nsplit) : nsplit;
#pragma unroll
      for (int j = 0; j < kMergeChunk; ++j) v[u][j] = (ok && k0 + j < ns) ? __ldcg(o + size_t(k0 + j) * kstride) : 0.f;
    }
  };
  float v[2][kMergeChunk];
  load_pair(tid, 0, v);
  // split weights w_k = 2^(lse_k - max) / sum_j 2^(lse_j - max), once per sequence: warp sq,
  // lane k (+32j) -> wts[sq][k] (0 for empty splits / an empty sequence)
  {
    const int sq = tid / 32, lane = tid % 32, s = s0 + sq;
    if (sq < SEQS) {
      const int ns = (s < B && seq_splits != nullptr) ? min(seq_splits[s], nsplit) : nsplit;
      float lk[kMergeMaxSplits / 32];
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < kMergeMaxSplits / 32; ++j) {
        const int k = lane + 32 * j;
        lk[j] = (s < B && k < ns) ? __ldcg(lse_part + (size_t(s) * nsplit * NB + b) * H + h + size_t(k) * NB * H)
                                      : -INFINITY;
        m = fmaxf(m, lk[j]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      {  // numeric status (attnkit/tensors.py:74-78)
        bool nan = false;
#pragma unroll
        for (int j = 0; j < kMergeMaxSplits / 32; ++j) nan |= lk[j] != lk[j];
        const bool any_nan = __any_sync(0xffffffffu, nan);
        if (status != nullptr && lane == 0 && s < B && (any_nan || m == -INFINITY))
          atomicOr(status, (any_nan ? kStatusNaN : 0) | (m == -INFINITY ? kStatusNoFinite : 0));
      }
      float tot = 0.f;
#pragma unroll
      for (int j = 0; j < kMergeMaxSplits / 32; ++j) {
        lk[j] = (m == -INFINITY || lk[j] == -INFINITY) ? 0.f : ex2(lk[j] - m);
        tot += lk[j];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
      const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
      for (int j = 0; j < kMergeMaxSplits / 32; ++j)
        if (lane + 32 * j < nsplit) wts[sq * kMergeMaxSplits + lane + 32 * j] = lk[j] * inv;
    }
  }
  __syncthreads();
  int ns_cta = nsplit;
  if (seq_splits != nullptr) {
    ns_cta = 0;
    for (int sq = 0; sq < SEQS && s0 + sq < B; ++sq) ns_cta = max(ns_cta, min(seq_splits[s0 + sq], nsplit));
  }
  for (int i0 = tid; i0 < DLAT * SEQS; i0 += 2 * THREADS) {
    float z[2] = {0.f, 0.f};
    for (int k0 = 0; k0 < ns_cta; k0 += kMergeChunk) {
      if (i0 != tid || k0 != 0) load_pair(i0, k0, v);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int sq = (i0 + u * THREADS) % SEQS;
#pragma unroll
        for (int j = 0; j < kMergeChunk; ++j)
          if (k0 + j < nsplit) z[u] = fmaf(wts[sq * kMergeMaxSplits + k0 + j], v[u][j], z[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (i0 + u * THREADS < DLAT * SEQS) zs[i0 + u * THREADS] = z[u];
  }
  if (use_mma) cp_async_wait_all();
  __syncthreads();
  MLRA_STAMP(2);
  if (!use_mma) mbar_wait(bar, 0);
  MLRA_STAMP(3);
  const bool cluster_sum = NB > 1 && !per_branch;
  if (use_mma) {
    // y[s][d] = alpha * sum_c Z[s][c] W[c][d]: rows = the SEQS sequences (of 16), warp w owns
    // columns [16w, 16w+16); Z enters as bf16 hi + lo (two MMAs: ~16-bit mantissa), fp32 sums
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3, q = lane >> 3;
    const uint32_t wbase = smem_u32(c4_smem);
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int kb = 0; kb < DLAT; kb += 16) {
      uint32_t ahi[4] = {0u, 0u, 0u, 0u}, alo[4] = {0u, 0u, 0u, 0u};
      if (g < SEQS) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int k = kb + 2 * t4 + 8 * hf;
          const float z0 = zs[k * SEQS + g], z1 = zs[(k + 1) * SEQS + g];
          const __nv_bfloat16 h0 = __float2bfloat16_rn(z0), h1 = __float2bfloat16_rn(z1);
          ahi[2 * hf] = pack_bf16_raw(h0, h1);
          alo[2 * hf] = pack_bf16(z0 - __bfloat162float(h0), z1 - __bfloat162float(h1));
        }
      }
      uint32_t bfr[4];
      const int k = kb + (q & 1) * 8 + (lane & 7);
      ldmatrix_x4_trans(bfr, wbase + k * 256 + (((warp * 2 + (q >> 1)) ^ (k & 7)) * 16));
      mma_m16n8k16_bf16(acc[0], ahi, bfr[0], bfr[1]);
      mma_m16n8k16_bf16(acc[0], alo, bfr[0], bfr[1]);
      mma_m16n8k16_bf16(acc[1], ahi, bfr[2], bfr[3]);
      mma_m16n8k16_bf16(acc[1], alo, bfr[2], bfr[3]);
    }
    if (g < SEQS) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int col = warp * 16 + j * 8 + 2 * t4;
        ys[g * DH + col] = acc[j][0] * alpha;
        ys[g * DH + col + 1] = acc[j][1] * alpha;
      }
    }
  } else {
    const int cq = tid / kG4Cols;
    const int q_len = (DLAT + kQ - 1) / kQ, cr0 = cq * q_len, cr1 = min(DLAT, cr0 + q_len);
    for (int d0 = 0; d0 < DH; d0 += kG4Cols) {
      const int d = d0 + tid % kG4Cols;
      float acc[SEQS];
#pragma unroll
      for (int s = 0; s < SEQS; ++s) acc[s] = 0.f;
      if (d < DH) {
        const __nv_bfloat16* wc = wsm + d;
#pragma unroll 4
        for (int c = cr0; c < cr1; ++c) {
          const float w = __bfloat162float(wc[size_t(c) * DH]);
#pragma unroll
          if constexpr (SEQS == 2) {
            const float2 z = *reinterpret_cast<const float2*>(zs + c * SEQS);
            acc[0] = fmaf(z.x, w, acc[0]);
            acc[1] = fmaf(z.y, w, acc[1]);
          } else {
#pragma unroll
            for (int s4 = 0; s4 < SEQS; s4 += 4) {
              const float4 z = *reinterpret_cast<const float4*>(zs + c * SEQS + s4);
              acc[s4 + 0] = fmaf(z.x, w, acc[s4 + 0]);
              acc[s4 + 1] = fmaf(z.y, w, acc[s4 + 1]);
              acc[s4 + 2] = fmaf(z.z, w, acc[s4 + 2]);
              acc[s4 + 3] = fmaf(z.w, w, acc[s4 + 3]);
            }
          }
        }
      }
      if (d0 > 0) __syncthreads();
      if (d < DH) {
#pragma unroll
        for (int s = 0; s < SEQS; ++s) ys[(cq * SEQS + s) * DH + d] = acc[s];
      }
    }
    __syncthreads();
    // quarters -> ys[0] (scaled); thread = (sequence, column)
    for (int i = tid; i < SEQS * DH; i += THREADS) {
      float v = ys[i];
#pragma unroll
      for (int q = 1; q < kQ; ++q) v += ys[q * SEQS * DH + i];
      ys[i] = v * alpha;
    }
  }  // FMA up-projection
  MLRA_STAMP(4);
  const bool tp_sum = tp.world > 1 && !per_branch;
  if (!cluster_sum) {
    __syncthreads();
    if (!tp_sum) {
      for (int i = tid; i < SEQS * DH; i += THREADS) {
        const int s = s0 + i / DH, d = i % DH;
        if (s >= B) continue;
        if (per_branch) out[((size_t(s) * NB + b) * H + h) * DH + d] = ys[i];
        else out[(size_t(s) * H + h) * DH + d] = ys[i];
      }
    }
  } else {
    // branch sum over the cluster (ranks = branches along z), ascending order
    cluster_arrive_release();
    cluster_wait_acquire();
    if (b == 0) {
      const uint32_t ys_addr = smem_u32(ys);
      for (int i = tid; i < SEQS * DH; i += THREADS) {
        const int s = s0 + i / DH, d = i % DH;
        float rv[4];
#pragma unroll
        for (int r = 1; r < 4; ++r) rv[r] = r < NB ? ld_shared_cluster_f32_batched(mapa_shared(ys_addr + i * 4, r)) : 0.f;
        float tot = ys[i];
#pragma unroll
        for (int r = 1; r < 4; ++r)
          if (r < NB) tot += rv[r];  // ascending branch order
        if (tp_sum) ys[i] = tot;  // own slot i only: the peers read their own smem, not ours
        else if (s < B) out[(size_t(s) * H + h) * DH + d] = tot;
      }
    }
    // keep every rank's smem alive until rank 0 has read it
    cluster_arrive_release();
    cluster_wait_acquire();
  }
  if (tp_sum && b == 0) {
    // one-shot sum over the TP ranks (the K5 protocol, fused): store this CTA's [SEQS][DH] tile
    // into slot [parity][my rank] of every rank, release the epoch into that rank's flag for
    // this CTA, wait for the world flags of this CTA in my region, add in ascending rank order
    const int W = tp.world, par = int(s_tp_epoch & 1u);
    const uint32_t epoch = s_tp_epoch;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x, nct = gridDim.x * gridDim.y;
    __syncthreads();
    for (int r = 0; r < W; ++r) {
      float* dst = tp.comm[r] + (size_t(par) * W + tp.rank) * tp_ns;
      for (int i = tid; i < SEQS * DH; i += THREADS) {
        const int s = s0 + i / DH;
        if (s < B) dst[(size_t(s) * H + h) * DH + i % DH] = ys[i];
      }
    }
    __syncthreads();
    if (tid < W) {
      __threadfence_system();
      uint32_t* flags = reinterpret_cast<uint32_t*>(tp.comm[tid] + ar_recv_floats(int(tp_n), W));
      ar_st_release_sys(flags + (size_t(par) * W + tp.rank) * kArFlagSlots + cta, epoch);
      const uint32_t* f = reinterpret_cast<const uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) +
                          (size_t(par) * W + tid) * kArFlagSlots + cta;
      const unsigned long long t0 = ar_globaltimer();
      while (ar_ld_acquire_sys(f) != epoch) {
        if (ar_globaltimer() - t0 > 4000000000ull) __trap();
        __nanosleep(32);
      }
    }
    __syncthreads();
    const float* recv = tp.comm[tp.rank] + size_t(par) * W * tp_ns;
    for (int i = tid; i < SEQS * DH; i += THREADS) {
      const int s = s0 + i / DH;
      if (s >= B) continue;
      const size_t o = (size_t(s) * H + h) * DH + i % DH;
      float sum = 0.f;
      for (int r = 0; r < W; ++r) sum += __ldcv(recv + size_t(r) * tp_ns + o);
      out[o] = sum;
    }
    if (tid == 0) {  // advance the rank's epoch once every CTA of the call has read it
      uint32_t* ctr = reinterpret_cast<uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) + ar_flag_words(W);
      __threadfence();
      if (atomicAdd(ctr + 1, 1u) == uint32_t(nct) - 1u) {
        ctr[1] = 0u;
        atomicExch(ctr, epoch);
      }
    }
  }
  MLRA_STAMP(5);
}

// ----------------------------------------------------------------------------- K3 (split-K, cluster)
// K3 for the summed output, with the split merge spread over a thread-block cluster:
// grid (ceil(B/4), H, KP), cluster (1, 1, KP), 256 threads. CTA (sequence group, head h, kp):
//   1. cp.async its slice of W^UV_b[h] for every branch b: rows [NB*DLAT], output columns
//      [kp*DH/KP, (kp+1)*DH/KP)  (kp owns those output columns);
//   2. merges splits [kp*nsplit/KP, (kp+1)*nsplit/KP) of all (sequence, branch, latent)
//      items into an unnormalised partial (local max m, sum l, mixture z) in its smem;
//   3. cluster barrier; reads the KP partials through DSMEM and forms the final merged
//      latent Z = sum_kp z_kp 2^(m_kp - M) / sum_kp l_kp 2^(m_kp - M) for every item;
//   4. cluster barrier (remote reads done); y[s, d] = alpha * sum_b sum_c Z[s,b,c] W_b[c, d]
//      for its columns, branches summed in ascending order inside the CTA (deterministic).
// The per-thread merge loop is nsplit/KP long instead of nsplit (small batches run up to
// 148 splits), and KP x more CTAs share the work.
constexpr int kSkThreads = 256;
template <int KP>
inline size_t combine_splitk_smem(int NB, int DLAT, int DH) {
  const size_t rows = size_t(NB) * DLAT;
  return rows * (DH / KP) * 2            // W slice
         + size_t(4) * rows * 4          // this CTA's partial z [4][NB*DLAT]
         + size_t(4) * NB * 2 * 4        // its (m, l) [4][NB]
         + rows * 16                     // merged Z [NB*DLAT][4]
         + size_t(4) * kSkThreads * 4;   // GEMV reduction [256/DSL][4][DSL]
}

template <int KP>
__global__ void __launch_bounds__(kSkThreads)
combine_splitk_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part,
                      const __nv_bfloat16* __restrict__ w_uv, float* __restrict__ out, int B, int H, int NB, int DLAT,
                      int DH, int nsplit, float alpha, int* __restrict__ status,
                      const int32_t* __restrict__ seq_splits) {
  extern __shared__ __align__(128) uint8_t sk_smem[];
  const int rows = NB * DLAT, DSL = DH / KP;
  __nv_bfloat16* wsl = reinterpret_cast<__nv_bfloat16*>(sk_smem);  // [rows][DSL]
  float* pz = reinterpret_cast<float*>(wsl + size_t(rows) * DSL);   // [4][rows]
  float* pml = pz + 4 * rows;                                       // [4][NB][2] (m, l)
  float4* zf = reinterpret_cast<float4*>(pml + 8 * NB);             // [rows] x 4 seqs
  float* red = reinterpret_cast<float*>(zf + rows);                 // [256/DSL][4][DSL]
  const int s0 = blockIdx.x * 4, h = blockIdx.y, kp = blockIdx.z, tid = threadIdx.x;
  const int d0 = kp * DSL;
  MLRA_STAMP(0);
  {
    // W^UV slice: row r = b*DLAT + c of head h, columns [d0, d0+DSL): DSL*2 bytes = 16-byte chunks
    const int cpr = DSL / 8;
    const __nv_bfloat16* src = w_uv + size_t(h) * rows * DH + d0;
    const uint32_t dst0 = smem_u32(wsl);
    for (int i = tid; i < rows * cpr; i += kSkThreads) {
      const int r = i / cpr, c = i % cpr;
      cp_async16(dst0 + uint32_t((r * DSL + c * 8) * 2), src + size_t(r) * DH + c * 8, 16u);
    }
  }
  griddep_wait();
  // ---- 2. local merge over this CTA's splits; item = (sequence q, row r = b*DLAT + c)
  const int k0 = int((long long)kp * nsplit / KP), k1_all = int((long long)(kp + 1) * nsplit / KP);
  const size_t kstride = size_t(NB) * H * DLAT;  // split stride of o_part
  for (int it = tid; it < 4 * rows; it += kSkThreads) {
    const int q = it / rows, r = it % rows, b = r / DLAT, c = r % DLAT, s = s0 + q;
    float m = -INFINITY, l = 0.f, z = 0.f;
    bool nan = false;
    if (s < B) {
      const float* lp = lse_part + (size_t(s) * nsplit * NB + b) * H + h;  // split stride NB*H
      const float* op = o_part + ((size_t(s) * nsplit * NB + b) * H + h) * DLAT + c;
      const int k1 = seq_splits != nullptr ? min(k1_all, min(seq_splits[s], nsplit)) : k1_all;
      for (int kb = k0; kb < k1; kb += kMergeChunk) {
        float lk[kMergeChunk], v[kMergeChunk];
#pragma unroll
        for (int j = 0; j < kMergeChunk; ++j) {
          const int k = min(kb + j, k1 - 1);
          lk[j] = __ldcg(lp + size_t(k) * NB * H);
          v[j] = __ldcg(op + size_t(k) * kstride);
          nan |= lk[j] != lk[j];
        }
        float mc = m;
#pragma unroll
        for (int j = 0; j < kMergeChunk; ++j) mc = (kb + j < k1) ? fmaxf(mc, lk[j]) : mc;
        if (mc != -INFINITY) {
          const float a = (m == -INFINITY) ? 0.f : ex2(m - mc);
          z *= a;
          l *= a;
#pragma unroll
          for (int j = 0; j < kMergeChunk; ++j) {
            const float w = (kb + j >= k1 || lk[j] == -INFINITY) ? 0.f : ex2(lk[j] - mc);
            l += w;
            z = fmaf(w, v[j], z);
          }
          m = mc;
        }
      }
    }
    pz[q * rows + r] = z;
    if (nan && c == 0 && status != nullptr) atomicOr(status, kStatusNaN);  // attnkit/tensors.py:74-75
    if (c == 0) {
      pml[(q * NB + b) * 2] = m;
      pml[(q * NB + b) * 2 + 1] = l;
    }
  }
  cp_async_wait_all();
  cluster_arrive_release();  // also a CTA barrier: partials and the W slice are in place
  cluster_wait_acquire();
  MLRA_STAMP(1);
  // ---- 3. combine the KP partials (DSMEM, ascending kp): merged latent for every item
  {
    const uint32_t pz_a = smem_u32(pz), pml_a = smem_u32(pml);
    for (int it = tid; it < 4 * rows; it += kSkThreads) {
      const int q = it / rows, r = it % rows, b = r / DLAT;
      if (s0 + q >= B) {  // padding sequence of the group: nothing to combine
        reinterpret_cast<float*>(zf)[r * 4 + q] = 0.f;
        continue;
      }
      float mk[KP], lk[KP], zk[KP];
#pragma unroll
      for (int j = 0; j < KP; ++j) {  // all 3*KP remote loads in flight together
        mk[j] = ld_shared_cluster_f32_batched(mapa_shared(pml_a + uint32_t(((q * NB + b) * 2) * 4), j));
        lk[j] = ld_shared_cluster_f32_batched(mapa_shared(pml_a + uint32_t(((q * NB + b) * 2 + 1) * 4), j));
        zk[j] = ld_shared_cluster_f32_batched(mapa_shared(pz_a + uint32_t((q * rows + r) * 4), j));
      }
      float M = -INFINITY;
#pragma unroll
      for (int j = 0; j < KP; ++j) M = fmaxf(M, mk[j]);
      if (M == -INFINITY && kp == 0 && r % DLAT == 0 && status != nullptr)
        atomicOr(status, kStatusNoFinite);  // no finite logit in the row (attnkit/tensors.py:76-77)
      float L = 0.f, Z = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int j = 0; j < KP; ++j) {
          const float w = mk[j] == -INFINITY ? 0.f : ex2(mk[j] - M);
          L = fmaf(lk[j], w, L);
          Z = fmaf(zk[j], w, Z);
        }
      }
      reinterpret_cast<float*>(zf)[r * 4 + q] = L > 0.f ? Z / L : 0.f;
    }
  }
  // every CTA of the cluster is done reading this CTA's partial before anyone moves on
  cluster_arrive_release();
  cluster_wait_acquire();
  MLRA_STAMP(2);
  // ---- 4. up-projection of this CTA's columns: thread = (column dd, eighth of the rows)
  {
    const int dd = tid % DSL, part = tid / DSL;  // DSL divides 256
    const int nparts = kSkThreads / DSL;
    const int rl = (rows + nparts - 1) / nparts, r0 = part * rl, r1 = min(rows, r0 + rl);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    {
#pragma unroll 4
      for (int r = r0; r < r1; ++r) {
        const float w = __bfloat162float(wsl[r * DSL + dd]);
        const float4 z = zf[r];
        acc[0] = fmaf(z.x, w, acc[0]);
        acc[1] = fmaf(z.y, w, acc[1]);
        acc[2] = fmaf(z.z, w, acc[2]);
        acc[3] = fmaf(z.w, w, acc[3]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) red[(part * 4 + q) * DSL + dd] = acc[q];
    __syncthreads();
    for (int i = tid; i < 4 * DSL; i += kSkThreads) {
      const int q = i / DSL, d = i % DSL, s = s0 + q;
      float v = 0.f;
      for (int j = 0; j < nparts; ++j) v += red[(j * 4 + q) * DSL + d];
      if (s < B) out[(size_t(s) * H + h) * DH + d0 + d] = v * alpha;
    }
  }
  MLRA_STAMP(3);
}

}  // namespace mlra
