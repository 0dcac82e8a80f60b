// K6 -- causal latent prefill attention (attnkit/latent.py:172-230
// latent_prefill, causal softmax at latent.py:164-169), tcgen05 + TMA.
//
// The absorbed form of latent_prefill per branch b and head h (Eq. 5 with the
// Step-1 / Step-3 rewrites, the reference's per-head K/V are never formed):
//   logits[q, k] = q~_(b,h)[q] . C_b[k] + q_rope_h[q] . K_rope[k]     (tau*log2e folded into q)
//   P = causal softmax over k <= q;  Z_b = P . C_b;  out_h = alpha * sum_b Z_b . W^UV_(b),(h)
// i.e. an MQA-style causal flash attention with a 192-wide (DLAT + DR) key and a DLAT-wide
// value that is the key's own latent columns (one smem tile serves as K and V).
//
// CTA = (128 consecutive queries, head h), ALL branches in ascending order, so the branch sum
// happens in TMEM in the reference's order (deterministic, no partial buffers):
//   for b: for key tiles j = 0..i (causal; the diagonal tile masked per row):
//            S = Q_b . K_j^T       (M = 128 query rows, N = 128 keys, K = DLAT + DR)
//            softmax rows (thread = query row: no cross-thread reductions), P -> smem bf16
//            O += P . V_j          (N = DLAT, V = the latent columns of K_j, MN-major)
//          Z_b = O / l -> smem as bf16 hi + lo (~16-bit mantissa)
//          OUT += Z_hi . W^UV_(b),(h) + Z_lo . W^UV_(b),(h)   (N = DH)
//   out[q, h, :] = alpha * OUT[q]
// TMEM: S double buffer (2 x 128 columns) + O (DLAT) + OUT (DH) <= 512.
// Warps: 0 = TMA producer, 1 = QK issuer, 10 = PV + up-projection issuer (elected lanes),
// 2..9 = softmax / epilogue (two warps per TMEM lane quarter; thread = (query row, half of
// the columns)). Lazy rescale: the running max moves only
// when a row's tile max exceeds it by 2^8, then O's row is rescaled in TMEM (after the PVs
// issued so far have completed).
//
// Queries: q~ head-major [H, n, NB, DLAT] (the batched absorption GEMM's output), q_rope
// [n, H, DRq]; both pre-scaled by tau*log2e.
// Grid: (ceil(n/128) * H): the longest query tiles (most key tiles) are scheduled first, the
// H heads of a query tile back to back (they stream the same key tiles: L2 reuse).
#pragma once
#include <cuda.h>
#include <cstdint>
#include <cmath>
#include <cstdio>
#include "ptx.cuh"

namespace mlra {

struct PrefillParams {
  const int32_t* block_table;  // [>= 1, max_pages]: the sequence's pages (row 0)
  float* out;                  // [n, H, DH] fp32
  int n, H, NB, DR, page_size, max_pages;
  float alpha;
  int rope_col;                // first rope column of a pool row (NB * DLAT)
  volatile int* progress;      // dev: per-CTA [16] progress words (one per warp) in mapped host memory, or null
  float* dbg_s;                // dev: raw S rows of CTA dbg_cta's first key tile [128][128], or null
  int dbg_cta;
};

#define PF_PROG(slot, v)                                                                  \
  do {                                                                                   \
    if (p.progress != nullptr && (threadIdx.x & 31) == 0) p.progress[blockIdx.x * 16 + (slot)] = (v); \
  } while (0)

constexpr int kPfThreads = 352;  // TMA warp, QK warp, 8 softmax warps (2 per TMEM lane quarter), PV warp
constexpr int kPfPvWarp = 10;
constexpr int kPfT = 128;        // query rows and key tokens per tile
constexpr int kPfChunk = kPfT * 128;  // [128 rows][64 bf16] SW128 chunk (16 KB)

template <int DLAT, int DH>
struct PrefillLayout {
  static constexpr int kLatChunks = DLAT / 64, kDhChunks = DH / 64;
  // smem: Q [lat chunks | rope chunk], KV ring 2 x ([lat chunks] + rope chunk), P 2 x (2 chunks).
  // At a branch's end the Q latent chunks are dead (its QKs are done): W^UV_(b),(h) lands there,
  // and Z_hi / Z_lo take the two P buffers.
  static constexpr int kQ = 0;
  static constexpr int kQBytes = (kLatChunks + 1) * kPfChunk;
  static constexpr int kKV = kQ + kQBytes;
  static constexpr int kKVStage = (kLatChunks + 1) * kPfChunk;
  static constexpr int kP = kKV + 2 * kKVStage;
  static constexpr int kPBytes = 2 * kPfChunk;  // 128 keys
  static constexpr int kW = kQ;
  static constexpr int kWBytes = kDhChunks * DLAT * 128;  // [DLAT rows][64 cols] per dh chunk
  static_assert(kWBytes <= kLatChunks * kPfChunk, "W^UV must fit the Q latent region");
  static constexpr int kBar = kP + 2 * kPBytes;
  static constexpr int kSmem = kBar + 192 + 6 * kPfT * 4;  // barriers, TMEM base, pair exchange slots
  static_assert(kLatChunks * kPfChunk <= kPBytes, "Z_hi must fit the P buffer");
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t S_COL = 0, O_COL = 2 * kPfT, OUT_COL = 2 * kPfT + DLAT;
  static_assert(OUT_COL + DH <= kTmemCols, "TMEM budget");
};

// Bounded mbarrier wait: a broken pipeline invariant traps (with the barrier id and phase
// printed) instead of hanging the GPU.
#ifdef MLRA_PF_WAIT_STATS
// dev build only (-DMLRA_PF_WAIT_STATS): per-barrier-id wait cycles of CTA 0 summed over the
// waiting threads (tools/prefill_waits.py); the product build has no hook in the wait path
__device__ unsigned long long* g_pf_wait_acc = nullptr;
#endif

__device__ __forceinline__ void pf_wait(uint64_t* bar, uint32_t parity, int id) {
#ifdef MLRA_PF_WAIT_STATS
  if (g_pf_wait_acc != nullptr && blockIdx.x == 0) {
    const long long ts = clock64();
    while (!mbar_try_wait(bar, parity)) {
    }
    atomicAdd(g_pf_wait_acc + id, (unsigned long long)(clock64() - ts));
    return;
  }
#endif
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
    if (clock64() - t0 > 4000000000ll) {
      printf("prefill_attention: stuck on barrier %d parity %u (cta %d, thread %d)\n", id, parity, int(blockIdx.x),
             int(threadIdx.x));
      __trap();
    }
  }
}

__device__ __forceinline__ uint32_t pf_tmem_lane(uint32_t base, int warp) {
  return base + ((uint32_t(warp & 3) * 32u) << 16);
}

template <int DLAT, int DH>
__global__ void __launch_bounds__(kPfThreads, 1)
    prefill_attention_kernel(const __grid_constant__ CUtensorMap lat_map, const __grid_constant__ CUtensorMap rope_map,
                             const __grid_constant__ CUtensorMap q_map, const __grid_constant__ CUtensorMap qr_map,
                             const __grid_constant__ CUtensorMap w_map, const PrefillParams p) {
  using L = PrefillLayout<DLAT, DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* q_full = bars + 0;      // Q (latent chunks of branch b; + rope for b = 0) landed
  uint64_t* w_full = bars + 1;      // W^UV_(b),(h) landed
  uint64_t* kv_full = bars + 2;     // [2]
  uint64_t* kv_empty = bars + 4;    // [2]
  uint64_t* s_full = bars + 6;      // [2]
  uint64_t* s_empty = bars + 8;     // [2]
  uint64_t* p_full = bars + 10;     // [2] P buffer ready for its PV
  uint64_t* pv_done = bars + 12;    // [2] the PV of that P buffer (and every MMA before it) completed
  uint64_t* z_full = bars + 14;     // Z_b hi / lo in smem
  uint64_t* up_done = bars + 15;    // branch b's up-projection (and everything before) completed
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(bars + 16);

  const int nqt = (p.n + kPfT - 1) / kPfT;
  const int lin = blockIdx.x;
  const int qt = nqt - 1 - lin / p.H, h = lin % p.H;  // longest query tiles first
  const int ntiles = qt + 1;                          // causal: key tiles 0..qt
  const int NB = p.NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    tma_prefetch_desc(&lat_map);
    tma_prefetch_desc(&rope_map);
    tma_prefetch_desc(&q_map);
    tma_prefetch_desc(&qr_map);
    tma_prefetch_desc(&w_map);
    mbar_init(q_full, 1);
    mbar_init(w_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 256);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], 256);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(z_full, 256);
    mbar_init(up_done, 1);
    fence_barrier_init();
  }
  PF_PROG(warp, 1);
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_sh);
  PF_PROG(warp, 2);
  tc_fence_before();
  __syncthreads();
  PF_PROG(warp, 3);
  tc_fence_after();
  const uint32_t tbase = *tmem_sh;
  const uint32_t sm = smem_u32(smem);

  if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0) {
      int g = 0;  // global key-tile counter (ring slot / phase)
      for (int b = 0; b < NB; ++b) {
        if (b > 0) pf_wait(up_done, (b - 1) & 1, 1);  // Q latent region / W region free again
        mbar_arrive_expect_tx(q_full, (L::kLatChunks + (b == 0 ? 1 : 0)) * kPfChunk);
        for (int c = 0; c < L::kLatChunks; ++c)
          tma_load_4d(&q_map, q_full, smem + L::kQ + c * kPfChunk, c * 64, b, qt * kPfT, h);
        if (b == 0) tma_load_3d(&qr_map, q_full, smem + L::kQ + L::kLatChunks * kPfChunk, 0, h, qt * kPfT);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int s = g & 1;
          PF_PROG(0, 100 + g);
          pf_wait(&kv_empty[s], ((g >> 1) & 1) ^ 1, 13);
          const int tok0 = j * kPfT;
          const int page = __ldg(p.block_table + min(tok0 / p.page_size, p.max_pages - 1));
          const int row = page * p.page_size + tok0 % p.page_size;
          uint8_t* dst = smem + L::kKV + s * L::kKVStage;
          mbar_arrive_expect_tx(&kv_full[s], L::kKVStage);
          tma_load_3d(&lat_map, &kv_full[s], dst, 0, row, b * L::kLatChunks);
          tma_load_2d(&rope_map, &kv_full[s], dst + L::kLatChunks * kPfChunk, p.rope_col, row);
        }
        // W^UV_(b),(h) into the Q latent region once the branch's MMAs (its last PV) completed
        pf_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 15);
        mbar_arrive_expect_tx(w_full, L::kWBytes);
        for (int c = 0; c < L::kDhChunks; ++c)
          tma_load_2d(&w_map, w_full, smem + L::kW + c * DLAT * 128, c * 64, (h * NB + b) * DLAT);
      }
    }
    __syncwarp();  // reconverge before the CTA barrier (an aligned barrier needs the whole warp)
  } else if (warp == 1 || warp == kPfPvWarp) {
    // ============================================================ MMA issuers (elected lane each)
    // Warp 1 issues every QK as soon as its K/V tile and S slot are there (up to two tiles
    // ahead of the softmax); warp 10 issues every PV as soon as its P is, then the branch's
    // up-projection. With one issuer, QK(j+2) queued behind the wait for P(j) and the
    // softmax sat idle waiting for S. tcgen05.commit tracks the issuing thread's MMAs: PV(j)
    // exists only after S(j) = QK(j) completed, so the PV warp's commits also release the K/V
    // stage QK(j) read.
    const uint64_t kmaj = make_sdesc(0, 16, 1024, kSw128);         // K-major, 128B swizzle
    const uint64_t vmaj = make_sdesc(0, kPfChunk, 1024, kSw128);   // MN-major V (LBO = next 64 columns)
    const uint64_t wmaj = make_sdesc(0, DLAT * 128, 1024, kSw128); // MN-major W^UV (LBO = next 64 columns)
    constexpr uint32_t idesc_qk = make_idesc_bf16(kPfT, kPfT, false, false);
    constexpr uint32_t idesc_pv = make_idesc_bf16(kPfT, DLAT, false, true);
    constexpr uint32_t idesc_up = make_idesc_bf16(kPfT, DH, false, true);
    const int kq_rope = (p.DR + 15) / 16;
    const uint32_t q_addr = sm + L::kQ, p_addr = sm + L::kP, w_addr = sm + L::kW;
    int g = 0;
    for (int b = 0; b < NB; ++b) {
      if (warp == 1) {
        pf_wait(q_full, b & 1, 2);
        tc_fence_after();
        PF_PROG(1, 100 + g);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int s = g & 1;
          pf_wait(&kv_full[s], (g >> 1) & 1, 3);
          pf_wait(&s_empty[s], ((g >> 1) & 1) ^ 1, 14);
          tc_fence_after();
          const uint32_t kv = sm + L::kKV + s * L::kKVStage;
          const uint32_t d = tbase + L::S_COL + s * kPfT;
          uint32_t acc = 0;
#pragma unroll
          for (int c = 0; c < L::kLatChunks; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              mma_bf16_ss_w(d, kmaj + ((q_addr + c * kPfChunk + kk * 32) >> 4),
                            kmaj + ((kv + c * kPfChunk + kk * 32) >> 4), idesc_qk, acc);
              acc = 1;
            }
          for (int kk = 0; kk < kq_rope; ++kk)
            mma_bf16_ss_w(d, kmaj + ((q_addr + L::kLatChunks * kPfChunk + kk * 32) >> 4),
                          kmaj + ((kv + L::kLatChunks * kPfChunk + kk * 32) >> 4), idesc_qk, 1);
          mma_commit_w(&s_full[s]);
        }
      } else {
        PF_PROG(kPfPvWarp, 100 + g);
        for (int j = 0; j < ntiles; ++j, ++g) {
          const int s = g & 1;
          pf_wait(&p_full[s], (g >> 1) & 1, 4);
          tc_fence_after();
          const uint32_t kv = sm + L::kKV + s * L::kKVStage, pb = p_addr + s * L::kPBytes;
#pragma unroll
          for (int k = 0; k < kPfT / 16; ++k)  // 16 keys per step: P chunk k/4, V rows 16k..
            mma_bf16_ss_w(tbase + L::O_COL, kmaj + ((pb + (k >> 2) * kPfChunk + (k & 3) * 32) >> 4),
                          vmaj + ((kv + k * 2048) >> 4), idesc_pv, (j > 0 || k > 0) ? 1u : 0u);
          mma_commit_w(&kv_empty[s]);
          mma_commit_w(&pv_done[s]);
        }
        // up-projection of branch b into OUT (ascending branch order: the reference's sum order)
        pf_wait(z_full, b & 1, 5);
        pf_wait(w_full, b & 1, 6);
        tc_fence_after();
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // Z_hi (P buffer 0), Z_lo (P buffer 1)
          const uint32_t z = p_addr + half * L::kPBytes;
#pragma unroll
          for (int k = 0; k < DLAT / 16; ++k)
            mma_bf16_ss_w(tbase + L::OUT_COL, kmaj + ((z + (k >> 2) * kPfChunk + (k & 3) * 32) >> 4),
                          wmaj + ((w_addr + k * 2048) >> 4), idesc_up, (b > 0 || half > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit_w(up_done);
      }
    }
  } else {
    // ============================================================ softmax / epilogue
    // Two warps per TMEM lane quarter: thread = (query row r, column half hf). The row max is
    // combined across the pair through smem (one named barrier per tile), each thread keeps
    // its half's softmax sum, rescales its half of O's row and writes its half of P (one P
    // chunk = 64 keys).
    const int sw = warp - 2, hf = sw >> 2;
    const int r = (warp & 3) * 32 + lane;  // TMEM lane = query row within the tile
    const int q = qt * kPfT + r;           // query token index
    const uint32_t trow = pf_tmem_lane(tbase, warp);
    uint8_t* prow = smem + L::kP + hf * kPfChunk + r * 128;  // + (g & 1) * kPBytes
    // pair exchange slots [3][2][128]: the tile max of global tile g in slot g & 1 (a thread is at
    // most one tile ahead of its partner: one pair barrier per tile), the row sums in slot 2
    float* xmax = reinterpret_cast<float*>(smem + L::kBar + 192);
    const int pair_bar = 1 + (warp & 3);                           // named barrier of the warp pair
    int g = 0;
    for (int b = 0; b < NB; ++b) {
      if (b > 0) pf_wait(up_done, (b - 1) & 1, 7);  // the P region held Z_hi of branch b-1
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < ntiles; ++j, ++g) {
        const int s = g & 1;
        PF_PROG(warp, 100 + g);
        pf_wait(&s_full[s], (g >> 1) & 1, 8);
        tc_fence_after();
        uint32_t sv[64];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld16(trow + L::S_COL + s * kPfT + hf * 64 + c * 16, sv + c * 16);
        tmem_ld_wait();
        if (p.dbg_s != nullptr && g == 0 && int(blockIdx.x) == p.dbg_cta)
          for (int c = 0; c < 64; ++c) p.dbg_s[r * kPfT + hf * 64 + c] = __uint_as_float(sv[c]);
        tc_fence_before();
        mbar_arrive(&s_empty[s]);
        // causal mask on the diagonal tile (and the sequence end): keys [0, kmax] visible
        const int kmax = min(q, p.n - 1) - j * kPfT - hf * 64;
        // (8 independent max / sum chains: a single 64-long dependent chain cost ~4 cycles an element)
        float tm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) tm[i] = -INFINITY;
        if (__all_sync(0xffffffffu, kmax >= 63)) {
#pragma unroll
          for (int c = 0; c < 64; ++c) tm[c & 7] = fmaxf(tm[c & 7], __uint_as_float(sv[c]));
        } else {
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const float x = c <= kmax ? __uint_as_float(sv[c]) : -INFINITY;
            sv[c] = __float_as_uint(x);
            tm[c & 7] = fmaxf(tm[c & 7], x);
          }
        }
        float tmax = fmaxf(fmaxf(fmaxf(tm[0], tm[1]), fmaxf(tm[2], tm[3])), fmaxf(fmaxf(tm[4], tm[5]), fmaxf(tm[6], tm[7])));
        float* xs = xmax + (g & 1) * 2 * kPfT;
        xs[hf * kPfT + r] = tmax;
        named_bar_sync(pair_bar, 64);
        tmax = fmaxf(tmax, xs[(hf ^ 1) * kPfT + r]);
        // Lazy rescale: a row moves its running max only when its tile max exceeds it by 2^8
        // (or on its first visible tile). tcgen05.ld / st are warp-collective, so the warp
        // rescales its half of O in TMEM if ANY of its rows moved (factor 1 for the others),
        // after the PVs issued so far have completed. Rows still fully masked hold O = 0.
        const bool move = tmax > m + 8.0f || m == -INFINITY;
        const float m_new = move ? fmaxf(m, tmax) : m;
        const float sc = (move && m != -INFINITY) ? ex2(m - m_new) : 1.f;
        if (j > 0 && __any_sync(0xffffffffu, sc != 1.f)) {
          pf_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 9);  // every PV so far completed
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < DLAT / 32; ++c) {
            uint32_t o[16];
            tmem_ld16(trow + L::O_COL + hf * (DLAT / 2) + c * 16, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * sc);
            tmem_st8(trow + L::O_COL + hf * (DLAT / 2) + c * 16, o);
            tmem_st8(trow + L::O_COL + hf * (DLAT / 2) + c * 16 + 8, o + 8);
          }
          tmem_st_wait();
        }
        l *= sc;
        m = m_new;
        const float mu = m;
        // P = 2^(S - m) as bf16 into the P buffer (free once the previous PV completed)
        if (g >= 2) pf_wait(&pv_done[g & 1], ((g >> 1) - 1) & 1, 10);  // this buffer's last PV read it
        float sm[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) sm[i] = 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t w4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k0 = u * 8 + 2 * e;
            const float p0 = (mu == -INFINITY) ? 0.f : ex2(__uint_as_float(sv[k0]) - mu);
            const float p1 = (mu == -INFINITY) ? 0.f : ex2(__uint_as_float(sv[k0 + 1]) - mu);
            sm[(2 * e) & 7] += p0;
            sm[(2 * e + 1) & 7] += p1;
            w4[e] = pack_bf16(p0, p1);
          }
          *reinterpret_cast<uint4*>(prow + s * L::kPBytes + ((u ^ (r & 7)) * 16)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        l += ((sm[0] + sm[1]) + (sm[2] + sm[3])) + ((sm[4] + sm[5]) + (sm[6] + sm[7]));
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[s]);
      }
      // Z_b = O / l -> bf16 hi (P region) + lo (Q latent region: the branch's QKs are done);
      // the row's sum is the pair's two halves
      xmax[4 * kPfT + hf * kPfT + r] = l;
      named_bar_sync(pair_bar, 64);
      const float lt = l + xmax[4 * kPfT + (hf ^ 1) * kPfT + r];
      pf_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1, 11);  // the branch's last PV (and all before)
      tc_fence_after();
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      uint8_t* zhi = smem + L::kP + r * 128;
      uint8_t* zlo = smem + L::kP + L::kPBytes + r * 128;
#pragma unroll
      for (int c = 0; c < DLAT / 32; ++c) {
        uint32_t o[16];
        const int col0 = hf * (DLAT / 2) + c * 16;
        tmem_ld16(trow + L::O_COL + col0, o);
        tmem_ld_wait();
#pragma unroll
        for (int u2 = 0; u2 < 2; ++u2) {
          uint32_t hv[4], lv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float z0 = __uint_as_float(o[u2 * 8 + 2 * e]) * inv, z1 = __uint_as_float(o[u2 * 8 + 2 * e + 1]) * inv;
            const __nv_bfloat16 h0 = __float2bfloat16_rn(z0), h1 = __float2bfloat16_rn(z1);
            hv[e] = pack_bf16_raw(h0, h1);
            lv[e] = pack_bf16(z0 - __bfloat162float(h0), z1 - __bfloat162float(h1));
          }
          const int col = col0 + u2 * 8;  // latent column of this 16-byte unit
          const int chunk = col / 64, u = (col % 64) / 8;
          *reinterpret_cast<uint4*>(zhi + chunk * kPfChunk + ((u ^ (r & 7)) * 16)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<uint4*>(zlo + chunk * kPfChunk + ((u ^ (r & 7)) * 16)) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(z_full);
    }
    // OUT -> alpha * OUT for the real query rows (each thread half of the columns)
    pf_wait(up_done, (NB - 1) & 1, 12);
    tc_fence_after();
    float* dst = p.out + (size_t(q) * p.H + h) * DH;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t o[16];
      const int col0 = hf * (DH / 2) + c * 16;
      tmem_ld16(trow + L::OUT_COL + col0, o);  // warp-collective: every lane, stores only real rows
      tmem_ld_wait();
      if (q < p.n) {
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(dst + col0 + e) =
              make_float4(__uint_as_float(o[e]) * p.alpha, __uint_as_float(o[e + 1]) * p.alpha,
                          __uint_as_float(o[e + 2]) * p.alpha, __uint_as_float(o[e + 3]) * p.alpha);
      }
    }
  }
  PF_PROG(warp, 5000);
  tc_fence_before();
  __syncthreads();
  PF_PROG(warp, 6000);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<L::kTmemCols>(tbase);
  }
}

// ---- prefill projection helpers (the n-row projections run as cuBLAS bf16 GEMMs) -----------
// rows_split: per row x -> (alpha * rmsnorm(x) when norm, else x) as bf16 hi + lo planes (row
// stride ldo: two [n, K] planes, or the halves of one [n, 2K] operand)
// (the GEMM's activations at ~16-bit mantissa; tensors.py:83-87 rmsnorm, latent.py:134).
__global__ void __launch_bounds__(256) rows_split_kernel(const float* __restrict__ x, int K, int ldx, int norm,
                                                         float alpha, float eps, __nv_bfloat16* __restrict__ hi,
                                                         __nv_bfloat16* __restrict__ lo, int ldo) {
  __shared__ float red[8];
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* xr = x + size_t(row) * ldx;
  float sc = 1.f;
  if (norm) {
    float ss = 0.f;
    for (int c = tid; c < K; c += 256) ss = fmaf(xr[c], xr[c], ss);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w];
    sc = alpha * rsqrtf(t / float(K) + eps);
  }
  for (int c = tid; c < K; c += 256) {
    const float v = xr[c] * sc;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi[size_t(row) * ldo + c] = h;
    lo[size_t(row) * ldo + c] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

// query_epilogue: y [n, ldy] fp32 = [q_x (nq) | q_r (H * dr)] -> q_out bf16 [n, nq] = q_scale * q_x,
// r_out bf16 [n, H, drq] = r_scale * rope(q_r, pos0 + row) (pairs (2l, 2l+1), rope.py:37-60),
// columns [dr, drq) zero. The row's dr/2 angles (fp64 product, reduced mod 2 pi) and their
// sin / cos are formed once into smem and shared by the H heads.
__global__ void __launch_bounds__(256) query_epilogue_kernel(const float* __restrict__ y, int ldy, int nq, int H,
                                                             int dr, int drq, int pos0, float rope_base,
                                                             float q_scale, float r_scale,
                                                             __nv_bfloat16* __restrict__ q_out,
                                                             __nv_bfloat16* __restrict__ r_out) {
  __shared__ float cs_sh[64], sn_sh[64];
  const int row = blockIdx.x, tid = threadIdx.x;
  const float* yr = y + size_t(row) * ldy;
  if (tid < dr / 2) {
    const double theta = pow(double(rope_base), -2.0 * tid / dr);
    const double a = double(pos0 + row) * theta;
    const double two_pi = 6.283185307179586476925286766559;
    float sn, cs;
    sincosf(float(a - two_pi * floor(a / two_pi)), &sn, &cs);
    cs_sh[tid] = cs;
    sn_sh[tid] = sn;
  }
  for (int c = tid * 4; c < nq; c += 256 * 4) {
    if (c + 4 <= nq && (nq % 4) == 0) {
      const float4 v = *reinterpret_cast<const float4*>(yr + c);
      uint2 o;
      o.x = pack_bf16(v.x * q_scale, v.y * q_scale);
      o.y = pack_bf16(v.z * q_scale, v.w * q_scale);
      *reinterpret_cast<uint2*>(q_out + size_t(row) * nq + c) = o;
    } else {
      for (int j = c; j < min(nq, c + 4); ++j) q_out[size_t(row) * nq + j] = __float2bfloat16_rn(yr[j] * q_scale);
    }
  }
  __syncthreads();
  for (int i = tid; i < H * (drq / 2); i += 256) {
    const int h = i / (drq / 2), l = i % (drq / 2);
    float e = 0.f, o = 0.f;
    if (2 * l + 1 < dr) {
      const float x0 = yr[nq + h * dr + 2 * l], x1 = yr[nq + h * dr + 2 * l + 1];
      e = (x0 * cs_sh[l] - x1 * sn_sh[l]) * r_scale;
      o = (x0 * sn_sh[l] + x1 * cs_sh[l]) * r_scale;
    }
    reinterpret_cast<__nv_bfloat162*>(r_out + (size_t(row) * H + h) * drq)[l] = __floats2bfloat162_rn(e, o);
  }
}

}  // namespace mlra
