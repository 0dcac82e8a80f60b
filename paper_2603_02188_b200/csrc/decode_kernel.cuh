// K2: split-KV flash-decode over the paged latent cache, tcgen05 tensor cores + TMA.
//
// Replaces the hot loop of attnkit/decode.py:217-230 (attend_local, latent branch):
//   logits_b = tau * (q~_b . C_b^T + q_rope . K_rope^T);  P = softmax;  Z_b = P . C_b
// for every branch b a GPU owns, over the tokens [tile range) of one sequence, and emits
// per-split partials (Z normalised by its own softmax sum, plus log2-sum-exp) that K3
// (combine_kernel.cuh) merges and up-projects.
//
// Swap-AB formulation: the MMA M dimension is the KV tile (tokens for QK^T, latent rows
// for PV), the N dimension is the (padded) head group. So one TMEM lane = one token (QK)
// or one latent row (PV) and the softmax reduction over tokens is a cross-lane reduction
// done with warp shuffles (reduce-scatter) plus one named barrier across the 4 lane
// quarters.
//
// Pool row layout (width W): [branch 0 latent | branch 1 latent | ... | rope], each branch
// latent = SUB sub-blocks of DLS columns. The same smem tile serves as K (K-major A
// operand of QK) and as V (MN-major A operand of PV): V = the latent columns of K.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer,
// warps 2..5 = softmax / rescale / epilogue (TMEM lane quarter = warp % 4).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>
#include "ptx.cuh"

namespace mlra {

struct DecodeParams {
  const __nv_bfloat16* q_abs;   // [B, NB, H, NB_LAT]  absorbed queries, pre-scaled by tau*log2(e)
  const __nv_bfloat16* q_rope;  // [B, H, DR]          rotary queries, pre-scaled by tau*log2(e)
  const int32_t* block_table;   // [B, max_pages]
  const int32_t* seqlens;       // [B]
  float* o_part;                // [B, nsplit, NB, H, DLAT]  Z / l per split
  float* lse_part;              // [B, nsplit, NB, H]        m + log2(l) per split (log2 domain)
  int B, H, NB, SUB, DR, W;     // W = NB*SUB*DLS + DR (pool row width, elements)
  int page_size, max_pages, nsplit;
  int lat_slots, rope_slots;    // ring depths (set by the host from the smem budget)
  float rescale_threshold;      // lazy-rescale threshold (log2 units)
};

constexpr int kNumThreads = 192;
constexpr float kRescaleThreshold = 8.0f;  // lazy rescale (log2 units): P stays <= 2^8

template <int T, int NPAD, int DLS>
struct DecodeLayout {
  static constexpr int kChunkBytes = T * 128;                   // [T rows x 64 cols] bf16, 128B swizzle
  static constexpr int kLatBytes = (DLS / 64) * kChunkBytes;    // one sub-block
  static constexpr int kRopeBytes = kChunkBytes;                // rope <= 64 cols
  static constexpr int kQChunkBytes = NPAD * 128;
  static constexpr int kPBytes = T * NPAD * 2;
  static constexpr int kPSbo = (T / 8) * 128;                   // MN-group stride of the P operand
  // red[2][4][NPAD] + mw[4][NPAD] + aw[4][NPAD] + m_run[4][4][NPAD] + l_run[4][4][NPAD] + invl[4][NPAD]
  static constexpr int kScratchBytes = ((52 * NPAD * 4 + 1023) / 1024) * 1024;
  static int smem_bytes(int NB, int SUB, int lat_slots, int rope_slots) {
    const int q_chunks = NB * SUB * (DLS / 64) + 1;
    return 1024 /*align slack*/ + lat_slots * kLatBytes + rope_slots * kRopeBytes + q_chunks * kQChunkBytes +
           2 * kPBytes + kScratchBytes;
  }
};

// Reduce NPAD per-thread values across the 32 lanes of a warp so that afterwards each
// lane holds the reduction for its own heads (reduce-scatter; 31 shuffles for NPAD=32).
// Head of value i in lane l: see head_of().
template <int NPAD>
struct LaneHeads {
  static constexpr int kVals = NPAD >= 32 ? NPAD / 32 : 1;
  __device__ static int head_of(int lane, int i) {
    if constexpr (NPAD >= 32) return lane * kVals + i;
    else return lane / (32 / NPAD);
  }
  __device__ static bool owner(int lane) {
    if constexpr (NPAD >= 32) return true;
    else return (lane % (32 / NPAD)) == 0;
  }
};

template <int NPAD, bool kMax>
__device__ __forceinline__ void reduce_scatter(float (&v)[NPAD], float (&out)[LaneHeads<NPAD>::kVals]) {
  const int lane = lane_id();
  // Level k halves the live array; lanes with the offset bit set keep the upper half.
  // Heads end up in lane-major order (head = lane*kVals + i for NPAD >= 32).
  constexpr int kLevels = (NPAD >= 32) ? 5 : (NPAD == 16 ? 4 : (NPAD == 8 ? 3 : 0));
  static_assert(NPAD == 16 || NPAD == 32 || NPAD == 64, "NPAD must be 16, 32 or 64");
#pragma unroll
  for (int lvl = 0; lvl < kLevels; ++lvl) {
    const int off = 16 >> lvl;
    const int half = NPAD >> (lvl + 1);
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = upper ? v[i + half] : v[i];
      const float send = upper ? v[i] : v[i + half];
      const float recv = __shfl_xor_sync(0xffffffffu, send, off);
      v[i] = kMax ? fmaxf(keep, recv) : keep + recv;
    }
  }
  if constexpr (NPAD >= 32) {
#pragma unroll
    for (int i = 0; i < NPAD / 32; ++i) out[i] = v[i];
  } else {
    // remaining lanes holding the same head: finish with butterflies on the low lane bits
    float x = v[0];
#pragma unroll
    for (int off = (32 / NPAD) / 2; off >= 1; off >>= 1) {
      const float y = __shfl_xor_sync(0xffffffffu, x, off);
      x = kMax ? fmaxf(x, y) : x + y;
    }
    out[0] = x;
  }
}

template <int T, int NPAD, int DLS>
__global__ void __launch_bounds__(kNumThreads, 1)
    mlra_decode_kernel(const __grid_constant__ CUtensorMap pool_map, const DecodeParams p) {
  using L = DecodeLayout<T, NPAD, DLS>;
  using LH = LaneHeads<NPAD>;
  static_assert(T == 64 || T == 128, "token tile must be 64 or 128");
  static_assert(DLS == 64 || DLS == 128, "sub-block width must be 64 or 128");

  const int NB = p.NB, SUB = p.SUB;
  const int DLAT = SUB * DLS;  // latent width of one branch
  const int seq = blockIdx.y, split = blockIdx.x, hg = blockIdx.z;
  const int len = p.seqlens[seq];
  const int ntiles_total = (len + T - 1) / T;
  const int per = (ntiles_total + p.nsplit - 1) / p.nsplit;
  const int t0 = min(split * per, ntiles_total);
  const int ntiles = min(per, ntiles_total - t0);
  const int R = ntiles * NB;  // rounds: (tile, branch)
  const int n_valid_pages = (len + p.page_size - 1) / p.page_size;

  // ------------------------------------------------------------- shared memory carve-up
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* lat_ring = base;
  uint8_t* rope_ring = lat_ring + p.lat_slots * L::kLatBytes;
  uint8_t* q_smem = rope_ring + p.rope_slots * L::kRopeBytes;
  const int q_chunks = NB * SUB * (DLS / 64) + 1;
  uint8_t* p_smem = q_smem + q_chunks * L::kQChunkBytes;
  float* scratch = reinterpret_cast<float*>(p_smem + 2 * L::kPBytes);
  float* red = scratch;                         // [2][4][NPAD] per-quarter tile maxima
  float* mw = red + 2 * 4 * NPAD;               // [4][NPAD] per-warp m in use
  float* aw = mw + 4 * NPAD;                    // [4][NPAD] per-warp rescale factor
  float* m_run = aw + 4 * NPAD;                 // [4][NB][NPAD]
  float* l_run = m_run + 4 * 4 * NPAD;          // [4][NB][NPAD]
  float* invl = l_run + 4 * 4 * NPAD;           // [NB][NPAD]

  __shared__ uint64_t lat_full[16], lat_empty[16], rope_full[8], rope_empty[8];
  __shared__ uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_done[4], o_final;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid / 32, lane = lane_id();
  // TMEM columns: S slots [0, 2*NPAD), O_{b,s} at 2*NPAD + (b*SUB+s)*NPAD
  constexpr uint32_t kTmemCols = 512;
  const uint32_t S_COL = 0, O_COL = 2 * NPAD;

  if (tid == 0) {
    for (int i = 0; i < p.lat_slots; ++i) { mbar_init(&lat_full[i], 1); mbar_init(&lat_empty[i], 1); }
    for (int i = 0; i < p.rope_slots; ++i) { mbar_init(&rope_full[i], 1); mbar_init(&rope_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], 128);
      mbar_init(&p_full[i], 128); mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&o_done[i], 1);
    mbar_init(&o_final, 1);
    fence_barrier_init();
    tma_prefetch_desc(&pool_map);
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&tmem_base_sh);

  // Absorbed + rotary queries of this (sequence, head group) -> K-major SW128 chunks.
  // Chunk (b, c) holds latent columns [c*64, c*64+64) of branch b; the last chunk is rope.
  {
    const int nlat_chunks = NB * SUB * (DLS / 64);
    const int units_per_row = 8;  // 16-byte units per 128-byte chunk row
    const int total = q_chunks * NPAD * units_per_row;
    for (int idx = tid; idx < total; idx += kNumThreads) {
      const int chunk = idx / (NPAD * units_per_row);
      const int rem = idx % (NPAD * units_per_row);
      const int r = rem / units_per_row, u = rem % units_per_row;
      const int h = hg * NPAD + r;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (h < p.H) {
        if (chunk < nlat_chunks) {
          const int b = chunk / (DLAT / 64), c = chunk % (DLAT / 64);
          const __nv_bfloat16* src = p.q_abs + ((size_t(seq) * NB + b) * p.H + h) * DLAT + c * 64 + u * 8;
          v = *reinterpret_cast<const uint4*>(src);
        } else if (u * 8 < p.DR) {
          v = *reinterpret_cast<const uint4*>(p.q_rope + (size_t(seq) * p.H + h) * p.DR + u * 8);
        }
      }
      *reinterpret_cast<uint4*>(q_smem + chunk * L::kQChunkBytes + r * 128 + ((u ^ (r & 7)) * 16)) = v;
    }
    for (int i = tid; i < 4 * 4 * NPAD; i += kNumThreads) { m_run[i] = -INFINITY; l_run[i] = 0.f; }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0 && R > 0) {
      const uint64_t policy = l2_policy_evict_first();
      const int rope_col = NB * DLAT;
      int li = 0;
      for (int t = 0; t < ntiles; ++t) {
        int rows[T / 64];
#pragma unroll
        for (int i = 0; i < T / 64; ++i) {
          const int tok0 = (t0 + t) * T + 64 * i;
          int page = tok0 / p.page_size;
          page = min(page, n_valid_pages - 1);
          rows[i] = p.block_table[size_t(seq) * p.max_pages + page] * p.page_size + (tok0 % p.page_size);
        }
        {
          const int slot = t % p.rope_slots;
          mbar_wait(&rope_empty[slot], ((t / p.rope_slots) & 1) ^ 1);
          mbar_arrive_expect_tx(&rope_full[slot], L::kRopeBytes);
#pragma unroll
          for (int i = 0; i < T / 64; ++i)
            tma_load_2d_hint(&pool_map, &rope_full[slot], rope_ring + slot * L::kRopeBytes + i * 8192, rope_col,
                             rows[i], policy);
        }
        for (int u = 0; u < NB * SUB; ++u, ++li) {
          const int slot = li % p.lat_slots;
          mbar_wait(&lat_empty[slot], ((li / p.lat_slots) & 1) ^ 1);
          mbar_arrive_expect_tx(&lat_full[slot], L::kLatBytes);
#pragma unroll
          for (int c = 0; c < DLS / 64; ++c)
#pragma unroll
            for (int i = 0; i < T / 64; ++i)
              tma_load_2d_hint(&pool_map, &lat_full[slot],
                               lat_ring + slot * L::kLatBytes + c * L::kChunkBytes + i * 8192, u * DLS + c * 64,
                               rows[i], policy);
        }
      }
    }
  } else if (warp == 1) {
    // ============================================================ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(T, NPAD, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(DLS, NPAD, true, true);
      const int kq_rope = (p.DR + 15) / 16;
      for (int r = 0; r <= R; ++r) {
        if (r < R) {
          const int t = r / NB, b = r % NB, sslot = r & 1;
          mbar_wait(&s_empty[sslot], ((r >> 1) & 1) ^ 1);
          mbar_wait(&rope_full[t % p.rope_slots], (t / p.rope_slots) & 1);
          const uint32_t d = tbase + S_COL + sslot * NPAD;
          uint32_t acc = 0;
          for (int s = 0; s < SUB; ++s) {
            const int li = (t * NB + b) * SUB + s;
            const int slot = li % p.lat_slots;
            mbar_wait(&lat_full[slot], (li / p.lat_slots) & 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(lat_ring + slot * L::kLatBytes);
            const uint32_t b0 = smem_u32(q_smem + ((b * SUB + s) * (DLS / 64)) * L::kQChunkBytes);
#pragma unroll
            for (int c = 0; c < DLS / 64; ++c)
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                mma_bf16_ss(d, make_sdesc(a0 + c * L::kChunkBytes + kk * 32, 16, 1024, kSw128),
                            make_sdesc(b0 + c * L::kQChunkBytes + kk * 32, 16, 1024, kSw128), idesc_qk, acc);
                acc = 1;
              }
          }
          tc_fence_after();
          {
            const uint32_t a0 = smem_u32(rope_ring + (t % p.rope_slots) * L::kRopeBytes);
            const uint32_t b0 = smem_u32(q_smem + (NB * SUB * (DLS / 64)) * L::kQChunkBytes);
            for (int kk = 0; kk < kq_rope; ++kk)
              mma_bf16_ss(d, make_sdesc(a0 + kk * 32, 16, 1024, kSw128), make_sdesc(b0 + kk * 32, 16, 1024, kSw128),
                          idesc_qk, 1);
          }
          mma_commit(&s_full[sslot]);
          if (b == NB - 1) mma_commit(&rope_empty[t % p.rope_slots]);
        }
        if (r >= 1) {
          const int rp = r - 1, t = rp / NB, b = rp % NB, pslot = rp & 1;
          mbar_wait(&p_full[pslot], (rp >> 1) & 1);
          tc_fence_after();
          const uint32_t pb = smem_u32(p_smem + pslot * L::kPBytes);
          for (int s = 0; s < SUB; ++s) {
            const int li = (t * NB + b) * SUB + s;
            const int slot = li % p.lat_slots;
            const uint32_t a0 = smem_u32(lat_ring + slot * L::kLatBytes);
            const uint32_t d = tbase + O_COL + (b * SUB + s) * NPAD;
#pragma unroll
            for (int k = 0; k < T / 16; ++k)
              mma_bf16_ss(d, make_sdesc(a0 + k * 2048, L::kChunkBytes, 1024, kSw128),
                          make_sdesc(pb + k * 256, 128, L::kPSbo, kSwNone), idesc_pv, (t > 0 || k > 0) ? 1u : 0u);
            mma_commit(&lat_empty[slot]);
          }
          mma_commit(&p_empty[pslot]);
          mma_commit(&o_done[b]);
        }
      }
      // Single-phase barrier for the epilogue: o_done[b] may lag by two phases there, which
      // a parity wait cannot disambiguate.
      if (R > 0) mma_commit(&o_final);
    }
  } else {
    // ============================================================ softmax / rescale / epilogue
    const int q = warp & 3;                       // TMEM lane quarter owned by this warp
    const bool lane_ok = (T == 128) || (lane < 16);
    const int tok_in_tile = (T == 128) ? q * 32 + lane : q * 16 + lane;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    for (int r = 0; r < R; ++r) {
      const int t = r / NB, b = r % NB, sslot = r & 1;
      mbar_wait(&s_full[sslot], (r >> 1) & 1);
      tc_fence_after();
      float s[NPAD];
      {
        uint32_t raw[NPAD];
#pragma unroll
        for (int c = 0; c < NPAD; c += 16) tmem_ld16(tbase + lane_off + S_COL + sslot * NPAD + c, raw + c);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < NPAD; ++c) s[c] = __uint_as_float(raw[c]);
      }
      tc_fence_before();
      mbar_arrive(&s_empty[sslot]);
      const int tok = (t0 + t) * T + tok_in_tile;
      if (!(lane_ok && tok < len)) {
#pragma unroll
        for (int c = 0; c < NPAD; ++c) s[c] = -INFINITY;
      }
      // ---- tile max per head (reduce over this warp's tokens, then over the 4 quarters)
      float tmp[NPAD];
#pragma unroll
      for (int c = 0; c < NPAD; ++c) tmp[c] = s[c];
      float mx[LH::kVals];
      reduce_scatter<NPAD, true>(tmp, mx);
      float* red_r = red + (r & 1) * 4 * NPAD;
      if (LH::owner(lane)) {
#pragma unroll
        for (int i = 0; i < LH::kVals; ++i) red_r[q * NPAD + LH::head_of(lane, i)] = mx[i];
      }
      named_bar_sync(1, 128);
      bool need = false;
      float alpha[LH::kVals];
#pragma unroll
      for (int i = 0; i < LH::kVals; ++i) {
        const int h = LH::head_of(lane, i);
        const float m_tile = fmaxf(fmaxf(red_r[h], red_r[NPAD + h]), fmaxf(red_r[2 * NPAD + h], red_r[3 * NPAD + h]));
        const float m_old = m_run[(q * 4 + b) * NPAD + h];
        const bool nd = (m_old == -INFINITY) || (m_tile > m_old + p.rescale_threshold);
        const float m_new = nd ? m_tile : m_old;
        alpha[i] = nd ? ex2(m_old - m_new) : 1.f;
        need |= nd;
        if (LH::owner(lane)) {
          mw[q * NPAD + h] = m_new;
          aw[q * NPAD + h] = alpha[i];
          m_run[(q * 4 + b) * NPAD + h] = m_new;
        }
      }
      const bool any_rescale = __any_sync(0xffffffffu, need);
      __syncwarp();
      // ---- probabilities (log2 domain; the score scale is folded into the queries)
      float pr[NPAD];
#pragma unroll
      for (int c = 0; c < NPAD; c += 4) {
        const float4 m4 = *reinterpret_cast<const float4*>(mw + q * NPAD + c);
        pr[c + 0] = ex2(s[c + 0] - m4.x);
        pr[c + 1] = ex2(s[c + 1] - m4.y);
        pr[c + 2] = ex2(s[c + 2] - m4.z);
        pr[c + 3] = ex2(s[c + 3] - m4.w);
      }
      const int pslot = r & 1;
      if (r >= 2) mbar_wait(&p_empty[pslot], ((r >> 1) - 1) & 1);
      if (lane_ok) {
        // B operand of PV, MN-major no-swizzle: (tok, head) at (h/8)*SBO + (tok/8)*128 + (tok%8)*16 + (h%8)*2
        uint8_t* prow = p_smem + pslot * L::kPBytes + (tok_in_tile / 8) * 128 + (tok_in_tile % 8) * 16;
#pragma unroll
        for (int g = 0; g < NPAD / 8; ++g) {
          uint4 v;
          v.x = pack_bf16(pr[g * 8 + 0], pr[g * 8 + 1]);
          v.y = pack_bf16(pr[g * 8 + 2], pr[g * 8 + 3]);
          v.z = pack_bf16(pr[g * 8 + 4], pr[g * 8 + 5]);
          v.w = pack_bf16(pr[g * 8 + 6], pr[g * 8 + 7]);
          *reinterpret_cast<uint4*>(prow + g * L::kPSbo) = v;
        }
      }
      // ---- running softmax sum: per-quarter partial, owned by the head's lane
      float ps[LH::kVals];
      reduce_scatter<NPAD, false>(pr, ps);
      if (LH::owner(lane)) {
#pragma unroll
        for (int i = 0; i < LH::kVals; ++i) {
          float* lr = l_run + (q * 4 + b) * NPAD + LH::head_of(lane, i);
          *lr = *lr * alpha[i] + ps[i];
        }
      }
      // ---- rare: the running max moved by more than the threshold -> rescale O_b in TMEM
      if (any_rescale && t > 0) {
        // PV(t-2, b) is complete (it was issued before QK(t, b), whose S we consumed), so
        // o_done[b] lags phase t-1 by at most one phase and the parity wait is exact.
        mbar_wait(&o_done[b], (t - 1) & 1);
        tc_fence_after();
        for (int sb = 0; sb < SUB; ++sb) {
          const uint32_t taddr = tbase + lane_off + O_COL + (b * SUB + sb) * NPAD;
          uint32_t raw[NPAD];
#pragma unroll
          for (int c = 0; c < NPAD; c += 16) tmem_ld16(taddr + c, raw + c);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < NPAD; ++c) raw[c] = __float_as_uint(__uint_as_float(raw[c]) * aw[q * NPAD + c]);
#pragma unroll
          for (int c = 0; c < NPAD; c += 8) tmem_st8(taddr + c, raw + c);
        }
        tmem_st_wait();
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[pslot]);
    }

    // ============================================================ epilogue: partials
    named_bar_sync(1, 128);
    const size_t part_row0 = (size_t(seq) * p.nsplit + split) * NB;  // (seq, split, b) row index
    for (int b = 0; b < NB; ++b) {
      if (q == 0 && LH::owner(lane)) {
#pragma unroll
        for (int i = 0; i < LH::kVals; ++i) {
          const int h = LH::head_of(lane, i);
          float lt = 0.f;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) lt += l_run[(qq * 4 + b) * NPAD + h];
          const float m = m_run[(0 * 4 + b) * NPAD + h];
          invl[b * NPAD + h] = lt > 0.f ? 1.f / lt : 0.f;
          const int hh = hg * NPAD + h;
          if (hh < p.H) p.lse_part[(part_row0 + b) * p.H + hh] = lt > 0.f ? m + log2f(lt) : -INFINITY;
        }
      }
    }
    named_bar_sync(1, 128);
    const bool row_ok = (DLS == 128) || (lane < 16);
    const int row = (DLS == 128) ? q * 32 + lane : q * 16 + lane;
    if (ntiles > 0) {
      mbar_wait(&o_final, 0);
      tc_fence_after();
    }
    for (int b = 0; b < NB; ++b) {
      for (int sb = 0; sb < SUB; ++sb) {
        float o[NPAD];
        if (ntiles > 0) {
          uint32_t raw[NPAD];
#pragma unroll
          for (int c = 0; c < NPAD; c += 16) tmem_ld16(tbase + lane_off + O_COL + (b * SUB + sb) * NPAD + c, raw + c);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < NPAD; ++c) o[c] = __uint_as_float(raw[c]) * invl[b * NPAD + c];
        } else {
#pragma unroll
          for (int c = 0; c < NPAD; ++c) o[c] = 0.f;
        }
        if (row_ok) {
          float* dst = p.o_part + ((part_row0 + b) * p.H) * size_t(DLAT) + sb * DLS + row;
#pragma unroll
          for (int c = 0; c < NPAD; ++c) {
            const int hh = hg * NPAD + c;
            if (hh < p.H) dst[size_t(hh) * DLAT] = o[c];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tbase);
  }
}

}  // namespace mlra
