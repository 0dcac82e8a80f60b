// Fused decode step: K1 (query absorption) in K2's prologue and K3 (split merge, W^UV
// up-projection, ascending branch sum, alpha, optional TP sum) in K2's epilogue, so one decode
// step of a batch is ONE launch of mlra_decode_kernel (p.fused != 0).
//
// Why: K1 and K3 are latency-bound (a few hundred KB of weights, one L2 round trip each) and as
// separate launches they sit on the critical path of a step (B = 16, 32K, TP4 rank: K1 3.7 us +
// K2 34.3 us + K3 6.2 us). Inside K2 they overlap with work that is already there:
//   * absorb: the 8 softmax warps of the first CTAs compute q~ = q_nope . W^UK (mma.sync,
//     16 sequences x 128 latent columns per unit) while warp 0 of EVERY CTA is already streaming
//     the cache into its ring (the ring holds ~4 us of a CTA's HBM share, so consumers may start
//     that late without losing bandwidth). The consumers wait on a device counter of finished
//     absorb units (grid-wide, all CTAs resident: one CTA per SM, grid <= #SMs, host-checked);
//   * combine: a CTA that has written its split partials bumps its sequence's completion
//     counter; the K3 work units (16-sequence group, head, <=128-wide latent chunk) are spread
//     over the CTAs, each waiting only for the counters of its own sequences, so the merge of
//     early sequences overlaps the decode tail of late ones. A head with several chunks
//     (MLRA-4 TP1: one per branch; MLA: 128-column slices of the 512 latent) is summed in
//     ascending chunk order by the unit that draws the head's last ticket (deterministic).
// The last CTA to exit resets every counter, so the next stream-ordered launch (or CUDA graph
// replay) starts from zero.
//
// Reference: attnkit/decode.py:155-167 (absorb_query), :217-230 (attend_local), :228 (the W^UV
// einsum), :264-285 (reduce_contributions: ascending branch order, then alpha_attn);
// tpsim.py:275-276 (device-order sum) for the TP epilogue.
#pragma once
#include <cstdint>
#include <cmath>
#include "ptx.cuh"
#include "peer_common.cuh"

namespace mlra {

constexpr int kFuseSeqs = 16;       // sequences per absorb / combine unit (the mma.sync M)
constexpr int kFuseMaxSplits = 160; // = kMergeMaxSplits
constexpr int kSyncAbsorb = 0, kSyncExit = 1, kSyncTpEpoch = 2, kSyncSeq = 16;

// Status word bits (include/mlra_b200.h): a softmax row saw a NaN logit / had no finite logit
// (attnkit/tensors.py:74-78).
constexpr int kStatusNaN = 1, kStatusNoFinite = 2;

__host__ __device__ inline int fuse_groups(int B) { return (B + kFuseSeqs - 1) / kFuseSeqs; }
// sync words: counters + per (sequence, head group) completion + per (group, head) tickets
__host__ __device__ inline size_t fuse_sync_words(int B, int H, int hgroups) {
  return size_t(kSyncSeq) + size_t(B) * hgroups + size_t(fuse_groups(B)) * H;
}

// Publication pattern (as CUTLASS's GenericBarrier): every thread's stores, a CTA barrier, then
// ONE thread's release (cumulative: it orders the barrier-synchronised stores of the CTA). No
// per-thread __threadfence (MEMBAR.SC.GPU + L1 invalidation costs microseconds per CTA).
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_acq_rel_add(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// Spin until *p >= target (acquire). Every waiter's producer is resident (host-checked), so
// this terminates; a 4 s bound turns a broken invariant into a trap instead of a hang.
__device__ __forceinline__ void wait_counter(const uint32_t* p, uint32_t target) {
  if (ld_acquire_u32(p) >= target) return;
  const unsigned long long t0 = ar_globaltimer();
  while (ld_acquire_u32(p) < target) {
    if (ar_globaltimer() - t0 > 4000000000ull) __trap();
    __nanosleep(64);
  }
}

struct FuseArgs {
  const __nv_bfloat16* q_nope;   // [B, H, DH] raw queries
  const __nv_bfloat16* q_rope;   // [B, H, DR] raw rotary queries
  const __nv_bfloat16* w_uk;     // [H, DH, NB*DLAT] (K1 pack)
  const __nv_bfloat16* w_uv;     // [H, NB*DLAT, DH] (K3 pack)
  __nv_bfloat16* q_abs;          // [B, NB, H, DLAT] out of the absorb phase (workspace)
  __nv_bfloat16* q_rope_s;       // [B, H, DR] scaled rotary queries (workspace)
  float* out;                    // [B, H, DH]
  float* ybuf;                   // [nchunks, B, H, DH] per-chunk up-projections (workspace)
  uint32_t* sync;                // fuse_sync_words(...) words, zero before the first launch
  int* status;                   // numeric status word (or null)
  TpSum tp;                      // world > 1: rank sum fused into the final tiles
  float score_scale, alpha;
  int DH, NB, DLAT, hgroups, npad;
  int absorb;                    // 1: run the absorb phase (else q_abs / q_rope_s are inputs)
  int combine;                   // 1: run the combine phase (else the partials are the output)
  int debug_reps;                // dev: each combine unit runs this many times (1)
  int debug_producer_wait;       // dev: the TMA producer waits for the absorbed queries
};

// ----------------------------------------------------------------------------- absorb phase
// Unit u = (16-sequence group G, head h, 64-column block cb of the NB*DLAT absorbed columns).
// The W^UK tile [DH][64] (128-byte rows, 16-byte units XOR-swizzled by row) and the queries
// [16][DH] are staged by cp.async into the CTA's query / P buffers (unused until the absorbed
// queries exist), then 8 warps x 8 columns run mma.sync m16n8k16 (ldmatrix / ldmatrix.trans
// operands, fp32 accumulation). Columns past NB*DLAT are skipped.
__host__ __device__ inline int absorb_units(int B, int H, int NB, int DLAT) {
  return fuse_groups(B) * H * ((NB * DLAT + 63) / 64);
}
__host__ __device__ inline size_t absorb_smem_bytes(int DH) { return size_t(DH) * 128 + size_t(16) * (DH + 8) * 2; }

__device__ __forceinline__ void fused_absorb(const FuseArgs& f, int B, int H, int DR, int cta, int ncta, int stid,
                                             uint8_t* stage) {
  const int warp = stid >> 5, lane = stid & 31, g = lane >> 2, t4 = lane & 3, lq = lane >> 3;
  const int NCOL = f.NB * f.DLAT, NCB = (NCOL + 63) / 64, DH = f.DH;
  const int nunits = absorb_units(B, H, f.NB, f.DLAT);
  const uint32_t wbase = smem_u32(stage), abase = wbase + uint32_t(DH) * 128;
  const int arow = (DH + 8) * 2;
  for (int u = cta; u < nunits; u += ncta) {
    const int cb = u % NCB, h = (u / NCB) % H, G = u / (NCB * H);
    // W^UK[h][k][cb*64 .. +64) -> row k, unit q ^ (k & 7); queries [16][DH] (rows past B zero)
    for (int i = stid; i < DH * 8; i += 256) {
      const int r = i >> 3, q = i & 7, col = cb * 64 + q * 8;
      const bool ok = col < NCOL;
      cp_async16(wbase + uint32_t(r * 128 + ((q ^ (r & 7)) * 16)),
                 ok ? static_cast<const void*>(f.w_uk + (size_t(h) * DH + r) * NCOL + col) : static_cast<const void*>(f.w_uk),
                 ok ? 16u : 0u);
    }
    const int units = DH / 8;
    for (int i = stid; i < 16 * units; i += 256) {
      const int r = i / units, q = i % units, s = G * kFuseSeqs + r;
      const bool ok = s < B;
      cp_async16(abase + uint32_t(r * arow + q * 16),
                 ok ? static_cast<const void*>(f.q_nope + (size_t(s) * H + h) * DH + q * 8) : static_cast<const void*>(f.q_nope),
                 ok ? 16u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    cp_async_wait_all();
    named_bar_sync(1, 256);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int kb = 0; kb < DH; kb += 16) {
      uint32_t a[4], bfr[2];
      ldmatrix_x4(a, abase + uint32_t(((lane & 7) + (lq & 1) * 8) * arow + (kb + (lq >> 1) * 8) * 2));
      const int k = kb + (lane & 7) + (lq & 1) * 8;
      ldmatrix_x2_trans(bfr, wbase + uint32_t(k * 128 + ((warp ^ (k & 7)) * 16)));
      mma_m16n8k16_bf16(acc, a, bfr[0], bfr[1]);
    }
    const int col = cb * 64 + warp * 8 + 2 * t4;
    if (col < NCOL) {
      const int bb = col / f.DLAT, cc = col % f.DLAT;  // DLAT even: the pair stays in one branch
      const int s0 = G * kFuseSeqs + g, s1 = s0 + 8;
      if (s0 < B)
        *reinterpret_cast<uint32_t*>(f.q_abs + ((size_t(s0) * f.NB + bb) * H + h) * f.DLAT + cc) =
            pack_bf16(acc[0] * f.score_scale, acc[1] * f.score_scale);
      if (s1 < B)
        *reinterpret_cast<uint32_t*>(f.q_abs + ((size_t(s1) * f.NB + bb) * H + h) * f.DLAT + cc) =
            pack_bf16(acc[2] * f.score_scale, acc[3] * f.score_scale);
    }
    if (cb == 0) {
      for (int i = stid; i < kFuseSeqs * DR; i += 256) {
        const int s = G * kFuseSeqs + i / DR;
        if (s < B) {
          const size_t off = (size_t(s) * H + h) * DR + i % DR;
          f.q_rope_s[off] = __float2bfloat16(__bfloat162float(f.q_rope[off]) * f.score_scale);
        }
      }
    }
    named_bar_sync(1, 256);  // staging reuse by the next unit; every store of the unit issued
  }
  if (stid == 0 && cta < nunits)  // one cumulative release for the CTA's units
    red_release_add(f.sync + kSyncAbsorb, uint32_t((nunits - 1 - cta) / ncta + 1));
}

// ----------------------------------------------------------------------------- combine phase
// Unit u = (16-sequence group G, head h, latent chunk j of CW = min(DLAT, 128) columns of one
// branch). Per unit: cp.async W^UV rows of the chunk into smem (row-XOR swizzled) while waiting
// for the group's sequences; split weights per sequence; merged latent Z [16][CW]; y = Z . W on
// mma.sync (Z as bf16 hi + lo: ~16-bit mantissa, fp32 sums); then either the head's output
// (one chunk per head) or a per-chunk partial plus a ticket: the unit drawing the head's last
// ticket adds the chunks in ascending order (ascending branch order, decode.py:264-285) and
// applies alpha. The TP sum over ranks runs on that final tile.
__host__ __device__ inline int combine_chunk_width(int DLAT) { return DLAT < 128 ? DLAT : 128; }
__host__ __device__ inline int combine_units(int B, int H, int NB, int DLAT) {
  return fuse_groups(B) * H * (NB * DLAT / combine_chunk_width(DLAT));
}
__host__ __device__ inline size_t combine_smem_bytes(int DH, int DLAT) {
  const int CW = combine_chunk_width(DLAT);
  return size_t(CW) * DH * 2 + size_t(kFuseSeqs) * CW * 4 + size_t(kFuseSeqs) * DH * 4 +
         size_t(kFuseSeqs) * kFuseMaxSplits * 4 + 64;
}

__device__ __forceinline__ void fused_combine(const FuseArgs& f, const float* __restrict__ o_part,
                                           const float* __restrict__ lse_part, int B, int H, int nsplit,
                                           uint8_t* sm, int cta, int ncta, int stid, uint32_t tp_epoch,
                                           long long* trace = nullptr) {
  // dev trace (MLRA_DEBUG_TRACE_PTR): phase stamps of the traced CTA's first unit
  auto stamp = [&](int k) {
    if (trace != nullptr && stid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
      trace[16384 + 8 * 160 + k] = (long long)t;
      trace[16384 + 8 * 160 + 8 + k] = clock64();
    }
  };
  const int DH = f.DH, DLAT = f.DLAT, NB = f.NB;
  const int CW = combine_chunk_width(DLAT), NCH = NB * DLAT / CW;
  const int nunits = combine_units(B, H, NB, DLAT);
  const int nG = fuse_groups(B);
  // smem carve-up (the K2 ring is free: every MMA of this CTA has completed)
  __nv_bfloat16* wsm = reinterpret_cast<__nv_bfloat16*>(sm);             // [CW][DH] swizzled
  float* zs = reinterpret_cast<float*>(sm + size_t(CW) * DH * 2);          // [CW][16]
  float* ys = zs + CW * kFuseSeqs;                                          // [16][DH]
  float* wts = ys + kFuseSeqs * DH;                                         // [16][kFuseMaxSplits]
  int* s_flag = reinterpret_cast<int*>(wts + kFuseSeqs * kFuseMaxSplits);  // [0] this unit holds the final tile
  const int warp = stid >> 5, lane = stid & 31;
  const uint32_t wbase = smem_u32(wsm);
  const int upr = DH / 8;  // 16-byte units per W row
  for (int ui = cta * f.debug_reps; ui < nunits * f.debug_reps; ui += ncta * f.debug_reps) {
   for (int rep = 0; rep < f.debug_reps; ++rep) {
    const int u = ui / f.debug_reps;
    const int j = u % NCH, h = (u / NCH) % H, G = u / (NCH * H);
    const int b = (j * CW) / DLAT, c0 = (j * CW) % DLAT;
    const int hg = h / f.npad;
    stamp(5);
    // 1. W^UV rows [b*DLAT + c0, +CW) of head h -> smem, 16-byte units XOR-swizzled by row
    {
      const __nv_bfloat16* src = f.w_uv + (size_t(h) * NB * DLAT + b * DLAT + c0) * DH;
      for (int i = stid; i < CW * upr; i += 256) {
        const int r = i / upr, q = i % upr;
        cp_async16(wbase + uint32_t(r * DH * 2 + ((q ^ (r & 7)) * 16)), src + size_t(r) * DH + q * 8, 16u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // 2. wait for every sequence of the group (all its splits' partials written)
    if (stid < kFuseSeqs) {
      const int s = G * kFuseSeqs + stid;
      if (s < B) wait_counter(f.sync + kSyncSeq + size_t(s) * f.hgroups + hg, uint32_t(nsplit));
    }
    named_bar_sync(1, 256);
    stamp(0);
    // 3. split weights w_k = 2^(lse_k - max) / sum: warp w handles sequences w and w + 8
    for (int sq = warp; sq < kFuseSeqs; sq += 8) {
      const int s = G * kFuseSeqs + sq;
      float lk[kFuseMaxSplits / 32];
      float m = -INFINITY;
      bool nan = false;
#pragma unroll
      for (int i = 0; i < kFuseMaxSplits / 32; ++i) {
        const int k = lane + 32 * i;
        lk[i] = (s < B && k < nsplit) ? __ldcg(lse_part + (size_t(s) * nsplit * NB + b) * H + h + size_t(k) * NB * H)
                                      : -INFINITY;
        nan |= lk[i] != lk[i];
        m = fmaxf(m, lk[i]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      const bool any_nan = __any_sync(0xffffffffu, nan);
      if (s < B && lane == 0 && f.status != nullptr && (any_nan || m == -INFINITY))
        atomicOr(f.status, (any_nan ? kStatusNaN : 0) | (m == -INFINITY ? kStatusNoFinite : 0));
      float tot = 0.f;
#pragma unroll
      for (int i = 0; i < kFuseMaxSplits / 32; ++i) {
        lk[i] = (m == -INFINITY || lk[i] == -INFINITY) ? 0.f : ex2(lk[i] - m);
        tot += lk[i];
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
      const float inv = tot > 0.f ? 1.f / tot : 0.f;
#pragma unroll
      for (int i = 0; i < kFuseMaxSplits / 32; ++i)
        if (lane + 32 * i < nsplit) wts[sq * kFuseMaxSplits + lane + 32 * i] = lk[i] * inv;
    }
    named_bar_sync(1, 256);
    stamp(1);
    // 4. merged latent Z[c][s] = sum_k w[s][k] O_k[s][b][h][c0 + c]. Item = (sequence, 4 latent
    //    columns): one float4 load per split. tpi threads (adjacent lanes) share an item's splits
    //    (many splits, few sequences: B = 1 runs 148) and meet through shuffles; a thread keeps up
    //    to two items x 10 splits of loads in flight (one L2 round trip at B = 16, 9 splits).
    {
      const int nreal = min(kFuseSeqs, B - G * kFuseSeqs);
      const int nc4 = CW / 4, nitems = nreal * nc4;
      int tpi = 1;
      while (tpi < 32 && nitems * tpi * 2 <= 256) tpi *= 2;
      const int slice = stid % tpi, it0 = stid / tpi, it1 = it0 + 256 / tpi;
      const size_t kstride = size_t(NB) * H * DLAT;
      const bool ok0 = it0 < nitems, ok1 = it1 < nitems;
      const int sq0 = ok0 ? it0 / nc4 : 0, sq1 = ok1 ? it1 / nc4 : 0;
      const float* o0 = o_part + ((size_t(G * kFuseSeqs + sq0) * nsplit * NB + b) * H + h) * DLAT + c0 + (it0 % nc4) * 4;
      const float* o1 = o_part + ((size_t(G * kFuseSeqs + sq1) * nsplit * NB + b) * H + h) * DLAT + c0 + (it1 % nc4) * 4;
      float4 z0 = make_float4(0.f, 0.f, 0.f, 0.f), z1 = z0;
      constexpr int KB = 10;
      for (int kb = slice; kb < nsplit; kb += KB * tpi) {
        float4 v0[KB], v1[KB];
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          const int k = kb + q * tpi;
          v0[q] = (ok0 && k < nsplit) ? __ldcg(reinterpret_cast<const float4*>(o0 + size_t(k) * kstride)) : z0;
          v1[q] = (ok1 && k < nsplit) ? __ldcg(reinterpret_cast<const float4*>(o1 + size_t(k) * kstride))
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          const int k = kb + q * tpi;
          if (k < nsplit) {
            const float w0 = wts[sq0 * kFuseMaxSplits + k], w1 = wts[sq1 * kFuseMaxSplits + k];
            z0.x = fmaf(w0, v0[q].x, z0.x); z0.y = fmaf(w0, v0[q].y, z0.y);
            z0.z = fmaf(w0, v0[q].z, z0.z); z0.w = fmaf(w0, v0[q].w, z0.w);
            z1.x = fmaf(w1, v1[q].x, z1.x); z1.y = fmaf(w1, v1[q].y, z1.y);
            z1.z = fmaf(w1, v1[q].z, z1.z); z1.w = fmaf(w1, v1[q].w, z1.w);
          }
        }
      }
      for (int o = 1; o < tpi; o <<= 1) {
        z0.x += __shfl_xor_sync(0xffffffffu, z0.x, o); z0.y += __shfl_xor_sync(0xffffffffu, z0.y, o);
        z0.z += __shfl_xor_sync(0xffffffffu, z0.z, o); z0.w += __shfl_xor_sync(0xffffffffu, z0.w, o);
        z1.x += __shfl_xor_sync(0xffffffffu, z1.x, o); z1.y += __shfl_xor_sync(0xffffffffu, z1.y, o);
        z1.z += __shfl_xor_sync(0xffffffffu, z1.z, o); z1.w += __shfl_xor_sync(0xffffffffu, z1.w, o);
      }
      // padding sequences of the group contribute zero rows to the up-projection
      for (int i = stid; i < CW * kFuseSeqs; i += 256)
        if (i % kFuseSeqs >= nreal) zs[i] = 0.f;
      if (slice == 0) {
        if (ok0) {
          const int c = (it0 % nc4) * 4;
          zs[(c + 0) * kFuseSeqs + sq0] = z0.x; zs[(c + 1) * kFuseSeqs + sq0] = z0.y;
          zs[(c + 2) * kFuseSeqs + sq0] = z0.z; zs[(c + 3) * kFuseSeqs + sq0] = z0.w;
        }
        if (ok1) {
          const int c = (it1 % nc4) * 4;
          zs[(c + 0) * kFuseSeqs + sq1] = z1.x; zs[(c + 1) * kFuseSeqs + sq1] = z1.y;
          zs[(c + 2) * kFuseSeqs + sq1] = z1.z; zs[(c + 3) * kFuseSeqs + sq1] = z1.w;
        }
      }
    }
    cp_async_wait_all();
    named_bar_sync(1, 256);
    stamp(2);
    // 5. y[s][d] = sum_c Z[s][c] W[c][d]: warp w owns 16-column blocks w, w + 8, ...
    {
      const int g = lane >> 2, t4 = lane & 3, q = lane >> 3;
      for (int nb16 = warp; nb16 < DH / 16; nb16 += 8) {
        float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        for (int kb = 0; kb < CW; kb += 16) {
          uint32_t ahi[4], alo[4];
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {  // rows g, g + 8
              const int k = kb + 2 * t4 + 8 * hf;
              const float z0 = zs[k * kFuseSeqs + g + 8 * rr], z1 = zs[(k + 1) * kFuseSeqs + g + 8 * rr];
              const __nv_bfloat16 h0 = __float2bfloat16_rn(z0), h1 = __float2bfloat16_rn(z1);
              ahi[2 * hf + rr] = pack_bf16_raw(h0, h1);
              alo[2 * hf + rr] = pack_bf16(z0 - __bfloat162float(h0), z1 - __bfloat162float(h1));
            }
          }
          uint32_t bfr[4];
          const int k = kb + (q & 1) * 8 + (lane & 7);
          ldmatrix_x4_trans(bfr, wbase + uint32_t(k * DH * 2 + (((nb16 * 2 + (q >> 1)) ^ (k & 7)) * 16)));
          mma_m16n8k16_bf16(acc[0], ahi, bfr[0], bfr[1]);
          mma_m16n8k16_bf16(acc[0], alo, bfr[0], bfr[1]);
          mma_m16n8k16_bf16(acc[1], ahi, bfr[2], bfr[3]);
          mma_m16n8k16_bf16(acc[1], alo, bfr[2], bfr[3]);
        }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int col = nb16 * 16 + jj * 8 + 2 * t4;
          ys[g * DH + col] = acc[jj][0];
          ys[g * DH + col + 1] = acc[jj][1];
          ys[(g + 8) * DH + col] = acc[jj][2];
          ys[(g + 8) * DH + col + 1] = acc[jj][3];
        }
      }
    }
    named_bar_sync(1, 256);
    stamp(3);
    // 6. single chunk: ys is the head's output; else publish the chunk and take a ticket
    bool final_tile = true;
    if (NCH > 1) {
      for (int i = stid; i < kFuseSeqs * DH; i += 256) {
        const int s = G * kFuseSeqs + i / DH;
        if (s < B) f.ybuf[((size_t(j) * B + s) * H + h) * DH + i % DH] = ys[i];
      }
      named_bar_sync(1, 256);
      if (stid == 0) {
        const uint32_t t = atom_acq_rel_add(f.sync + kSyncSeq + size_t(B) * f.hgroups + size_t(G) * H + h, 1u);
        s_flag[0] = (t == uint32_t(NCH - 1)) ? 1 : 0;
      }
      named_bar_sync(1, 256);
      final_tile = s_flag[0] != 0;
      if (final_tile) {  // thread 0's acquire + the barrier order the other chunks' stores before these loads
        for (int i = stid; i < kFuseSeqs * DH; i += 256) {
          const int s = G * kFuseSeqs + i / DH;
          float tot = 0.f;
          if (s < B)
            for (int jj = 0; jj < NCH; ++jj) tot += __ldcg(f.ybuf + ((size_t(jj) * B + s) * H + h) * DH + i % DH);
          ys[i] = tot;
        }
        named_bar_sync(1, 256);
      }
    }
    if (final_tile) {
      if (f.tp.world <= 1) {
        for (int i = stid; i < kFuseSeqs * DH; i += 256) {
          const int s = G * kFuseSeqs + i / DH;
          if (s < B) f.out[(size_t(s) * H + h) * DH + i % DH] = ys[i] * f.alpha;
        }
      } else {
        // one-shot sum over the TP ranks (the K5 protocol): tile -> slot [parity][my rank] of
        // every rank, release the epoch into that rank's flag for this tile, wait for the world
        // flags of this tile in my region, add in ascending rank order (bit-identical on all ranks)
        const TpSum& tp = f.tp;
        const int W = tp.world;
        const size_t tp_n = size_t(B) * H * DH, tp_ns = ar_stride(int(tp_n));
        const uint32_t epoch = tp_epoch;
        const int par = int(epoch & 1u), slot = G * H + h;
        for (int r = 0; r < W; ++r) {
          float* dst = tp.comm[r] + (size_t(par) * W + tp.rank) * tp_ns;
          for (int i = stid; i < kFuseSeqs * DH; i += 256) {
            const int s = G * kFuseSeqs + i / DH;
            if (s < B) dst[(size_t(s) * H + h) * DH + i % DH] = ys[i] * f.alpha;
          }
        }
        named_bar_sync(1, 256);
        if (stid < W) {
          __threadfence_system();
          uint32_t* flags = reinterpret_cast<uint32_t*>(tp.comm[stid] + ar_recv_floats(int(tp_n), W));
          ar_st_release_sys(flags + (size_t(par) * W + tp.rank) * kArFlagSlots + slot, epoch);
          const uint32_t* fl = reinterpret_cast<const uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) +
                               (size_t(par) * W + stid) * kArFlagSlots + slot;
          const unsigned long long t0 = ar_globaltimer();
          while (ar_ld_acquire_sys(fl) != epoch) {
            if (ar_globaltimer() - t0 > 4000000000ull) __trap();
            __nanosleep(32);
          }
        }
        named_bar_sync(1, 256);
        const float* recv = tp.comm[tp.rank] + size_t(par) * W * tp_ns;
        for (int i = stid; i < kFuseSeqs * DH; i += 256) {
          const int s = G * kFuseSeqs + i / DH;
          if (s >= B) continue;
          const size_t o = (size_t(s) * H + h) * DH + i % DH;
          float sum = 0.f;
          for (int r = 0; r < W; ++r) sum += __ldcv(recv + size_t(r) * tp_ns + o);
          f.out[o] = sum;
        }
        if (stid == 0) {  // advance the rank's epoch once every final tile of the call has read it
          uint32_t* ctr = reinterpret_cast<uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) + ar_flag_words(W);
          __threadfence();
          if (atomicAdd(ctr + 1, 1u) == uint32_t(nG * H) - 1u) {
            ctr[1] = 0u;
            atomicExch(ctr, epoch);
          }
        }
      }
    }
    named_bar_sync(1, 256);  // smem reuse by the next unit
    stamp(4);
   }
  }
}


// ============================================================================= cluster step
// One-branch-per-device steps (an MLRA-4 TP rank, an MLA TP rank: NB = 1, one head group) with
// the nsplit split CTAs of a sequence launched as ONE thread-block cluster (nsplit <= 16):
// K1 and K3 run inside the cluster, their hand-offs go through distributed shared memory
// instead of global memory round trips.
//   prologue: CTA `rank` absorbs the query rows r = rank, rank + nsplit, ... of its sequence
//     (q~_r = q_nope_r . W^UK_r, FMA with coalesced W^UK rows; padding rows zero) and stores
//     them, with the scaled rotary query, straight into the K-major SW128 query chunks of EVERY
//     CTA of the cluster (st.shared::cluster); cluster barrier. The TMA producer streams
//     meanwhile (it only arrives at the barrier).
//   epilogue: every CTA keeps its split's normalised latent mixture O [NPAD][DLAT] and
//     log2-sum-exp [NPAD] in its (now idle) ring; cluster barrier; CTA `rank` merges the
//     splits of its heads over DSMEM (split weights 2^(lse_k - max) / sum, ascending k),
//     up-projects with the W^UV rows it prefetched before the barrier (FMA) and writes
//     out[seq][h] (or runs the TP sum); cluster barrier before exit (DSMEM stays alive).
// Reference: attnkit/decode.py:155-167, :217-230, :264-285; tpsim.py:275-276.

__device__ __forceinline__ void st_shared_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__host__ __device__ inline int cluster_heads_per_cta(int H, int nsplit) { return (H + nsplit - 1) / nsplit; }
// ring bytes the cluster epilogue needs: O [npad][dlat] + lse [npad] + W^UV of the CTA's heads +
// merged Z [dlat] + split weights [16] + up-projection halves [2][DH] + y [heads][DH]
__host__ __device__ inline size_t cluster_epilogue_bytes(int npad, int dlat, int dh, int heads) {
  return size_t(npad) * dlat * 4 + size_t(npad) * 4 + 64 + size_t(heads) * dlat * dh * 2 + size_t(dlat) * 4 + 64 +
         size_t(2) * dh * 4 + size_t(heads) * dh * 4 + 256;
}

// K-major SW128 query chunk address of (row r, column col) in a CTA's q buffer
__device__ __forceinline__ uint32_t q_chunk_addr(uint32_t q_base, int chunk_bytes, int r, int col) {
  const int chunk = col >> 6, u = (col & 63) >> 3;
  return q_base + uint32_t(chunk * chunk_bytes + r * 128 + ((u ^ (r & 7)) * 16) + (col & 7) * 2);
}

// Prologue: rows r = rank, rank + nsplit, ... < npad of sequence seq (softmax warps, stid 0..255).
// red: 256 floats of scratch (the P buffer).
__device__ __forceinline__ void cluster_absorb(const FuseArgs& f, int H, int DR, int DLAT, int npad, int seq,
                                               int rank, int nsplit, uint32_t q_base, int chunk_bytes, int nlat_chunks,
                                               float* red, int stid) {
  const int DH = f.DH;
  const int c = stid & 127, kh = stid >> 7, kh_len = DH / 2, k0 = kh * kh_len;
  const int lane = stid & 31;
  float* qrow = red + 256;  // the query row, fp32
  for (int r = rank; r < npad; r += nsplit) {
    const bool real = r < H;
    const __nv_bfloat16* w = f.w_uk + size_t(r) * DH * DLAT;
    if (stid < DH) qrow[stid] = real ? __bfloat162float(f.q_nope[(size_t(seq) * H + r) * DH + stid]) : 0.f;
    named_bar_sync(1, 256);
    for (int c0 = 0; c0 < DLAT; c0 += 128) {
      float acc = 0.f;
      if (real && c0 + c < DLAT) {
        const __nv_bfloat16* wc = w + c0 + c;
#pragma unroll 32
        for (int k = k0; k < k0 + kh_len; ++k) acc = fmaf(qrow[k], __bfloat162float(__ldg(wc + size_t(k) * DLAT)), acc);
      }
      red[stid] = acc;
      named_bar_sync(1, 256);
      if (kh == 0) {
        const float v = (acc + red[stid + 128]) * f.score_scale;
        const float vn = __shfl_down_sync(0xffffffffu, v, 1);
        if ((lane & 1) == 0 && c0 + c < DLAT) {
          const uint32_t packed = pack_bf16(v, vn);  // zero for padding rows (acc = 0)
          const uint32_t addr = q_chunk_addr(q_base, chunk_bytes, r, c0 + c);
          for (int k = 0; k < nsplit; ++k) st_shared_cluster_u32(mapa_shared(addr, uint32_t(k)), packed);
        }
      }
      named_bar_sync(1, 256);
    }
    // rotary chunk: scaled q_rope (zero past DR and for padding rows)
    if (stid < 32) {
      const int d = 2 * stid;
      float v0 = 0.f, v1 = 0.f;
      if (real && d < DR) {
        const __nv_bfloat16* qr = f.q_rope + (size_t(seq) * H + r) * DR;
        v0 = __bfloat162float(qr[d]) * f.score_scale;
        v1 = (d + 1 < DR) ? __bfloat162float(qr[d + 1]) * f.score_scale : 0.f;
      }
      const uint32_t addr = q_chunk_addr(q_base, chunk_bytes, r, nlat_chunks * 64 + d);
      const uint32_t packed = pack_bf16(v0, v1);
      for (int k = 0; k < nsplit; ++k) st_shared_cluster_u32(mapa_shared(addr, uint32_t(k)), packed);
    }
  }
}

// Epilogue, after the CTA wrote its O / lse into cm (ring) and the cluster barrier: merge and
// up-project this CTA's heads of sequence seq. wbuf: the W^UV rows of those heads (prefetched).
__device__ __forceinline__ void cluster_combine(const FuseArgs& f, int B, int H, int DLAT, int npad, int seq, int rank,
                                                int nsplit, const float* cm_o, const float* cm_lse,
                                                const __nv_bfloat16* wbuf, float* zsm, float* wts, float* ysum,
                                                float* ysm, int stid, uint32_t tp_epoch) {
  const int DH = f.DH, lane = stid & 31;
  int i = 0;
  for (int h = rank; h < H; h += nsplit, ++i) {
    // split weights (warp 0): lane k < nsplit reads split k's lse over DSMEM
    if (stid < 32) {
      const float lk = lane < nsplit ? ld_shared_cluster_f32(mapa_shared(smem_u32(cm_lse + h), uint32_t(lane))) : -INFINITY;
      const bool nan = lk != lk;
      float m = lk;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      const bool any_nan = __any_sync(0xffffffffu, nan);
      if (lane == 0 && f.status != nullptr && (any_nan || m == -INFINITY))
        atomicOr(f.status, (any_nan ? kStatusNaN : 0) | (m == -INFINITY ? kStatusNoFinite : 0));
      float wk = (m == -INFINITY || lk == -INFINITY || lane >= nsplit) ? 0.f : ex2(lk - m);
      float tot = wk;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
      if (lane < nsplit) wts[lane] = tot > 0.f ? wk / tot : 0.f;
    }
    named_bar_sync(1, 256);
    // merged latent Z[c] = sum_k w_k O_k[h][c] (every split's DSMEM load in flight together)
    for (int cc = stid; cc < DLAT; cc += 256) {
      const uint32_t a = smem_u32(cm_o + size_t(h) * DLAT + cc);
      float v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = k < nsplit ? ld_shared_cluster_f32(mapa_shared(a, uint32_t(k))) : 0.f;
      float z = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < nsplit) z = fmaf(wts[k], v[k], z);
      zsm[cc] = z;
    }
    named_bar_sync(1, 256);
    // y[d] = alpha * sum_c Z[c] W[c][d]: thread (d, half of c)
    {
      const __nv_bfloat16* wi = wbuf + size_t(i) * DLAT * DH;
      const int nh = 256 / DH;  // parts of the contraction per column (DH <= 256)
      const int d = stid % DH, part = stid / DH, clen = DLAT / nh;
      float acc = 0.f;
      if (part < nh) {
#pragma unroll 8
        for (int cc = part * clen; cc < (part + 1) * clen; ++cc) acc = fmaf(zsm[cc], __bfloat162float(wi[size_t(cc) * DH + d]), acc);
      }
      if (part < nh) ysum[part * DH + d] = acc;
      named_bar_sync(1, 256);
      if (stid < DH) {
        float y = 0.f;
        for (int q = 0; q < nh; ++q) y += ysum[q * DH + stid];
        ysm[i * DH + stid] = y * f.alpha;
      }
      named_bar_sync(1, 256);
    }
  }
  const int nheads = i;
  if (f.tp.world <= 1) {
    for (int j = stid; j < nheads * DH; j += 256)
      f.out[(size_t(seq) * H + rank + (j / DH) * nsplit) * DH + j % DH] = ysm[j];
    return;
  }
  // one-shot sum over the TP ranks (the K5 protocol) on this CTA's heads of sequence seq
  const TpSum& tp = f.tp;
  const int W = tp.world;
  const size_t tp_n = size_t(B) * H * DH, tp_ns = ar_stride(int(tp_n));
  const uint32_t epoch = tp_epoch;
  const int par = int(epoch & 1u), slot = seq * nsplit + rank;
  for (int r = 0; r < W; ++r) {
    float* dst = tp.comm[r] + (size_t(par) * W + tp.rank) * tp_ns;
    for (int j = stid; j < nheads * DH; j += 256)
      dst[(size_t(seq) * H + rank + (j / DH) * nsplit) * DH + j % DH] = ysm[j];
  }
  named_bar_sync(1, 256);
  if (stid < W) {
    __threadfence_system();
    uint32_t* flags = reinterpret_cast<uint32_t*>(tp.comm[stid] + ar_recv_floats(int(tp_n), W));
    ar_st_release_sys(flags + (size_t(par) * W + tp.rank) * kArFlagSlots + slot, epoch);
    const uint32_t* fl = reinterpret_cast<const uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) +
                         (size_t(par) * W + stid) * kArFlagSlots + slot;
    const unsigned long long t0 = ar_globaltimer();
    while (ar_ld_acquire_sys(fl) != epoch) {
      if (ar_globaltimer() - t0 > 4000000000ull) __trap();
      __nanosleep(32);
    }
  }
  named_bar_sync(1, 256);
  const float* recv = tp.comm[tp.rank] + size_t(par) * W * tp_ns;
  for (int j = stid; j < nheads * DH; j += 256) {
    const size_t o = (size_t(seq) * H + rank + (j / DH) * nsplit) * DH + j % DH;
    float sum = 0.f;
    for (int r = 0; r < W; ++r) sum += __ldcv(recv + size_t(r) * tp_ns + o);
    f.out[o] = sum;
  }
  if (stid == 0) {  // advance the rank's epoch once every CTA of the call has read it
    uint32_t* ctr = reinterpret_cast<uint32_t*>(tp.comm[tp.rank] + ar_recv_floats(int(tp_n), W)) + ar_flag_words(W);
    if (atom_acq_rel_add(ctr + 1, 1u) == uint32_t(B * nsplit) - 1u) {
      ctr[1] = 0u;
      atomicExch(ctr, epoch);
    }
  }
}

}  // namespace mlra
