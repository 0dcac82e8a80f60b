// K2: split-KV flash-decode over the paged latent cache, tcgen05 tensor cores + TMA.
//
// Replaces the hot loop of attnkit/decode.py:217-230 (attend_local, latent branch):
//   logits_b = tau * (q~_b . C_b^T + q_rope . K_rope^T);  P = softmax;  Z_b = P . C_b
// for every branch b a GPU owns, over the token tiles [t0, t0+ntiles) of one sequence,
// and emits per-split partials (Z normalised by its own softmax sum, plus log2-sum-exp)
// that K3 (aux_kernels.cuh, combine_kernel) merges and up-projects.
//
// Swap-AB formulation: the MMA M dimension is the KV tile (tokens for QK^T, latent rows
// for PV), N is the (padded) head group. One TMEM lane = one token (S) or one latent row
// (O). Per round (tile, branch):
//   MMA  : S = KV . Q_b^T                      (K-major A = the TMA tile, K-major B = Q_b)
//   soft : scores shifted by the running max; one bar.red.or vote asks whether any score
//          exceeded it by more than 2^8 (lazy rescale). Only then is the exact per-head
//          tile max taken (redux.sync.max.f32 + smem across the 4 lane quarters) and O_b
//          rescaled in TMEM. P = exp2(S - m) goes to smem as bf16; the softmax
//          denominators accumulate in registers (one partial per token lane).
//   MMA  : O_b += C_b^T . P                     (MN-major A = the same smem tile as V)
// The same smem tile serves as K and as V: V = the latent columns of K (FlashMLA's trick).
//
// Pool row layout (width W): [branch 0 latent | ... | branch NB-1 latent | rope]; each
// branch latent = SUB sub-blocks of DLS columns (MLA: SUB = 4).
//
// Warp roles (352 threads): warp 0 = TMA producer, warp 1 = TMEM owner + QK issuer,
// warps 2..9 = softmax / rescale / epilogue in two groups of four (one warp per TMEM lane
// quarter each; the groups split the heads of every round), warp 10 = PV issuer. QK and PV
// are issued by different warps so that neither waits behind the other's dependencies
// (a QK waiting for its tile no longer holds back the PV that frees a ring slot).
// With NB > 1 branches per tile the rope logits (identical in every branch, Eq. 5) are
// computed once per tile into their own TMEM slot and added by the softmax warps.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cmath>
#include "ptx.cuh"
#include "fused_step.cuh"

namespace mlra {

struct DecodeParams {
  const __nv_bfloat16* q_abs;   // [B, NB, H, DLAT] absorbed queries, pre-scaled by tau*log2(e)
  const __nv_bfloat16* q_rope;  // [B, H, DR]       rotary queries, pre-scaled by tau*log2(e)
  const int32_t* block_table;   // [B, max_pages]
  const int32_t* seqlens;       // [B]
  float* o_part;                // [B, nsplit, NB, H, DLAT]  Z / l per split
  float* lse_part;              // [B, nsplit, NB, H]        m + log2(l) per split (log2 domain)
  int B, H, SUB, DR, W;         // W = NB*SUB*DLS + DR (pool row width, elements)
  int page_size, max_pages, nsplit;
  int lat_slots, rope_slots;    // ring depths (set by the host from the smem budget)
  int p_slots;                  // P buffers (1 or 2)
  int box_rows;                 // token rows per TMA box: T when pages hold whole tiles, else 64
  float rescale_threshold;      // lazy-rescale threshold (log2 units)
  long long* trace;             // debug: per-round clock64 events of CTA `trace_cta`, or null
  int trace_cta;                // debug: linear CTA index traced (x fastest)
  // ---- GQA comparison variant (template GQA = true) ------------------------------------------
  // Pool row [K_0 | ... | K_{G-1} | V_0 | ... | V_{G-1}] (each DLS wide, post-RoPE keys), no
  // rope part (DR = 0). "Branch" = KV head: blockIdx.z selects NB of the nb_total KV heads,
  // H = query heads per KV head. q_abs holds the unscaled queries [B, nb_total, H, DLS]; the
  // score scale tau*log2(e) is applied in fp32 by the softmax (qk_scale).
  int nb_total;
  float qk_scale;
  int pdl;                      // host side: launch with programmatic stream serialization
  const int32_t* plan;          // ragged-batch work items [gridDim.x][4] (mlra_decode_plan), or null
  int plan_ctas;                // host side: gridDim.x with a plan
  int late_trigger;             // release the dependent launch (K3) at the epilogue, not at the start
  // ---- fused step (fused_step.cuh): K1 in the prologue, K3 (+ TP sum) in the epilogue -------
  int fused;                    // 0: partials only (K1 / K3 run as separate kernels)
  int hgroups;                  // head groups (gridDim.z) -- completion-counter stride
  FuseArgs fz;
};

// The single-launch / cluster step experiments (fused_step.cuh, opt-in, measured slower) are
// compiled into K2 only with -DMLRA_K2_FUSED_STEP: their branches cost the product kernel.
#ifdef MLRA_K2_FUSED_STEP
constexpr bool kK2FusedBuild = true;
#else
constexpr bool kK2FusedBuild = false;
#endif

constexpr int kNumThreads = 352;  // TMA warp, QK warp, 2 x 4 softmax warps, PV warp
constexpr int kPvWarp = 10;
constexpr int kSoftThreads = 256;

constexpr float kRescaleThreshold = 8.0f;  // P stays <= 2^8 between rescales
constexpr int kMaxLat = 16, kMaxRope = 8;

template <int T, int NPAD, int DLS>
struct DecodeLayout {
  static constexpr int kChunkBytes = T * 128;                 // [T rows x 64 cols] bf16, 128B swizzle
  static constexpr int kLatBytes = (DLS / 64) * kChunkBytes;  // one sub-block
  static constexpr int kRopeBytes = kChunkBytes;              // rope <= 64 cols
  static constexpr int kQChunkBytes = NPAD * 128;
  static constexpr int kPBytes = T * NPAD * 2;
  static constexpr int kPSbo = (T / 8) * 128;                 // MN-group stride of the P operand
  // red[2][4][NPAD] + aw[8][NPAD] + m_run[8][4][NPAD]; the epilogue's lred[4][4][NPAD] and
  // invl[4][NPAD] alias the P buffer (dead once the last PV has completed)
  static constexpr int kScratchFloats = 8 * NPAD + 8 * NPAD + 32 * NPAD;
  static_assert(20 * NPAD * 4 <= kPBytes, "epilogue scratch must fit in one P buffer");
  static constexpr int kBarOff = ((kScratchFloats * 4 + 127) / 128) * 128;
  static constexpr int kNumBars = 2 * kMaxLat + 2 * kMaxRope + 8 + 4 + 1 + 2;
  static constexpr int kScratchBytes = kBarOff + kNumBars * 8 + 16;  // + tmem base, debug word, TP epoch
  static int smem_bytes(int NB, int SUB, int lat_slots, int rope_slots, int p_slots) {
    const int q_chunks = NB * SUB * (DLS / 64) + 1;
    return lat_slots * kLatBytes + rope_slots * kRopeBytes + q_chunks * kQChunkBytes + p_slots * kPBytes +
           kScratchBytes;
  }
};

__device__ __forceinline__ bool is_trace_cta(int trace_cta) {
  return int((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) == trace_cta;
}

__device__ __forceinline__ void trace_event(long long* trace, int trace_cta, int ev, int r) {
  // events: 0 TMA issue of unit r, 1 QK(r) issue, 2 PV(r) issue, 3 S(r) seen, 4 P(r) done,
  //         5 MMA iteration r done, 6 QK(r) data ready (lat_full observed)
  //         (softmax sub-phases) 7 S in registers, 8 vote done, 9 P slot free, 10 P stored
  if (trace != nullptr && r < 256 && is_trace_cta(trace_cta))
    trace[(ev < 7 ? ev * 256 : 12032 + (ev - 7) * 256) + r] = clock64();
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
  return t;
}

__device__ __forceinline__ float warp_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

template <int T, int NPAD, int DLS, int NB, bool GQA = false>
__global__ void __launch_bounds__(kNumThreads, 1)
    mlra_decode_kernel(const __grid_constant__ CUtensorMap lat_map, const __grid_constant__ CUtensorMap rope_map,
                       const DecodeParams p) {
  using L = DecodeLayout<T, NPAD, DLS>;
  static_assert(T == 64 || T == 128, "token tile must be 64 or 128");
  static_assert(DLS == 64 || DLS == 128, "sub-block width must be 64 or 128");
  static_assert(NPAD == 16 || NPAD == 32 || NPAD == 64, "head group must be 16, 32 or 64");
  static_assert(NB >= 1 && NB <= 4, "1..4 branches per device");
  constexpr int kHG = NPAD / 2;  // heads (TMEM columns) per softmax group

  const int SUB = GQA ? 1 : p.SUB;
  const int DLAT = SUB * DLS;
  // Work item: uniform grid (split, sequence) -- or, with a ragged-batch plan (mlra_decode_plan),
  // item blockIdx.x of the plan: {sequence, split slot, first tile, tile count}; surplus CTAs
  // (sequence < 0) leave at once.
  int4 item = make_int4(int(blockIdx.y), int(blockIdx.x), 0, -1);
  if (p.plan != nullptr) {
    item = __ldg(reinterpret_cast<const int4*>(p.plan) + blockIdx.x);
    if (item.x < 0) return;
  }
  const int seq = item.x, split = item.y;
  // MLRA/MLA: blockIdx.z = head group; GQA: blockIdx.z = group of NB KV heads (all its heads)
  const int hg = GQA ? 0 : blockIdx.z;
  const int branch0 = GQA ? blockIdx.z * NB : 0;  // first branch of this CTA in the q/partials layout
  const int nbq = GQA ? p.nb_total : NB;           // branches in the q_abs / o_part / lse layouts
  const int len = p.seqlens[seq];
  const int ntiles_total = (len + T - 1) / T;
  const int per = (ntiles_total + p.nsplit - 1) / p.nsplit;
  const int t0 = p.plan != nullptr ? min(item.z, ntiles_total) : min(split * per, ntiles_total);
  const int ntiles = p.plan != nullptr ? max(0, min(item.w, ntiles_total - t0)) : min(per, ntiles_total - t0);
  const int R = ntiles * NB;  // rounds: (tile, branch)
  const int n_valid_pages = (len + p.page_size - 1) / p.page_size;
  const int HV = min(NPAD, p.H - hg * NPAD);  // real heads in this head group

  // ------------------------------------------------------------- shared memory carve-up
  // (no static __shared__: the dynamic window starts 1024-aligned, and every pointer below
  //  is derived from smem by pointer arithmetic so accesses stay in the shared state space)
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* lat_ring = smem;
  uint8_t* rope_ring = lat_ring + p.lat_slots * L::kLatBytes;
  uint8_t* q_smem = rope_ring + p.rope_slots * L::kRopeBytes;
  const int q_chunks = NB * SUB * (DLS / 64) + 1;
  uint8_t* p_smem = q_smem + q_chunks * L::kQChunkBytes;
  uint8_t* scratch = p_smem + p.p_slots * L::kPBytes;
  float* red = reinterpret_cast<float*>(scratch);  // [2][4][NPAD] per-quarter tile maxima
  float* aw = red + 8 * NPAD;                      // [8][NPAD] per-softmax-warp rescale factor
  float* m_run = aw + 8 * NPAD;                    // [8][4][NPAD] per-softmax-warp running max per branch
  float* lred = reinterpret_cast<float*>(p_smem);  // [4][4][NPAD] per-quarter softmax sums (epilogue)
  float* invl = lred + 16 * NPAD;                  // [4][NPAD]
  uint64_t* bars = reinterpret_cast<uint64_t*>(scratch + L::kBarOff);
  uint64_t* lat_full = bars;
  uint64_t* lat_empty = lat_full + kMaxLat;
  uint64_t* rope_full = lat_empty + kMaxLat;
  uint64_t* rope_empty = rope_full + kMaxRope;
  uint64_t* s_full = rope_empty + kMaxRope;  // [2]
  uint64_t* s_empty = s_full + 2;            // [2]
  uint64_t* p_full = s_empty + 2;            // [2]
  uint64_t* p_empty = p_full + 2;            // [2]
  uint64_t* o_done = p_empty + 2;            // [4]
  uint64_t* o_final = o_done + 4;
  uint64_t* sr_empty = o_final + 1;          // [2] shared rope logits slot consumed (NB > 1)
  uint32_t* tmem_base_sh = reinterpret_cast<uint32_t*>(sr_empty + 2);

  const int tid = threadIdx.x, warp = tid / 32, lane = lane_id();
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (!p.late_trigger) griddep_launch_dependents();  // a dependent launch may start its prologue
  if (kK2FusedBuild && p.fused == 2) cluster_arrive_relaxed();  // cluster step, phase 0: this CTA has started
  if (p.trace != nullptr && tid == 0 && cta_lin < 1024) {
    p.trace[7 * 256 + 2 * cta_lin] = (long long)global_ns();
    p.trace[13824 + 2 * cta_lin] = clock64();
  }
  // TMEM columns: S slots [0, 2*NPAD); (NB > 1) rope-logit slots [2*NPAD, 4*NPAD);
  // O_{b,s} at O_COL + (b*SUB+s)*NPAD
  constexpr uint32_t kTmemCols = 512;
  constexpr bool kSharedRope = NB > 1 && !GQA;
  const uint32_t S_COL = 0, SR_COL = 2 * NPAD, O_COL = (kSharedRope ? 4 : 2) * NPAD;

  if (tid == 0) {  // the producer's first TMA needs both descriptors: fetch them first
    tma_prefetch_desc(&lat_map);
    tma_prefetch_desc(&rope_map);
  }
  if (tid == 32) {  // barrier init off the producer warp: it overlaps the page-id loads
    for (int i = 0; i < p.lat_slots; ++i) { mbar_init(&lat_full[i], 1); mbar_init(&lat_empty[i], 1); }
    for (int i = 0; i < p.rope_slots; ++i) { mbar_init(&rope_full[i], 1); mbar_init(&rope_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1); mbar_init(&s_empty[i], kSoftThreads);
      mbar_init(&p_full[i], kSoftThreads); mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&o_done[i], 1);
    mbar_init(o_final, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&sr_empty[i], kSoftThreads);
    tmem_base_sh[1] = 0;  // debug-trace check of the final CTA barrier
    fence_barrier_init();
  }
  // The TMA producer (warp 0) fetches its first page ids while warp 1 initialises the
  // mbarriers; it waits for them (named barrier 7 with warp 1) only before its first mbarrier
  // use, and never for the TMEM allocation or the consumers' setup (barrier 6, warps 1-10).
  if (warp != 0) {
    if (warp == 1) {
      __syncwarp();
      named_bar_arrive(7, 64);
      tmem_alloc<kTmemCols>(tmem_base_sh);
    }
    for (int i = tid - 32; i < 32 * NPAD; i += kNumThreads - 32) m_run[i] = 0.f;  // set exactly on tile 0
    fence_proxy_async_smem();
    tc_fence_before();
    named_bar_sync(6, kNumThreads - 32);
    tc_fence_after();
  }
  const uint32_t tbase = warp == 0 ? 0u : *tmem_base_sh;
  const int ncta = gridDim.x * gridDim.y * gridDim.z;
  const bool cm = kK2FusedBuild && p.fused == 2;  // cluster step (fused_step.cuh): the split CTAs of a sequence are one cluster
  if (warp != 0) {
    if (cm) {
      cluster_wait_acquire();  // phase 0: every CTA of the cluster runs (its shared memory may be written)
      if (warp >= 2 && warp < 2 + kSoftThreads / 32)
        cluster_absorb(p.fz, p.H, p.DR, DLAT, NPAD, seq, split, p.nsplit, smem_u32(q_smem), L::kQChunkBytes,
                       NB * SUB * (DLS / 64), reinterpret_cast<float*>(p_smem), tid - 64);
      if (tid == 64 && p.fz.tp.world > 1)  // this call's TP epoch (advanced after every CTA read it)
        tmem_base_sh[2] = *reinterpret_cast<volatile uint32_t*>(
                              reinterpret_cast<uint32_t*>(p.fz.tp.comm[p.fz.tp.rank] +
                                                          ar_recv_floats(p.B * p.H * p.fz.DH, p.fz.tp.world)) +
                              ar_flag_words(p.fz.tp.world)) + 1u;
      cluster_arrive_release();  // phase A: the cluster's absorbed query rows are in every q buffer
      cluster_wait_acquire();
      fence_proxy_async_smem();  // generic-proxy (DSMEM) stores -> visible to the tensor-core reads
    } else if (kK2FusedBuild && p.fused) {
      // Fused step: the softmax warps run this CTA's share of the absorb units (K1) while the
      // producer streams; every consumer then waits for the grid's absorbed queries.
      if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 0] = (long long)global_ns();
      if (p.fz.absorb) {
        if (warp >= 2 && warp < 2 + kSoftThreads / 32)
          fused_absorb(p.fz, p.B, p.H, p.DR, cta_lin, ncta, tid - 64, q_smem);  // stages in q / P buffers
        if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 1] = (long long)global_ns();
        if (tid == 64) wait_counter(p.fz.sync + kSyncAbsorb, uint32_t(absorb_units(p.B, p.H, p.fz.NB, p.fz.DLAT)));
        if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 2] = (long long)global_ns();
      }
      if (tid == 64 && p.fz.tp.world > 1)  // this call's TP epoch (advanced after every final tile read it)
        tmem_base_sh[2] = *reinterpret_cast<volatile uint32_t*>(
                              reinterpret_cast<uint32_t*>(p.fz.tp.comm[p.fz.tp.rank] +
                                                          ar_recv_floats(p.B * p.H * p.fz.DH, p.fz.tp.world)) +
                              ar_flag_words(p.fz.tp.world)) + 1u;
      named_bar_sync(5, kNumThreads - 32);
    } else {
      // Under PDL this kernel overlaps K1's tail: the TMA producer is already streaming the
      // cache (written before K1 started); the queries are K1's output.
      griddep_wait();
    }
    // ---- absorbed + rotary queries of this (sequence, head group) -> K-major SW128 chunks.
    //      Chunk (b, c) holds latent columns [c*64, c*64+64) of branch b; the last is rope.
    //      (cluster step: already written by the cluster's absorb)
    if (!cm) {
      const int nlat_chunks = NB * SUB * (DLS / 64);
      const int total = q_chunks * NPAD * 8;  // 16-byte units
      for (int idx = tid - 32; idx < total; idx += kNumThreads - 32) {
        const int chunk = idx / (NPAD * 8);
        const int rem = idx % (NPAD * 8);
        const int r = rem / 8, u = rem % 8;
        const int h = hg * NPAD + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (h < p.H) {
          if (chunk < nlat_chunks) {
            const int b = chunk / (DLAT / 64), c = chunk % (DLAT / 64);
            v = __ldcg(reinterpret_cast<const uint4*>(p.q_abs + ((size_t(seq) * nbq + branch0 + b) * p.H + h) * DLAT + c * 64 +
                                                      u * 8));
          } else if (u * 8 < p.DR) {
            v = __ldcg(reinterpret_cast<const uint4*>(p.q_rope + (size_t(seq) * p.H + h) * p.DR + u * 8));
          }
        }
        *reinterpret_cast<uint4*>(q_smem + chunk * L::kQChunkBytes + r * 128 + ((u ^ (r & 7)) * 16)) = v;
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    named_bar_sync(2, kNumThreads - 32);
    tc_fence_after();
  }

  if (warp == 0) {
    // ============================================================ TMA producer (whole warp)
    // lat_map: 3-D view {64 cols, rows, latent chunk} of the pool, so one box brings a whole
    // DLS-wide sub-block of a T-token tile; rope_map: 2-D {64 cols, box_rows rows} view.
    // The page ids of the next 32/nbox tiles are fetched by the 32 lanes in one round trip
    // (no dependent block-table load per tile), then lane 0 issues the boxes.
    if (lane == 0) trace_event(p.trace, p.trace_cta, 11, 0);  // producer start (len known below)
    if (R == 0) {
      named_bar_sync(7, 64);
      if (cm) { cluster_wait_acquire(); cluster_arrive_relaxed(); }  // phase 0 done; phase A: nothing to publish
    }
    if (kK2FusedBuild && p.fused && p.fz.debug_producer_wait && lane == 0)  // dev: no streaming until q~ is ready
      wait_counter(p.fz.sync + kSyncAbsorb, uint32_t(absorb_units(p.B, p.H, p.fz.NB, p.fz.DLAT)));
    __syncwarp();
    if (R > 0) {
      const uint64_t policy = l2_policy_evict_first();
      const int rope_col = NB * DLAT;
      const int nbox = T / p.box_rows;
      const int box_bytes = p.box_rows * 128;
      const int tiles_per_fetch = 32 / nbox;
      int lslot = 0, lphase = 0, my_row = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int tf = t % tiles_per_fetch;
        if (tf == 0) {
          const int tt = t + lane / nbox;
          my_row = 0;
          if (tt < ntiles) {
            const int tok0 = (t0 + tt) * T + p.box_rows * (lane % nbox);
            const int page = min(tok0 / p.page_size, n_valid_pages - 1);
            my_row = __ldg(p.block_table + size_t(seq) * p.max_pages + page) * p.page_size + (tok0 % p.page_size);
          }
        }
        int rows[T / 64];
#pragma unroll
        for (int i = 0; i < T / 64; ++i) rows[i] = __shfl_sync(0xffffffffu, my_row, tf * nbox + (i < nbox ? i : 0));
        if (t == 0) {
          if (lane == 0) trace_event(p.trace, p.trace_cta, 11, 1);  // page ids of the first tiles in
          named_bar_sync(7, 64);  // mbarriers initialised by warp 1
          if (cm) { cluster_wait_acquire(); cluster_arrive_relaxed(); }  // phase 0 done; phase A: nothing to publish
          if (lane == 0) trace_event(p.trace, p.trace_cta, 11, 2);
        }
        if (!GQA) {
          const int slot = t % p.rope_slots;
          mbar_wait(&rope_empty[slot], ((t / p.rope_slots) & 1) ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&rope_full[slot], L::kRopeBytes);
            for (int i = 0; i < nbox; ++i)
              tma_load_2d_hint(&rope_map, &rope_full[slot], rope_ring + slot * L::kRopeBytes + i * box_bytes, rope_col,
                               rows[i], policy);
            if (t == 0) trace_event(p.trace, p.trace_cta, 11, 3);
          }
        }
        // units of the tile: MLRA/MLA the NB*SUB latent sub-blocks; GQA K_b then V_b per KV head
        for (int u = 0; u < (GQA ? 2 * NB : NB * SUB); ++u) {
          const int ch0 = GQA ? ((u & 1) ? p.nb_total + branch0 + (u >> 1) : branch0 + (u >> 1)) * (DLS / 64)
                              : u * (DLS / 64);  // first 64-column chunk of the unit in the row
          mbar_wait(&lat_empty[lslot], lphase ^ 1);
          if (lane == 0) {
            mbar_arrive_expect_tx(&lat_full[lslot], L::kLatBytes);
            uint8_t* dst = lat_ring + lslot * L::kLatBytes;
            if (nbox == 1) {
              // one box = [DLS/64 chunks][T rows][128 B]: exactly the chunk-major smem layout
              tma_load_3d_hint(&lat_map, &lat_full[lslot], dst, 0, rows[0], ch0, policy);
            } else {
              // pages of 64 tokens: per chunk, per 64-row page box (2-D view)
              for (int c = 0; c < DLS / 64; ++c)
                for (int i = 0; i < nbox; ++i)
                  tma_load_2d_hint(&rope_map, &lat_full[lslot], dst + c * L::kChunkBytes + i * box_bytes,
                                   (ch0 + c) * 64, rows[i], policy);
            }
            trace_event(p.trace, p.trace_cta, 0, t * NB * SUB + u);
          }
          __syncwarp();
          if (++lslot == p.lat_slots) { lslot = 0; lphase ^= 1; }
        }
      }
    }
  } else if (warp == 1 || warp == kPvWarp) {
    // ============================================================ MMA issuers (one warp each, elected lane)
    // Warp 1 issues every QK in round order; QK(r) needs its tile and the S slot freed by
    // softmax(r-2), so it runs up to two rounds ahead of the softmax. Warp 10 issues every
    // PV(r) as soon as P(r) is ready. Each warp runs its loop converged (descriptors in
    // uniform registers); elect.sync picks the issuing lane. tcgen05.commit tracks the
    // issuing thread's own MMAs: QK(r) is complete before P(r) exists, so the PV warp's
    // commit after PV(r) is a valid release of the latent slot both used.
    if (R > 0) {
      // descriptor templates (start address 0); per use: + (smem byte address >> 4)
      const uint64_t kdesc_sw128 = make_sdesc(0, 16, 1024, kSw128);              // K-major, 128B swizzle
      const uint64_t vdesc_sw128 = make_sdesc(0, L::kChunkBytes, 1024, kSw128);  // MN-major V (LBO = chunk)
      const uint64_t pdesc = make_sdesc(0, 128, L::kPSbo, kSwNone);               // MN-major P, interleaved
      const uint32_t lat_base = smem_u32(lat_ring), rope_base = smem_u32(rope_ring);
      const uint32_t q_base = smem_u32(q_smem), p_base = smem_u32(p_smem);
      if (warp == 1) {
        constexpr uint32_t idesc_qk = make_idesc_bf16(T, NPAD, false, false);
        const int kq_rope = (p.DR + 15) / 16;
        const uint32_t q_rope_addr = q_base + (NB * SUB * (DLS / 64)) * L::kQChunkBytes;
        int lslot = 0, lphase = 0;
        for (int t = 0; t < ntiles; ++t) {
          const int rslot = GQA ? 0 : t % p.rope_slots;
          const uint64_t ra0 = kdesc_sw128 + ((rope_base + rslot * L::kRopeBytes) >> 4);
          const uint64_t rb0 = kdesc_sw128 + (q_rope_addr >> 4);
          if (lane == 0) trace_event(p.trace, p.trace_cta, 12, t * NB);
          if (!GQA) mbar_wait(&rope_full[rslot], (t / p.rope_slots) & 1);
          if constexpr (kSharedRope) {
            // rope logits of the tile, once for all branches
            mbar_wait(&sr_empty[t & 1], ((t >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tbase + SR_COL + (t & 1) * NPAD;
            for (int kk = 0; kk < kq_rope; ++kk) mma_bf16_ss_w(d, ra0 + kk * 2, rb0 + kk * 2, idesc_qk, kk > 0 ? 1u : 0u);
            mma_commit_w(&rope_empty[rslot]);
          }
#pragma unroll 1
          for (int b = 0; b < NB; ++b) {
            const int r = t * NB + b;
            const int sslot = r & 1;
            mbar_wait(&s_empty[sslot], ((r >> 1) & 1) ^ 1);
            if (lane == 0) trace_event(p.trace, p.trace_cta, 13, r);
            const uint32_t d = tbase + S_COL + sslot * NPAD;
            uint32_t acc = 0;
            for (int s = 0; s < SUB; ++s) {
              mbar_wait(&lat_full[lslot], lphase);
              if (lane == 0 && s == 0) trace_event(p.trace, p.trace_cta, 6, r);
              tc_fence_after();
              const uint64_t a0 = kdesc_sw128 + ((lat_base + lslot * L::kLatBytes) >> 4);
              const uint64_t b0 = kdesc_sw128 + ((q_base + (b * SUB + s) * (DLS / 64) * L::kQChunkBytes) >> 4);
#pragma unroll
              for (int c = 0; c < DLS / 64; ++c)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  mma_bf16_ss_w(d, a0 + ((c * L::kChunkBytes + kk * 32) >> 4),
                                b0 + ((c * L::kQChunkBytes + kk * 32) >> 4), idesc_qk, acc);
                  acc = 1;
                }
              if constexpr (GQA) {
                // K_b is QK's alone: release it here; then step over V_b (the PV warp's)
                mma_commit_w(&lat_empty[lslot]);
                if (++lslot == p.lat_slots) { lslot = 0; lphase ^= 1; }
              }
              if (++lslot == p.lat_slots) { lslot = 0; lphase ^= 1; }
            }
            if (lane == 0) trace_event(p.trace, p.trace_cta, 1, r);
            if constexpr (GQA) {
              mma_commit_w(&s_full[sslot]);
            } else if constexpr (!kSharedRope) {
              for (int kk = 0; kk < kq_rope; ++kk) mma_bf16_ss_w(d, ra0 + kk * 2, rb0 + kk * 2, idesc_qk, 1);
              mma_commit_w(&s_full[sslot]);
              mma_commit_w(&rope_empty[rslot]);
            } else {
              mma_commit_w(&s_full[sslot]);  // also covers the tile's rope logits (issued earlier)
            }
          }
        }
      } else {
        constexpr uint32_t idesc_pv = make_idesc_bf16(DLS, NPAD, true, true);
        int lslot = 0, lphase = 0;
        for (int t = 0; t < ntiles; ++t) {
#pragma unroll 1
          for (int b = 0; b < NB; ++b) {
            const int r = t * NB + b;
            const int pslot = r % p.p_slots;
            if constexpr (GQA) {
              // step over K_b (the QK warp's) to V_b, and wait for V_b itself
              if (++lslot == p.lat_slots) { lslot = 0; lphase ^= 1; }
              mbar_wait(&lat_full[lslot], lphase);
            }
            mbar_wait(&p_full[pslot], (r / p.p_slots) & 1);
            if (lane == 0) trace_event(p.trace, p.trace_cta, 2, r);
            tc_fence_after();
            const uint64_t pb = pdesc + ((p_base + pslot * L::kPBytes) >> 4);
            const uint32_t acc0 = t > 0 ? 1u : 0u;
            for (int s = 0; s < SUB; ++s) {
              const uint64_t a0 = vdesc_sw128 + ((lat_base + lslot * L::kLatBytes) >> 4);
              const uint32_t d = tbase + O_COL + (b * SUB + s) * NPAD;
#pragma unroll
              for (int k = 0; k < T / 16; ++k)
                mma_bf16_ss_w(d, a0 + k * (2048 >> 4), pb + k * (256 >> 4), idesc_pv, acc0 | k);
              mma_commit_w(&lat_empty[lslot]);
              if (++lslot == p.lat_slots) { lslot = 0; lphase ^= 1; }
            }
            mma_commit_w(&p_empty[pslot]);
            mma_commit_w(&o_done[b]);
            if (lane == 0) trace_event(p.trace, p.trace_cta, 5, r);
          }
        }
        // Single-phase barrier for the epilogue: o_done[b] may lag by two phases there, which
        // a parity wait cannot disambiguate.
        mma_commit_w(o_final);
      }
    }
  } else {
    // ============================================================ softmax / rescale / epilogue
    // Two groups of 4 warps (one warp per TMEM lane quarter each) split every round's heads:
    // group g owns heads [h_lo, h_lo + h_cnt) with h_lo in {0, NPAD/2} (tcgen05.ld/st column
    // addresses stay aligned to the access width).
    // Fast path per round: scores are shifted by the running max m_run (smem); one bar.red.or
    // across both groups asks "did any score exceed m_run + threshold?". Only then (first
    // tile of the split, or a large jump) does the slow path compute the exact tile max per
    // head and rescale this group's O_b columns and softmax sums.
    const int ws = warp - 2;  // softmax warp slot 0..7
    const int grp = ws >> 2;
    const int q = warp & 3;   // TMEM lane quarter owned by this warp
    const int h_lo = grp * kHG;
    const int h_cnt = max(0, min(kHG, HV - h_lo));
    const bool lane_ok = (T == 128) || (lane < 16);
    const int tok_in_tile = (T == 128) ? q * 32 + lane : q * 16 + lane;
    const uint32_t lane_off = uint32_t(q * 32) << 16;
    const float thr = p.rescale_threshold;
    // P row of this thread's token: (tok, h) at (h/8)*SBO + (tok/8)*128 + (tok%8)*16 + (h%8)*2
    uint8_t* const prow0 = p_smem + (tok_in_tile / 8) * 128 + (tok_in_tile % 8) * 16;
    float lsum[NB][kHG];  // per-token-lane softmax-sum partials, reduced once in the epilogue
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int c = 0; c < kHG; ++c) lsum[bb][c] = 0.f;

    for (int t = 0; t < ntiles; ++t) {
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int r = t * NB + b;
        const int sslot = r & 1;
        mbar_wait(&s_full[sslot], (r >> 1) & 1);
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 3, r);
        tc_fence_after();
        float s[kHG];
        {
          uint32_t raw[kHG];
          const uint32_t taddr = tbase + lane_off + S_COL + sslot * NPAD + h_lo;
          if constexpr (kHG == 8) {
            tmem_ld8(taddr, raw);
          } else {
#pragma unroll
            for (int c = 0; c < kHG; c += 16) tmem_ld16(taddr + c, raw + c);
          }
          if constexpr (kSharedRope) {
            // + the tile's rope logits (complete: s_full of this round covers them)
            uint32_t rr[kHG];
            const uint32_t raddr = tbase + lane_off + SR_COL + (t & 1) * NPAD + h_lo;
            if constexpr (kHG == 8) {
              tmem_ld8(raddr, rr);
            } else {
#pragma unroll
              for (int c = 0; c < kHG; c += 16) tmem_ld16(raddr + c, rr + c);
            }
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kHG; ++c) s[c] = __uint_as_float(raw[c]) + __uint_as_float(rr[c]);
          } else if constexpr (GQA) {
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kHG; ++c) s[c] = __uint_as_float(raw[c]) * p.qk_scale;
          } else {
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kHG; ++c) s[c] = __uint_as_float(raw[c]);
          }
        }
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 7, r);
        tc_fence_before();
        mbar_arrive(&s_empty[sslot]);
        if (kSharedRope && b == NB - 1) mbar_arrive(&sr_empty[t & 1]);
        if ((t0 + t + 1) * T > len || !lane_ok) {  // partial tile / unused M=64 lanes
          const int tok = (t0 + t) * T + tok_in_tile;
          if (!(lane_ok && tok < len)) {
#pragma unroll
            for (int c = 0; c < kHG; ++c) s[c] = -INFINITY;
          }
        }
        float* mrun = m_run + (ws * 4 + b) * NPAD + h_lo;  // this warp's copy (branch b, own heads)
        float dmax = -INFINITY;
#pragma unroll
        for (int c = 0; c < kHG; c += 4) {
          const float4 m4 = *reinterpret_cast<const float4*>(mrun + c);
          s[c + 0] -= m4.x;
          s[c + 1] -= m4.y;
          s[c + 2] -= m4.z;
          s[c + 3] -= m4.w;
          const float mx = fmaxf(fmaxf(s[c + 0], s[c + 1]), fmaxf(s[c + 2], s[c + 3]));
          dmax = (c < h_cnt) ? fmaxf(dmax, mx) : dmax;
        }
        // m_run is finite (0 before the first tile), so masked lanes stay at -inf. Head groups of
        // <= 16 heads per thread (NPAD <= 32) take the exact-max path on the first tile: measured
        // K2 TP1 B=16 32K 105.8 -> 102.3 us, TP4 rank 35.8 -> 35.3 us against the vote
        // (profiles/r3_k2_first_tile.md). At 64 heads (32 per thread) the
        // tile keeps the reference max 0 unless a score could overflow P (> 2^thr) or a head's
        // scores could underflow it (< 2^-64): the exact-max slow path (warp + quarter maxima,
        // a second barrier) is then taken only when needed -- it cost a CTA's first round ~2K
        // cycles. (per group: the groups own disjoint heads, so their decisions are independent)
        bool vote = dmax > thr;
        if constexpr (NPAD <= 32) {
          if (t == 0) vote = true;
        } else if (t == 0) {
          float dmin = INFINITY;
#pragma unroll
          for (int c = 0; c < kHG; ++c)
            if (c < h_cnt && s[c] != -INFINITY) dmin = fminf(dmin, s[c]);
          vote = vote || dmin < -64.f;
        }
        const bool slow = named_bar_or(3 + grp, kSoftThreads / 2, vote);
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 8, r);
        bool rescale = false;
        if (slow) {
          // exact tile max per head: warp max, then across the 4 quarters through smem
#pragma unroll
          for (int c = 0; c < kHG; ++c) s[c] += mrun[c];  // back to raw scores (old m_run)
          float wm[kHG];
#pragma unroll
          for (int c = 0; c < kHG; ++c) wm[c] = (c < h_cnt) ? warp_max(s[c]) : -INFINITY;
          float* red_r = red + (r & 1) * 4 * NPAD + h_lo;
          if (lane == 0) {
#pragma unroll
            for (int c = 0; c < kHG; c += 4)
              *reinterpret_cast<float4*>(red_r + q * NPAD + c) = make_float4(wm[c], wm[c + 1], wm[c + 2], wm[c + 3]);
          }
          named_bar_sync(3 + grp, kSoftThreads / 2);
          if (lane < h_cnt) {
            const float m_tile =
                fmaxf(fmaxf(red_r[lane], red_r[NPAD + lane]), fmaxf(red_r[2 * NPAD + lane], red_r[3 * NPAD + lane]));
            const float m_old = mrun[lane];
            const float m_new = (t == 0) ? m_tile : fmaxf(m_old, m_tile);
            aw[ws * NPAD + h_lo + lane] = (t == 0) ? 0.f : ex2(m_old - m_new);
            mrun[lane] = m_new;
          }
          __syncwarp();
#pragma unroll
          for (int c = 0; c < kHG; ++c) {
            s[c] -= mrun[c];
            lsum[b][c] *= aw[ws * NPAD + h_lo + c];
          }
          rescale = t > 0;
        }
        // ---- probabilities (log2 domain; the score scale is folded into the queries)
        const int pslot = r % p.p_slots;
        if (r >= p.p_slots) mbar_wait(&p_empty[pslot], ((r / p.p_slots) - 1) & 1);
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 9, r);
        if (lane_ok) {
          uint8_t* prow = prow0 + pslot * L::kPBytes;
#pragma unroll
          for (int c = 0; c < kHG; c += 8) {
            if (c < h_cnt) {
              const int h = h_lo + c;  // 8-aligned: one 16-byte core-matrix row
              float e[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                e[j] = ex2(s[c + j]);
                lsum[b][c + j] += e[j];
              }
              uint4 v;
              v.x = pack_bf16(e[0], e[1]);
              v.y = pack_bf16(e[2], e[3]);
              v.z = pack_bf16(e[4], e[5]);
              v.w = pack_bf16(e[6], e[7]);
              *reinterpret_cast<uint4*>(prow + (h >> 3) * L::kPSbo) = v;
            }
          }
        }
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 10, r);
        // ---- rare: the running max moved -> rescale this group's O_b columns
        if (rescale) {
          // PV(t-2, b) is complete (it was issued before QK(t, b), whose S we consumed), so
          // o_done[b] lags phase t-1 by at most one phase and the parity wait is exact.
          mbar_wait(&o_done[b], (t - 1) & 1);
          tc_fence_after();
          for (int sb = 0; sb < SUB; ++sb) {
            const uint32_t taddr = tbase + lane_off + h_lo + O_COL + (b * SUB + sb) * NPAD;
            uint32_t raw[kHG];
            if constexpr (kHG == 8) {
              tmem_ld8(taddr, raw);
            } else {
#pragma unroll
              for (int c = 0; c < kHG; c += 16) tmem_ld16(taddr + c, raw + c);
            }
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < kHG; ++c)
              raw[c] = __float_as_uint(__uint_as_float(raw[c]) * aw[ws * NPAD + h_lo + c]);
#pragma unroll
            for (int c = 0; c < kHG; c += 8) tmem_st8(taddr + c, raw + c);
          }
          tmem_st_wait();
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[pslot]);
        if (ws == 0 && lane == 0) trace_event(p.trace, p.trace_cta, 4, r);
      }
    }

    // ============================================================ epilogue: partials
    // (late trigger: the merge kernel may launch once every CTA has reached this point -- its
    // launch and W^UV staging overlap the epilogues)
    if (p.late_trigger) griddep_launch_dependents();
    // softmax sums: reduce this warp's 32 token lanes for all NB*kHG (branch, head) values at
    // once by recursive halving (a lane keeps one half and receives the partner's other half:
    // V/2 + V/4 + ... shuffles instead of 5*V), then the 4 quarters in smem.
    constexpr int V = NB * kHG;
    float vals[V];
    int base = 0;  // original index of vals[0] on this lane
    {
#pragma unroll
      for (int i = 0; i < V; ++i) vals[i] = lsum[i / kHG][i % kHG];
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int o = 16 >> k;
        const int live = V >> k;
        if (live >= 2) {
          const int half = live / 2;
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const float send = up ? vals[i] : vals[i + half];
            const float keep = up ? vals[i + half] : vals[i];
            vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
          base += up ? half : 0;
        } else {
          vals[0] += __shfl_xor_sync(0xffffffffu, vals[0], o);
        }
      }
    }
    if (p.trace != nullptr && tid == 64 && cta_lin < 1024 && true) p.trace[7 * 256 + 2048 + 8 * cta_lin + 3] = clock64();
    if (ntiles > 0) {
      mbar_wait(o_final, 0);  // every PV done: the P buffer (lred/invl) and TMEM O are final
      tc_fence_after();
    }
    // cluster step: O / lse of this split stay in the (now idle) ring for the cluster's merge; the
    // W^UV rows of this CTA's heads are prefetched meanwhile
    const int cm_heads = cm ? cluster_heads_per_cta(p.H, p.nsplit) : 0;
    float* cm_o = reinterpret_cast<float*>(smem);                   // [NPAD][DLAT]
    float* cm_lse = cm_o + NPAD * DLAT;                               // [NPAD]
    __nv_bfloat16* cm_w = reinterpret_cast<__nv_bfloat16*>(cm_lse + ((NPAD + 15) / 16) * 16);  // [heads][DLAT][DH]
    float* cm_z = reinterpret_cast<float*>(cm_w + size_t(cm_heads) * DLAT * p.fz.DH);           // [DLAT]
    float* cm_wts = cm_z + DLAT;                                      // [16]
    float* cm_ysum = cm_wts + 16;                                     // [256]
    float* cm_y = cm_ysum + 256;                                      // [heads][DH]
    if (cm) {
      const int DH = p.fz.DH, per_head = DLAT * DH / 8;  // 16-byte chunks per head's W^UV rows
      const uint32_t wb = smem_u32(cm_w);
      for (int i = tid - 64; i < cm_heads * per_head; i += kSoftThreads) {
        const int hi = i / per_head, ch = i % per_head, h = split + hi * p.nsplit;
        if (h < p.H)
          cp_async16(wb + uint32_t(i) * 16, p.fz.w_uv + size_t(h) * DLAT * DH + size_t(ch) * 8, 16u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    {
      constexpr int kLive = (V >> 5) >= 1 ? (V >> 5) : 1;
#pragma unroll
      for (int i = 0; i < kLive; ++i) {
        const int idx = base + i;
        lred[((idx / kHG) * 4 + q) * NPAD + h_lo + idx % kHG] = vals[i];
      }
    }
    named_bar_sync(1, kSoftThreads);
    if (p.trace != nullptr && tid == 64 && cta_lin < 1024 && true) p.trace[7 * 256 + 2048 + 8 * cta_lin + 4] = clock64();
    const size_t part_row0 = (size_t(seq) * p.nsplit + split) * nbq + branch0;  // (seq, split, b) row index
    if (q == 0 && lane < h_cnt) {
      const int h = h_lo + lane;
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        const float lt = lred[(bb * 4 + 0) * NPAD + h] + lred[(bb * 4 + 1) * NPAD + h] +
                         lred[(bb * 4 + 2) * NPAD + h] + lred[(bb * 4 + 3) * NPAD + h];
        const float m = m_run[(ws * 4 + bb) * NPAD + h];
        invl[bb * NPAD + h] = lt > 0.f ? 1.f / lt : 0.f;
        // empty split (no tile, or every probability 0) -> -inf; a NaN logit leaves lt = NaN and
        // the NaN is passed on so the merge can flag it (attnkit/tensors.py:74-75)
        const float lse = lt > 0.f ? m + log2f(lt) : (lt == 0.f ? -INFINITY : __int_as_float(0x7fc00000));
        if (cm) cm_lse[h] = lse;
        else p.lse_part[(part_row0 + bb) * p.H + hg * NPAD + h] = lse;
      }
    }
    named_bar_sync(1, kSoftThreads);
    const bool row_ok = (DLS == 128) || (lane < 16);
    const int row = (DLS == 128) ? q * 32 + lane : q * 16 + lane;
    if constexpr (NB > 1) {
      // one sub-block per branch (SUB = 1): every branch's TMEM load in flight, one wait
      uint32_t raw[NB][kHG];
      if (ntiles > 0) {
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          const uint32_t taddr = tbase + lane_off + O_COL + bb * NPAD + h_lo;
          if constexpr (kHG == 8) {
            tmem_ld8(taddr, raw[bb]);
          } else {
#pragma unroll
            for (int c = 0; c < kHG; c += 16) tmem_ld16(taddr + c, raw[bb] + c);
          }
        }
        tmem_ld_wait();
      }
      if (row_ok) {
#pragma unroll
        for (int bb = 0; bb < NB; ++bb) {
          float* dst = p.o_part + ((part_row0 + bb) * p.H + hg * NPAD + h_lo) * size_t(DLAT) + row;
#pragma unroll
          for (int c = 0; c < kHG; ++c)
            if (c < h_cnt) dst[size_t(c) * DLAT] = ntiles > 0 ? __uint_as_float(raw[bb][c]) * invl[bb * NPAD + h_lo + c] : 0.f;
        }
      }
    } else
    for (int bb = 0; bb < NB; ++bb) {
      for (int sb = 0; sb < SUB; ++sb) {
        float o[kHG];
        if (ntiles > 0) {
          uint32_t raw[kHG];
          const uint32_t taddr = tbase + lane_off + O_COL + (bb * SUB + sb) * NPAD + h_lo;
          if constexpr (kHG == 8) {
            tmem_ld8(taddr, raw);
          } else {
#pragma unroll
            for (int c = 0; c < kHG; c += 16) tmem_ld16(taddr + c, raw + c);
          }
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < kHG; ++c) o[c] = __uint_as_float(raw[c]) * invl[bb * NPAD + h_lo + c];
        } else {
#pragma unroll
          for (int c = 0; c < kHG; ++c) o[c] = 0.f;
        }
        if (row_ok) {
          float* dst = cm ? cm_o + size_t(h_lo) * DLAT + sb * DLS + row
                          : p.o_part + ((part_row0 + bb) * p.H + hg * NPAD + h_lo) * size_t(DLAT) + sb * DLS + row;
#pragma unroll
          for (int c = 0; c < kHG; ++c)
            if (c < h_cnt) dst[size_t(c) * DLAT] = o[c];
        }
      }
    }
    if (p.trace != nullptr && tid == 64 && cta_lin < 1024) p.trace[7 * 256 + 2048 + 8 * cta_lin + 5] = clock64();
    if (cm) {
      cluster_arrive_release();  // phase B: every split's O / lse of the sequence is in place
      cluster_wait_acquire();
      cp_async_wait_all();
      named_bar_sync(1, kSoftThreads);
      if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 3] = (long long)global_ns();
      cluster_combine(p.fz, p.B, p.H, DLAT, NPAD, seq, split, p.nsplit, cm_o, cm_lse, cm_w, cm_z, cm_wts, cm_ysum, cm_y,
                      tid - 64, tmem_base_sh[2]);
      if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 4] = (long long)global_ns();
      cluster_arrive_release();  // phase C: the cluster's DSMEM reads of this CTA are done
      cluster_wait_acquire();
    } else if (kK2FusedBuild && p.fused) {
      // publish this split's partials (barrier + one cumulative release), then this CTA's share
      // of the K3 units
      named_bar_sync(1, kSoftThreads);
      if (tid == 64) red_release_add(p.fz.sync + kSyncSeq + size_t(seq) * p.hgroups + hg, 1u);
      if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 3] = (long long)global_ns();
      if (p.fz.combine)
        fused_combine(p.fz, p.o_part, p.lse_part, p.B, p.H, p.nsplit, smem, cta_lin, ncta, tid - 64, tmem_base_sh[2],
                      cta_lin == p.trace_cta ? p.trace : nullptr);
      if (p.trace != nullptr && tid == 64 && cta_lin < 160) p.trace[16384 + 8 * cta_lin + 4] = (long long)global_ns();
    }
  }
  if (cm && (warp < 2 || warp == kPvWarp)) {
    // the producer and MMA warps take part in every cluster phase (barrier.cluster counts all threads)
    if (warp == 0) cluster_wait_acquire();  // phase A (arrived at its start)
    cluster_arrive_release();               // phase B
    cluster_wait_acquire();
    cluster_arrive_release();               // phase C
    cluster_wait_acquire();
  }
  if (p.late_trigger && !(warp >= 2 && warp < 2 + kSoftThreads / 32)) griddep_launch_dependents();
  tc_fence_before();
  if (p.trace != nullptr && warp >= 2) atomicAdd(&tmem_base_sh[1], 1u);
  __syncthreads();
  if (p.trace != nullptr && tid == 0 && cta_lin < 1024) {
    p.trace[7 * 256 + 2 * cta_lin + 1] = (long long)global_ns();
    p.trace[13824 + 2 * cta_lin + 1] = clock64();
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tbase);
  }
  if (kK2FusedBuild && p.fused == 1 && tid == 0) {
    // the last CTA out resets the step's counters for the next stream-ordered launch (visible to
    // it at the kernel boundary)
    if (atom_acq_rel_add(p.fz.sync + kSyncExit, 1u) == uint32_t(ncta - 1)) {
      const size_t nw = fuse_sync_words(p.B, p.H, p.hgroups);
      for (size_t i = 0; i < nw; ++i) p.fz.sync[i] = 0u;
    }
  }
}

}  // namespace mlra
