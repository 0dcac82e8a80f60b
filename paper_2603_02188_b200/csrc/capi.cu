// C ABI of libmlra_b200.so (include/mlra_b200.h): argument validation, TMA descriptor
// encoding, kernel selection and launch. No allocation; no synchronisation except in
// mlra_check_status (which exists to read the status word).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include "host_common.cuh"
#include "aux_kernels.cuh"
#include "outproj_kernel.cuh"
#include "allreduce_kernel.cuh"
#include "prefill_kernel.cuh"

namespace mlra_host {
thread_local char g_err[512] = "";
MLRA_DECODE_INSTANCES(MLRA_EXTERN_DECODE)
}  // namespace mlra_host

using namespace mlra_host;

namespace {

// TMA views of a pool [rows, W] bf16 (pure host descriptors, cached per thread so a decode
// loop over the same pool does not re-encode them every step):
//   lat  = 3-D {64 columns, rows, nlat 64-column chunks} (chunk stride 128 B), box
//          {64, T, DLS/64}: one box brings a DLS-wide sub-block of a T-token tile;
//   rope = 2-D {W, rows}, box {64, box_rows} (rope tiles, and sub-blocks of 64-token pages).
struct PoolMaps {
  const void* pool;
  cuuint64_t rows;
  int W, T, box_rows, DLS, nlat;
  CUtensorMap lat, rope;
};

int get_pool_maps(const void* pool, cuuint64_t total_rows, int W, int T, int box_rows, int DLS, int nlat,
                  const PoolMaps** out) {
  auto encode = get_encode();
  if (!encode) return fail(MLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  thread_local PoolMaps cache[8];
  thread_local int cache_next = 0;
  for (auto& e : cache)
    if (e.pool == pool && e.rows == total_rows && e.W == W && e.T == T && e.box_rows == box_rows && e.DLS == DLS &&
        e.nlat == nlat) {
      *out = &e;
      return MLRA_OK;
    }
  PoolMaps e{pool, total_rows, W, T, box_rows, DLS, nlat, {}, {}};
  {
    cuuint64_t dims[2] = {cuuint64_t(W), total_rows};
    cuuint64_t strides[1] = {cuuint64_t(W) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&e.rope, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(MLRA_ERR_CONFIG, "cuTensorMapEncodeTiled(2d) failed (%d): W=%d", int(cr), W);
  }
  {
    cuuint64_t dims[3] = {64, total_rows, cuuint64_t(nlat)};
    cuuint64_t strides[2] = {cuuint64_t(W) * 2, 128};
    cuuint32_t box[3] = {64, cuuint32_t(T), cuuint32_t(DLS / 64)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = encode(&e.lat, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(pool), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(MLRA_ERR_CONFIG, "cuTensorMapEncodeTiled(3d) failed (%d): W=%d", int(cr), W);
  }
  cache[cache_next] = e;
  *out = &cache[cache_next];
  cache_next = (cache_next + 1) % 8;
  return MLRA_OK;
}

// TMEM columns used: 2 S slots (+ 2 rope-logit slots when NB > 1) + NB*SUB O blocks, NPAD each (<= 512).
int pick_npad(int H, int NB, int SUB) {
  if (const char* e = getenv("MLRA_DEBUG_NPAD")) {  // dev: force the head-group width (16/32/64)
    const int v = atoi(e);
    const int slots = 2 + (NB > 1 ? 2 : 0) + NB * SUB;
    if ((v == 16 || v == 32 || v == 64) && slots * v <= 512 && !(NB == 4 && v == 64)) return v;
  }
  // registers: the softmax keeps NB x NPAD/2 sum partials per thread; cap NB = 4 at NPAD = 32
  if (NB == 4) return H <= 16 ? 16 : 32;
  // S slots (2) + shared rope-logit slots (2, NB > 1) + one O block per sub-block
  const int slots = 2 + (NB > 1 ? 2 : 0) + NB * SUB;
  for (int npad : {16, 32, 64}) {
    if (H <= npad && slots * npad <= 512) return npad;
  }
  return slots * 64 <= 512 ? 64 : 32;  // more head groups, each re-reading the tile
}

}  // namespace

extern "C" {

int mlra_version(void) { return 200; }

const char* mlra_last_error(void) { return g_err; }

int mlra_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(MLRA_ERR_CUDA, "cudaGetDevice failed");
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return fail(MLRA_ERR_CUDA, "cudaDeviceGetAttribute failed");
  return n;
}

int mlra_cache_append(const void* rows, const int32_t* block_table, int32_t* positions, int B, int W,
                      int page_size, int max_pages, int advance, void* pool, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (W <= 0 || W % 8 != 0) return fail(MLRA_ERR_SHAPE, "cache_append: row width %d must be a positive multiple of 8", W);
  if (page_size <= 0 || max_pages <= 0) return fail(MLRA_ERR_CONFIG, "cache_append: bad page geometry");
  launch_ex(mlra::cache_append_kernel, dim3(B), dim3(64), 0, static_cast<cudaStream_t>(stream), false, 
      static_cast<const __nv_bfloat16*>(rows), block_table, positions, W, page_size, max_pages, advance,
      static_cast<__nv_bfloat16*>(pool));
  return cuda_check("cache_append launch");
}

static int absorb_impl(const void* q_nope, const void* q_rope, const void* w_uk, void* q_abs, void* q_rope_out, int B,
                       int H, int DH, int NB, int DLAT, int DR, float score_scale, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (H <= 0 || DH <= 0 || NB <= 0 || DLAT <= 0 || DLAT % 2 != 0 || DR < 0)
    return fail(MLRA_ERR_SHAPE, "absorb_query: bad dims H=%d DH=%d NB=%d DLAT=%d DR=%d", H, DH, NB, DLAT, DR);
  if (DLAT % 8 != 0) return fail(MLRA_ERR_SHAPE, "absorb_query: DLAT=%d not a multiple of 8", DLAT);
  if (DH > 1024) return fail(MLRA_ERR_SHAPE, "absorb_query: DH=%d too large", DH);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (DH % 32 != 0) {
    // small/odd head widths (the reference's test dims): per-head GEMM, whole K in smem
    constexpr int NT = 32;
    const size_t smem = mlra::head_gemm_smem<NT>(DH);
    auto kern = mlra::head_gemm_kernel<__nv_bfloat16, true, NT>;
    static unsigned hg_done = 0;
    if (int rc = set_smem_once(kern, hg_done, 200 * 1024)) return rc;
    const int NCOL = NB * DLAT;
    dim3 grid((NCOL + NT - 1) / NT, H, (B + mlra::kHG_S - 1) / mlra::kHG_S);
    launch_ex(kern, dim3(grid), dim3(mlra::kHG_THREADS), smem, st, false, static_cast<const __nv_bfloat16*>(q_nope),
                                                static_cast<const __nv_bfloat16*>(w_uk), q_abs, B, H, DH, NCOL, 1,
                                                score_scale, NB, DLAT, static_cast<const __nv_bfloat16*>(q_rope),
                                                DR > 0 ? static_cast<__nv_bfloat16*>(q_rope_out) : nullptr, DR);
    return cuda_check("absorb_query launch");
  }
  if ((reinterpret_cast<uintptr_t>(w_uk) & 15) != 0)
    return fail(MLRA_ERR_CONFIG, "absorb_query: w_uk must be 16-byte aligned");
  // CTA = (128 latent columns, head, 4 sequences): W^UK tile staged in smem, one column per thread
  const size_t smem = mlra::absorb4_smem();
  const int NCOL = NB * DLAT;
  // tensor-core K1 when its grid (128 columns x head x 16 sequences per CTA) has >= 64 CTAs;
  // below that (one branch per device: TP4 ranks) the 4-sequence FMA kernel spreads wider
  const long am_ctas = long((NCOL + 127) / 128) * H * ((B + 15) / 16);
  if (DH % 16 == 0 && DH <= mlra::kAmMaxDH && (reinterpret_cast<uintptr_t>(q_nope) & 15) == 0 &&
      (am_ctas >= 64 || getenv("MLRA_K1_MMA") != nullptr) && getenv("MLRA_K1_FMA") == nullptr) {
    const size_t asmem = mlra::absorb_mma_smem(DH);
    static unsigned am_done = 0;
    if (int rc = set_smem_once(mlra::absorb_mma_kernel, am_done, int(mlra::absorb_mma_smem(mlra::kAmMaxDH)))) return rc;
    dim3 agrid((NCOL + 127) / 128, H, (B + 15) / 16);
    if (launch_ex(mlra::absorb_mma_kernel, agrid, dim3(mlra::kAmThreads), asmem, st, false,
                  static_cast<const __nv_bfloat16*>(q_nope), static_cast<const __nv_bfloat16*>(w_uk),
                  static_cast<__nv_bfloat16*>(q_abs), B, H, DH, NB, DLAT, score_scale,
                  static_cast<const __nv_bfloat16*>(q_rope), DR > 0 ? static_cast<__nv_bfloat16*>(q_rope_out) : nullptr,
                  DR) != cudaSuccess)
      return cuda_check("absorb_query launch");
    return cuda_check("absorb_query launch");
  }
  dim3 grid((NCOL + mlra::kG4Cols - 1) / mlra::kG4Cols, H, (B + mlra::kG4Seqs - 1) / mlra::kG4Seqs);
  if (launch_ex(mlra::absorb4_kernel, grid, dim3(mlra::kG4Threads), smem, st, false,
                static_cast<const __nv_bfloat16*>(q_nope), static_cast<const __nv_bfloat16*>(w_uk),
                static_cast<__nv_bfloat16*>(q_abs), B, H, DH, NB, DLAT, score_scale,
                static_cast<const __nv_bfloat16*>(q_rope), DR > 0 ? static_cast<__nv_bfloat16*>(q_rope_out) : nullptr,
                DR) != cudaSuccess)
    return cuda_check("absorb_query launch");
  return cuda_check("absorb_query launch");
}

int mlra_cache_append_latent(const float* kv_raw, const float* kr_raw, const int32_t* rope_pos, int32_t* slots,
                             const int32_t* block_table, int B, int d_c, int branches, int block0, int nblocks,
                             int dlp, int dr, int drp, float alpha_kv, float rope_base, float eps, int page_size,
                             int max_pages, int norm_groups, int advance, void* pool, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (norm_groups < 1 || norm_groups > 4 || d_c % norm_groups != 0)
    return fail(MLRA_ERR_CONFIG, "cache_append_latent: %d RMS groups over d_c=%d", norm_groups, d_c);
  if (d_c <= 0 || branches <= 0 || d_c % branches != 0)
    return fail(MLRA_ERR_SHAPE, "cache_append_latent: d_c=%d not split into %d branches", d_c, branches);
  const int bs = d_c / branches;
  if (block0 < 0 || nblocks < 1 || block0 + nblocks > branches || dlp < bs)
    return fail(MLRA_ERR_CONFIG, "cache_append_latent: blocks [%d, %d) of %d (width %d, padded %d)", block0,
                block0 + nblocks, branches, bs, dlp);
  if (dr < 0 || dr % 2 != 0 || drp < dr || drp % 2 != 0)
    return fail(MLRA_ERR_CONFIG, "cache_append_latent: rope width %d (padded %d) must be even", dr, drp);
  if (page_size <= 0 || max_pages <= 0) return fail(MLRA_ERR_CONFIG, "cache_append_latent: bad page geometry");
  launch_ex(mlra::cache_append_latent_kernel, dim3(B), dim3(mlra::kK0Threads), 0, static_cast<cudaStream_t>(stream),
            (advance & 2) != 0 && getenv("MLRA_NO_PDL") == nullptr,
      kv_raw, kr_raw, rope_pos, slots, block_table, d_c, bs, block0, nblocks, dlp, dr, drp, alpha_kv, rope_base, eps,
      page_size, max_pages, norm_groups, advance, static_cast<__nv_bfloat16*>(pool));
  return cuda_check("cache_append_latent launch");
}

int mlra_absorb_query(const void* q_nope, const void* q_rope, const void* w_uk, void* q_abs, void* q_rope_out, int B,
                      int H, int DH, int NB, int DLAT, int DR, float score_scale, void* stream) {
  return absorb_impl(q_nope, q_rope, w_uk, q_abs, q_rope_out, B, H, DH, NB, DLAT, DR, score_scale, stream);
}

// Workspace of mlra_decode_step: [status word | q~ | scaled q_rope | o_part | lse_part | merge /
// per-chunk scratch | fused-step counters], each 256-byte aligned. The status word (int32, the
// first 4 bytes of every workspace) collects the kernels' numeric flags (mlra_check_status).
constexpr int kPlanMaxCtas = 1024;
struct WsLayout {
  size_t q_abs, q_rope, o_part, lse, zbuf, sync, plan, total;
};

static WsLayout ws_layout(int B, int H, int NB, int DLAT, int DR, int nsplit) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  WsLayout w;
  size_t o = 256;  // status word
  w.q_abs = o; o += al(size_t(B) * NB * H * DLAT * 2);
  w.q_rope = o; o += al(size_t(B) * H * (DR > 0 ? DR : 1) * 2);
  w.o_part = o; o += al(size_t(B) * nsplit * NB * H * DLAT * 4);
  w.lse = o; o += al(size_t(B) * nsplit * NB * H * 4);
  w.zbuf = o; o += al(size_t(B) * NB * H * DLAT * 4);
  // fused-step counters: head groups <= ceil(H / 16) (the smallest head group is 16)
  w.sync = o; o += al(mlra::fuse_sync_words(B, H, (H + 15) / 16) * 4);
  w.plan = o; o += al(size_t(kPlanMaxCtas) * 4 * 4 + size_t(B) * 4);  // ragged-batch work items + split counts
  w.total = o;
  return w;
}

size_t mlra_workspace_bytes(int B, int H, int NB, int DLAT, int DR, int nsplit) {
  return ws_layout(B, H, NB, DLAT, DR, nsplit).total;
}

int mlra_check_status(int32_t* status, int reset, void* stream) {
  if (status == nullptr) return fail(MLRA_ERR_CONFIG, "check_status: null status word");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t v = 0;
  if (cudaMemcpyAsync(&v, status, sizeof v, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return cuda_check("check_status copy");
  if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_check("check_status sync");
  if (v != 0 && reset) {
    if (cudaMemsetAsync(status, 0, sizeof v, st) != cudaSuccess) return cuda_check("check_status reset");
  }
  if (v & mlra::kStatusNaN) return fail(MLRA_ERR_NUMERIC, "softmax_rows: NaN in input (status 0x%x)", v);
  if (v & mlra::kStatusNoFinite) return fail(MLRA_ERR_NUMERIC, "softmax_rows: row with no finite entry (status 0x%x)", v);
  return MLRA_OK;
}

int mlra_default_splits_heads(int B, int max_seqlen, int NB, int SUB, int H) {
  const int groups = H > 0 ? (H + pick_npad(H, NB, SUB) - 1) / pick_npad(H, NB, SUB) : 1;
  return mlra_default_splits(B * groups, max_seqlen, NB, SUB);
}

int mlra_default_splits(int B, int max_seqlen, int NB, int SUB) {
  int sms = mlra_num_sms();
  if (sms <= 0) sms = 148;
  const int T = (SUB == 1) ? 128 : 64;
  const int tiles = (max_seqlen + T - 1) / T;
  int s = sms / B;  // one wave of CTAs (1 CTA / SM); a partial second wave costs a full round
  if (s < 1) s = 1;
  if (s > tiles) s = tiles;
  if (s > mlra::kMergeMaxSplits) s = mlra::kMergeMaxSplits;
  return s < 1 ? 1 : s;
}

static int decode_impl(const void* q_abs, const void* q_rope, const void* pool, const int32_t* block_table,
                       const int32_t* seqlens, float* o_part, float* lse_part, int B, int H, int NB, int SUB, int DLS,
                       int DR, int page_size, int max_pages, int num_pages, int nsplit, void* stream,
                       bool pdl = false, const mlra::FuseArgs* fz = nullptr, int fuse_mode = 1,
                       const int32_t* plan = nullptr, int plan_ctas = 0, int late = -1);

int mlra_decode_partials(const void* q_abs, const void* q_rope, const void* pool, const int32_t* block_table,
                         const int32_t* seqlens, float* o_part, float* lse_part, int B, int H, int NB, int SUB,
                         int DLS, int DR, int page_size, int max_pages, int num_pages, int nsplit, void* stream) {
  return decode_impl(q_abs, q_rope, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR, page_size,
                     max_pages, num_pages, nsplit, stream, false);
}

static int decode_impl(const void* q_abs, const void* q_rope, const void* pool, const int32_t* block_table,
                       const int32_t* seqlens, float* o_part, float* lse_part, int B, int H, int NB, int SUB, int DLS,
                       int DR, int page_size, int max_pages, int num_pages, int nsplit, void* stream,
                       bool pdl, const mlra::FuseArgs* fz, int fuse_mode, const int32_t* plan, int plan_ctas,
                       int late) {
  if (B <= 0) return MLRA_OK;
  if (NB < 1 || NB > 4) return fail(MLRA_ERR_CONFIG, "decode: NB=%d branches per device not in [1,4]", NB);
  if (SUB < 1 || NB * SUB > 8) return fail(MLRA_ERR_CONFIG, "decode: SUB=%d sub-blocks not supported", SUB);
  if (DLS != 64 && DLS != 128) return fail(MLRA_ERR_CONFIG, "decode: sub-block width %d not in {64,128}", DLS);
  if (DR < 16 || DR > 64 || DR % 16 != 0) return fail(MLRA_ERR_CONFIG, "decode: rope width %d not in {16..64}/16", DR);
  if (page_size <= 0 || page_size % 64 != 0) return fail(MLRA_ERR_CONFIG, "decode: page_size %d not a multiple of 64", page_size);
  if (nsplit < 1 || nsplit > mlra::kMergeMaxSplits) return fail(MLRA_ERR_CONFIG, "decode: nsplit %d not in [1,%d]", nsplit, mlra::kMergeMaxSplits);
  if (H < 1) return fail(MLRA_ERR_SHAPE, "decode: H=%d", H);
  if (NB == 3) return fail(MLRA_ERR_CONFIG, "decode: NB=3 branches per device is not a TP layout");
  if (SUB > 1 && NB != 1) return fail(MLRA_ERR_CONFIG, "decode: multi-block latents (SUB>1) need NB=1");
  const int DLAT = SUB * DLS;
  const int W = NB * DLAT + DR;
  const int T = (SUB == 1) ? 128 : 64;  // SUB > 1 (MLA) keeps 2*SUB sub-blocks resident: 64-token tiles
  const int box_rows = (page_size % T == 0) ? T : 64;
  const cuuint64_t total_rows = cuuint64_t(num_pages) * cuuint64_t(page_size);
  const PoolMaps* hit = nullptr;
  if (int rc = get_pool_maps(pool, total_rows, W, T, box_rows, DLS, NB * DLAT / 64, &hit)) return rc;
  const CUtensorMap& lat_map = hit->lat;
  const CUtensorMap& rope_map = hit->rope;

  mlra::DecodeParams p{};
  p.q_abs = static_cast<const __nv_bfloat16*>(q_abs);
  p.q_rope = static_cast<const __nv_bfloat16*>(q_rope);
  p.block_table = block_table;
  p.seqlens = seqlens;
  p.o_part = o_part;
  p.lse_part = lse_part;
  p.B = B; p.H = H; p.SUB = SUB; p.DR = DR; p.W = W;
  p.page_size = page_size; p.max_pages = max_pages; p.nsplit = nsplit; p.box_rows = box_rows;
  p.pdl = pdl ? 1 : 0;
  p.plan = plan;
  p.plan_ctas = plan_ctas;
  p.late_trigger = late >= 0 ? late : getenv("MLRA_K3_PDL") != nullptr;
  if (fz != nullptr) {
    if (!mlra::kK2FusedBuild) return fail(MLRA_ERR_CONFIG, "fused / cluster step: library built without MLRA_K2_FUSED_STEP");
    p.fused = fuse_mode;
    p.fz = *fz;
    p.pdl = 0;  // the fused step reads the cache and the raw queries from its first instruction
  }
  p.rescale_threshold = mlra::kRescaleThreshold;
  if (const char* e = getenv("MLRA_DEBUG_RESCALE_THRESHOLD")) p.rescale_threshold = float(atof(e));
  if (const char* e = getenv("MLRA_DEBUG_TRACE_PTR")) p.trace = reinterpret_cast<long long*>(strtoull(e, nullptr, 0));
  if (const char* e = getenv("MLRA_DEBUG_TRACE_CTA")) p.trace_cta = atoi(e);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool t128 = (T == 128);
  const int npad = pick_npad(H, NB, SUB);
  const int hgroups = (H + npad - 1) / npad;
#define MLRA_NPAD(TT, DD, NBB)                                                      \
  do {                                                                              \
    if (npad == 16) return launch_decode<TT, 16, DD, NBB>(lat_map, rope_map, p, hgroups, st); \
    if (npad == 32) return launch_decode<TT, 32, DD, NBB>(lat_map, rope_map, p, hgroups, st); \
    return launch_decode<TT, 64, DD, NBB>(lat_map, rope_map, p, hgroups, st);     \
  } while (0)
#define MLRA_DISPATCH(TT, DD)                                                                 \
  do {                                                                                        \
    if (NB == 1) MLRA_NPAD(TT, DD, 1);                                                        \
    if (NB == 2) MLRA_NPAD(TT, DD, 2);                                                        \
    if (npad == 16) return launch_decode<TT, 16, DD, 4>(lat_map, rope_map, p, hgroups, st);   \
    return launch_decode<TT, 32, DD, 4>(lat_map, rope_map, p, hgroups, st);                   \
  } while (0)
  if (DLS == 128) {
    if (t128) MLRA_DISPATCH(128, 128);
    MLRA_NPAD(64, 128, 1);
  }
  if (t128) MLRA_DISPATCH(128, 64);
  MLRA_NPAD(64, 64, 1);
#undef MLRA_DISPATCH
#undef MLRA_NPAD
}

// ----------------------------------------------------------------------------- GQA variant
// KV heads per CTA: the largest of {4, 2, 1} dividing the device's KV-head count.
static int gqa_nbc(int G) { return G % 4 == 0 ? 4 : (G % 2 == 0 ? 2 : 1); }

static int gqa_decode_impl(const void* q, const void* pool, const int32_t* block_table, const int32_t* seqlens,
                           float* o_part, float* lse_part, int B, int G, int R, int DH, int page_size, int max_pages,
                           int num_pages, int nsplit, float score_scale, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (G < 1) return fail(MLRA_ERR_CONFIG, "gqa decode: G=%d KV heads", G);
  if (R < 1 || R > 16) return fail(MLRA_ERR_CONFIG, "gqa decode: %d query heads per KV head not in [1,16]", R);
  if (DH != 64 && DH != 128) return fail(MLRA_ERR_CONFIG, "gqa decode: padded head width %d not in {64,128}", DH);
  if (page_size <= 0 || page_size % 64 != 0) return fail(MLRA_ERR_CONFIG, "gqa decode: page_size %d not a multiple of 64", page_size);
  if (nsplit < 1 || nsplit > mlra::kMergeMaxSplits) return fail(MLRA_ERR_CONFIG, "gqa decode: nsplit %d not in [1,%d]", nsplit, mlra::kMergeMaxSplits);
  const int W = 2 * G * DH;
  const int T = 128;
  const int box_rows = (page_size % T == 0) ? T : 64;
  const cuuint64_t total_rows = cuuint64_t(num_pages) * cuuint64_t(page_size);
  const PoolMaps* maps = nullptr;
  if (int rc = get_pool_maps(pool, total_rows, W, T, box_rows, DH, W / 64, &maps)) return rc;
  mlra::DecodeParams p{};
  p.q_abs = static_cast<const __nv_bfloat16*>(q);
  p.q_rope = nullptr;
  p.block_table = block_table;
  p.seqlens = seqlens;
  p.o_part = o_part;
  p.lse_part = lse_part;
  p.B = B; p.H = R; p.SUB = 1; p.DR = 0; p.W = W;
  p.page_size = page_size; p.max_pages = max_pages; p.nsplit = nsplit; p.box_rows = box_rows;
  p.nb_total = G;
  p.qk_scale = score_scale;
  p.rescale_threshold = mlra::kRescaleThreshold;
  if (const char* e = getenv("MLRA_DEBUG_TRACE_PTR")) p.trace = reinterpret_cast<long long*>(strtoull(e, nullptr, 0));
  if (const char* e = getenv("MLRA_DEBUG_TRACE_CTA")) p.trace_cta = atoi(e);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nbc = gqa_nbc(G), z = G / nbc;
#define MLRA_GQA(DD)                                                                      \
  do {                                                                                    \
    if (nbc == 4) return launch_decode<128, 16, DD, 4, true>(maps->lat, maps->rope, p, z, st); \
    if (nbc == 2) return launch_decode<128, 16, DD, 2, true>(maps->lat, maps->rope, p, z, st); \
    return launch_decode<128, 16, DD, 1, true>(maps->lat, maps->rope, p, z, st);          \
  } while (0)
  if (DH == 128) MLRA_GQA(128);
  MLRA_GQA(64);
#undef MLRA_GQA
}

// K3 needs a [B, H, NB*DLAT] fp32 scratch for the merged latent when it up-projects; the
// standalone entry point allocates it from a per-thread cache (mlra_decode_step passes the
// workspace slice instead).
static int allreduce_launch(mlra::AllReduceParams& p, int nlocal, bool sim, cudaStream_t st);
static int combine_variant(const float* o_part, const float* lse_part, const void* w_uv, float* out, float* zbuf,
                           int B, int H, int NB, int DLAT, int DH, int nsplit, float alpha, int upproj, cudaStream_t st,
                           bool pdl, const mlra::TpSum* tp, int32_t* status, const int32_t* seq_splits);

// After a K3 variant without the fused TP sum: K5 on the output, in place, same region.
static int tp_sum_after(const mlra::TpSum* tp, float* out, int n, cudaStream_t st) {
  if (tp == nullptr || tp->world <= 1) return MLRA_OK;
  mlra::AllReduceParams p = {};
  p.x[0] = out;
  p.y[0] = out;
  for (int r = 0; r < tp->world; ++r) p.comm[r] = tp->comm[r];
  p.n = n, p.world = tp->world, p.rank0 = tp->rank;
  return allreduce_launch(p, 1, false, st);
}

static int combine_impl(const float* o_part, const float* lse_part, const void* w_uv, float* out, float* zbuf, int B,
                        int H, int NB, int DLAT, int DH, int nsplit, float alpha, int upproj, cudaStream_t st,
                        bool pdl = false, const mlra::TpSum* tp = nullptr, int32_t* status = nullptr,
                        const int32_t* seq_splits = nullptr) {
  if (int rc = combine_variant(o_part, lse_part, w_uv, out, zbuf, B, H, NB, DLAT, DH, nsplit, alpha, upproj, st, pdl, tp,
                               status, seq_splits))
    return rc == 1 ? tp_sum_after(tp, out, B * H * DH, st) : rc;
  return MLRA_OK;
}

// Returns MLRA_OK when the output is complete (TP sum fused in K3 when requested), 1 when a
// requested TP sum still has to run (the K3 variant has no fused sum), < 0 on error.
// K3 variant: 1 split-K clusters, 3 the split merge + head GEMM, 0 the per-branch CTAs (or, when
// their smem does not fit, the merge + head GEMM as a fallback)
static int k3_variant(int B, int H, int NB, int DLAT, int DH, int nsplit, int upproj, const void* w_uv,
                      const int32_t* seq_splits) {
  const int KP = nsplit > 24 ? 8 : 4;
  const size_t sksmem = KP == 8 ? mlra::combine_splitk_smem<8>(NB, DLAT, DH) : mlra::combine_splitk_smem<4>(NB, DLAT, DH);
  // Cost model in dependent L2 round trips per thread (12 split loads in flight per item):
  // per-branch CTAs (combine4) 2 * ceil(nsplit/12); split-K CTAs (all branches, 1/KP of the
  // splits each) 2*NB * ceil(ceil(nsplit/KP)/12), plus two cluster barriers -- worth it at
  // 1.5x fewer round trips (small batches: many splits per sequence).
  const int rt_c4 = 2 * ((nsplit + 11) / 12);
  const int rt_sk = 2 * NB * (((nsplit + KP - 1) / KP + 11) / 12);
  // dev: MLRA_K3_FORCE = 1 split-K cluster, 2 per-branch CTAs, 3 merge + head GEMM
  const int force = getenv("MLRA_K3_FORCE") ? atoi(getenv("MLRA_K3_FORCE")) : 0;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Split-K clusters while their grid fits one wave; beyond that, at batch 1 (many heads: 64 x 8
  // CTAs) the one-round-trip merge plus the head GEMM measured faster (64 heads, B = 1, 128K:
  // K3 13.4 -> 8.4 us). Ragged plans (per-sequence split counts, most sequences have few) take
  // the per-branch CTAs.
  const long sk_ctas = long((B + 3) / 4) * H * KP;
  const bool many_splits = 3 * rt_sk < 2 * rt_c4;
  const bool sk_ok = seq_splits == nullptr && upproj == 1 && NB * DLAT <= 512 && DH % (8 * KP) == 0 &&
                     256 % (DH / KP) == 0 && sksmem <= size_t(kSmemBudget) &&
                     (reinterpret_cast<uintptr_t>(w_uv) & 15) == 0;
  if (force == 1) return sk_ok ? 1 : 0;
  if (force == 3) return 3;
  if (force == 2) return 0;
  // Measured per shape (MLRA_K3_FORCE, tools/gpu_r3s.sh / gpu_r3u.sh): the split-K clusters win
  // only for 1-2 sequences, the merge + head GEMM only at batch 1 beyond one split-K wave; from
  // 4 sequences on (and at 2 beyond one wave) the per-branch CTAs are faster (MLRA-4 TP4 rank
  // B = 8 4K 25.6 -> 16.2 us, 32K 38.7 -> 29.2; MLA TP4 rank B = 8 4K 33.1 -> 24.6 us, 32K
  // 73.8 -> 65.3; 64 heads B = 4 4K 21.1 -> 17.7).
  if (sk_ok && many_splits) {
    if (sk_ctas <= sms && B <= 2) return 1;
    if (sk_ctas > sms && B == 1) return 3;
    // two sequences with very many splits: the clusters even over a second partial wave
    // (MLRA-4 TP4 rank B = 2 32K: 22.1 -> 19.0 us)
    if (B == 2 && sk_ctas <= 2L * sms && 4 * rt_sk <= rt_c4) return 1;
    // two sequences over many heads (> 2 split-K waves) and >= 64 splits: the merge + head GEMM
    // (64 heads B = 2 32K / 128K: 24.2 / 35.9 -> 23.4 / 34.8 us; at 33 splits it loses)
    if (B == 2 && sk_ctas > 2L * sms && nsplit >= 64) return 3;
  }
  return 0;
}

// K3 released at K2's epilogue (programmatic dependent): only for the merge + head GEMM over
// many heads (64 heads at batch 1: step 29.4 -> 27.6 us; 24 heads measured 0.4 us slower)
static bool k3_late(int B, int H, int NB, int DLAT, int DH, int nsplit, const void* w_uv) {
  if (getenv("MLRA_K3_PDL") != nullptr) return true;
  return k3_variant(B, H, NB, DLAT, DH, nsplit, 1, w_uv, nullptr) == 3 &&
         long((B + 3) / 4) * H * (nsplit > 24 ? 8 : 4) > 2L * mlra_num_sms();
}

static int combine_variant(const float* o_part, const float* lse_part, const void* w_uv, float* out, float* zbuf,
                           int B, int H, int NB, int DLAT, int DH, int nsplit, float alpha, int upproj, cudaStream_t st,
                           bool pdl, const mlra::TpSum* tp, int32_t* status, const int32_t* seq_splits) {
  const int tp_pending = (tp != nullptr && tp->world > 1 && upproj == 1) ? 1 : 0;
  const int rows = B * NB * H;
  // summed output: split-K merge over a cluster of KP CTAs (KP = 8 once the splits are many)
  const int KP = nsplit > 24 ? 8 : 4;
  const size_t sksmem = KP == 8 ? mlra::combine_splitk_smem<8>(NB, DLAT, DH) : mlra::combine_splitk_smem<4>(NB, DLAT, DH);
  const int variant = k3_variant(B, H, NB, DLAT, DH, nsplit, upproj, w_uv, seq_splits);
  const bool merge_gemm = variant == 3;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (variant == 1) {
    auto kern = KP == 8 ? mlra::combine_splitk_kernel<8> : mlra::combine_splitk_kernel<4>;
    static unsigned attr4 = 0, attr8 = 0;
    if (int rc = set_smem_once(kern, KP == 8 ? attr8 : attr4, kSmemBudget)) return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((B + 3) / 4, H, KP);
    cfg.blockDim = dim3(mlra::kSkThreads);
    cfg.dynamicSmemBytes = sksmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = KP;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kern, o_part, lse_part, static_cast<const __nv_bfloat16*>(w_uv), out, B, H, NB, DLAT,
                           DH, nsplit, alpha, status, seq_splits) != cudaSuccess)
      return cuda_check("combine launch");
    if (int rc = cuda_check("combine launch")) return rc;
    return tp_pending;
  }
  // 2 sequences per CTA (one merge item per thread) while the grid stays within one wave
  // (4 CTAs per SM), else 4
  const bool seq2 = long((B + 1) / 2) * H * NB <= 4L * sms && getenv("MLRA_K3_SEQ4") == nullptr;
  // many sequences (prefill's pseudo-sequences): 8 per CTA halves the W^UV re-reads
  const bool seq8 = !seq2 && B >= 256;
  const size_t c4smem = seq2   ? mlra::combine4_smem<2>(DLAT, DH, nsplit)
                        : seq8 ? mlra::combine4_smem<8>(DLAT, DH, nsplit)
                               : mlra::combine4_smem<4>(DLAT, DH, nsplit);
  if (upproj != 0 && !merge_gemm && c4smem <= size_t(kSmemBudget) && (size_t(DLAT) * DH * 2) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(w_uv) & 15) == 0) {
    // CTA = (2 or 4 sequences, head, branch); with a summed output the NB branch CTAs of a
    // (sequence group, head) form a cluster and add their results through DSMEM.
    // (8 sequences per CTA measured slower even where 4 needs 1.3 waves.)
    auto kern = seq2 ? mlra::combine4_kernel<2> : seq8 ? mlra::combine4_kernel<8> : mlra::combine4_kernel<4>;
    static unsigned attr_done2 = 0, attr_done4 = 0, attr_done8 = 0;
    if (int rc = set_smem_once(kern, seq2 ? attr_done2 : seq8 ? attr_done8 : attr_done4, kSmemBudget)) return rc;
    const int per_branch = upproj == 2 ? 1 : 0;
    const int seqs = seq2 ? 2 : seq8 ? 8 : 4;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((B + seqs - 1) / seqs, H, NB);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = c4smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = (NB > 1 && !per_branch) ? NB : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // TP sum fused into the epilogue when every CTA of the grid is resident (flag waits)
    mlra::TpSum tps = {};
    int fused = 0;
    if (tp_pending) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, c4smem);
      if (long(cfg.gridDim.x) * cfg.gridDim.y * cfg.gridDim.z <= long(sms) * per_sm &&
          long(cfg.gridDim.x) * cfg.gridDim.y <= mlra::kArFlagSlots) {
        tps = *tp;
        fused = 1;
      }
    }
    if (cudaLaunchKernelEx(&cfg, kern, o_part, lse_part, static_cast<const __nv_bfloat16*>(w_uv), out, B, H, NB, DLAT,
                           DH, nsplit, alpha, per_branch, tps, status, seq_splits) != cudaSuccess)
      return cuda_check("combine launch");
    if (int rc = cuda_check("combine launch")) return rc;
    return fused ? MLRA_OK : tp_pending;
  }
  // merge: 32 columns x 16 split groups per CTA when the rows are few and the splits many
  // (batch-1 decode), else 128 columns x 4; PDL: the CTAs start while K2 drains
  const bool wide = long(rows) * ((DLAT + 127) / 128) < 148 && nsplit > 16;
  const int mcw = wide ? 32 : 128;
  auto merge = wide ? mlra::merge_splits_kernel<mlra::kMergeQWide> : mlra::merge_splits_kernel<mlra::kMergeQ>;
  const dim3 mgrid(rows, (DLAT + mcw - 1) / mcw), mblock(512);
  if (upproj == 0) {
    launch_ex(merge, mgrid, mblock, 0, st, pdl, o_part, lse_part, out, B, NB, H, DLAT, nsplit, alpha, 1, status,
              seq_splits);
    return cuda_check("merge launch");
  }
  launch_ex(merge, mgrid, mblock, 0, st, pdl, o_part, lse_part, zbuf, B, NB, H, DLAT, nsplit, 1.f, 0, status,
            seq_splits);
  const int kparts = (upproj == 2) ? NB : 1;
  constexpr int NT = 32;
  const int kp = NB * DLAT / kparts;
  const size_t smem = mlra::head_gemm_smem<NT>(kp);
  if (smem > 200 * 1024) return fail(MLRA_ERR_SHAPE, "combine: latent width %d too large", kp);
  auto kern = mlra::head_gemm_kernel<float, false, NT>;
  static unsigned attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32 || !(attr_done & (1u << dev))) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (dev < 32) attr_done |= 1u << dev;
  }
  dim3 grid((DH + NT - 1) / NT, H, ((B + mlra::kHG_S - 1) / mlra::kHG_S) * kparts);
  launch_ex(kern, dim3(grid), dim3(mlra::kHG_THREADS), smem, st, getenv("MLRA_NO_PDL") == nullptr, zbuf,
            static_cast<const __nv_bfloat16*>(w_uv), out, B, H, NB * DLAT,
                                              DH, kparts, alpha, 0, 0, nullptr, nullptr, 0);
  if (int rc = cuda_check("up-projection launch")) return rc;
  return tp_pending;
}

int mlra_combine(const float* o_part, const float* lse_part, const void* w_uv, float* out, float* scratch, int B,
                 int H, int NB, int DLAT, int DH, int nsplit, float alpha, int upproj, int32_t* status, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (NB < 1 || NB > 4 || nsplit < 1 || nsplit > mlra::kMergeMaxSplits) return fail(MLRA_ERR_CONFIG, "combine: NB=%d nsplit=%d", NB, nsplit);
  if (upproj < 0 || upproj > 2) return fail(MLRA_ERR_CONFIG, "combine: upproj mode %d", upproj);
  if (upproj && (DH % 8 != 0)) return fail(MLRA_ERR_SHAPE, "combine: DH=%d not a multiple of 8", DH);
  if (upproj && scratch == nullptr) return fail(MLRA_ERR_CONFIG, "combine: up-projection needs a scratch buffer");
  // PDL: the merge's prologue overlaps K2's drain when K2 is the previous launch on the stream
  return combine_impl(o_part, lse_part, w_uv, out, scratch, B, H, NB, DLAT, DH, nsplit, alpha, upproj,
                      static_cast<cudaStream_t>(stream), getenv("MLRA_NO_PDL") == nullptr, nullptr, status);
}

static int decode_step_impl(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv,
                            const void* pool, const int32_t* block_table, const int32_t* seqlens, float* out,
                            void* workspace, int B, int H, int DH, int NB, int SUB, int DLS, int DR, int page_size,
                            int max_pages, int num_pages, int nsplit, float score_scale, float alpha, void* stream,
                            const mlra::TpSum* tp);

int mlra_decode_step(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv, const void* pool,
                     const int32_t* block_table, const int32_t* seqlens, float* out, void* workspace, int B, int H,
                     int DH, int NB, int SUB, int DLS, int DR, int page_size, int max_pages, int num_pages,
                     int nsplit, float score_scale, float alpha, void* stream) {
  return decode_step_impl(q_nope, q_rope, w_uk, w_uv, pool, block_table, seqlens, out, workspace, B, H, DH, NB, SUB,
                          DLS, DR, page_size, max_pages, num_pages, nsplit, score_scale, alpha, stream, nullptr);
}

int mlra_decode_step_tp(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv, const void* pool,
                        const int32_t* block_table, const int32_t* seqlens, float* out, void* workspace, int B, int H,
                        int DH, int NB, int SUB, int DLS, int DR, int page_size, int max_pages, int num_pages,
                        int nsplit, float score_scale, float alpha, int rank, int world, void* const* comm,
                        void* stream) {
  if (world < 1 || world > mlra::kArMaxRanks || rank < 0 || rank >= world)
    return fail(MLRA_ERR_CONFIG, "decode_step_tp: rank %d of %d", rank, world);
  if (world > 1 && comm == nullptr) return fail(MLRA_ERR_CONFIG, "decode_step_tp: no communication regions");
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return fail(MLRA_ERR_CONFIG, "decode_step_tp: out not 16-byte aligned");
  mlra::TpSum tp = {};
  tp.world = world;
  tp.rank = rank;
  for (int r = 0; r < world && world > 1; ++r) tp.comm[r] = static_cast<float*>(comm[r]);
  return decode_step_impl(q_nope, q_rope, w_uk, w_uv, pool, block_table, seqlens, out, workspace, B, H, DH, NB, SUB,
                          DLS, DR, page_size, max_pages, num_pages, nsplit, score_scale, alpha, stream,
                          world > 1 ? &tp : nullptr);
}

static int decode_step_impl(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv,
                            const void* pool, const int32_t* block_table, const int32_t* seqlens, float* out,
                            void* workspace, int B, int H, int DH, int NB, int SUB, int DLS, int DR, int page_size,
                            int max_pages, int num_pages, int nsplit, float score_scale, float alpha, void* stream,
                            const mlra::TpSum* tp) {
  if (B <= 0) return MLRA_OK;
  const int DLAT = SUB * DLS;
  const WsLayout wl = ws_layout(B, H, NB, DLAT, DR, nsplit);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int32_t* status = reinterpret_cast<int32_t*>(ws);
  void* q_abs = ws + wl.q_abs;
  void* q_rope_s = ws + wl.q_rope;
  float* o_part = reinterpret_cast<float*>(ws + wl.o_part);
  float* lse_part = reinterpret_cast<float*>(ws + wl.lse);
  float* zbuf = reinterpret_cast<float*>(ws + wl.zbuf);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (w_uk == nullptr) {
    // Pre-absorbed queries (mlra_proj_query with W^UQ.W^UK_b pre-multiplied wrote q~ and the
    // scaled rotary query): K2 as a programmatic dependent of the projection, then K3.
    const bool late = k3_late(B, H, NB, DLAT, DH, nsplit, w_uv);
    int rc = decode_impl(q_nope, q_rope, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR,
                         page_size, max_pages, num_pages, nsplit, stream, getenv("MLRA_NO_PDL") == nullptr, nullptr, 1,
                         nullptr, 0, late ? 1 : 0);
    if (rc) return rc;
    return combine_impl(o_part, lse_part, w_uv, out, zbuf, B, H, NB, DLAT, DH, nsplit, alpha, 1, st, late, tp, status);
  }
  // One launch per step when the whole grid is co-resident (fused_step.cuh): K1 in K2's prologue,
  // K3 (+ the TP sum) in its epilogue. Otherwise (or with MLRA_NO_FUSE) the three kernels below.
  const int CW = mlra::combine_chunk_width(DLAT);
  const bool fusable = getenv("MLRA_NO_FUSE") == nullptr && DH % 16 == 0 && DLAT % 16 == 0 && NB * DLAT % CW == 0 &&
                       (NB * DLAT == CW || DH <= CW) && DR % 2 == 0 && (reinterpret_cast<uintptr_t>(w_uv) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(q_nope) & 3) == 0 &&
                       (tp == nullptr || long(mlra::fuse_groups(B)) * H <= mlra::kArFlagSlots);
  // Cluster step (one branch per device: an MLRA-4 / MLA TP rank): K1 and K3 inside the cluster of
  // a sequence's split CTAs, hand-offs through DSMEM (fused_step.cuh).
  if (getenv("MLRA_FUSE_CLUSTER") != nullptr && NB == 1 &&
      (DH == 64 || DH == 128 || DH == 256) && DR % 2 == 0 && DR <= 64 && nsplit >= 2 && nsplit <= 16 &&
      (reinterpret_cast<uintptr_t>(w_uv) & 15) == 0 &&
      (tp == nullptr || long(B) * nsplit <= mlra::kArFlagSlots)) {
    mlra::FuseArgs f = {};
    f.q_nope = static_cast<const __nv_bfloat16*>(q_nope);
    f.q_rope = static_cast<const __nv_bfloat16*>(q_rope);
    f.w_uk = static_cast<const __nv_bfloat16*>(w_uk);
    f.w_uv = static_cast<const __nv_bfloat16*>(w_uv);
    f.out = out;
    f.status = status;
    if (tp != nullptr) f.tp = *tp;
    f.score_scale = score_scale;
    f.alpha = alpha;
    f.DH = DH, f.NB = NB, f.DLAT = DLAT;
    // The cluster size is the split count of the step; the largest one <= nsplit whose B clusters
    // are all resident at once (e.g. 16 x 9 CTAs do not fit the GPCs, 16 x 8 do). The choice
    // depends only on the shape: cached per thread.
    struct Pick { int B, H, DLAT, DR, nsplit, dev, ns; };
    thread_local Pick picks[8];
    thread_local int pick_next = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int ns = 0;
    for (auto& e : picks)
      if (e.nsplit == nsplit && e.B == B && e.H == H && e.DLAT == DLAT && e.DR == DR && e.dev == dev && e.ns != 0) ns = e.ns;
    if (ns == 0) {
      ns = -1;
      for (int c = std::min(nsplit, 16); c >= 2 && 2 * c >= nsplit; --c) {
        const int rc = decode_impl(q_abs, q_rope_s, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS,
                                   DR, page_size, max_pages, num_pages, c, stream, false, &f, 2);
        if (rc == kNotFusable) continue;
        if (rc != MLRA_OK) return rc;
        ns = c;
        break;
      }
      picks[pick_next] = {B, H, DLAT, DR, nsplit, dev, ns};
      pick_next = (pick_next + 1) % 8;
      if (ns > 0) return MLRA_OK;  // launched while probing
    } else if (ns > 0) {
      const int rc = decode_impl(q_abs, q_rope_s, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR,
                                 page_size, max_pages, num_pages, ns, stream, false, &f, 2);
      if (rc != kNotFusable) return rc;
    }
  }
  if (fusable && getenv("MLRA_FUSE_GRID") != nullptr) {  // dev: the grid-wide fused step
    mlra::FuseArgs f = {};
    f.q_nope = static_cast<const __nv_bfloat16*>(q_nope);
    f.q_rope = static_cast<const __nv_bfloat16*>(q_rope);
    f.w_uk = static_cast<const __nv_bfloat16*>(w_uk);
    f.w_uv = static_cast<const __nv_bfloat16*>(w_uv);
    f.q_abs = static_cast<__nv_bfloat16*>(q_abs);
    f.q_rope_s = static_cast<__nv_bfloat16*>(q_rope_s);
    f.out = out;
    f.ybuf = zbuf;
    f.sync = reinterpret_cast<uint32_t*>(ws + wl.sync);
    f.status = status;
    if (tp != nullptr) f.tp = *tp;
    f.score_scale = score_scale;
    f.alpha = alpha;
    f.DH = DH, f.NB = NB, f.DLAT = DLAT;
    f.absorb = 1;
    f.combine = 1;
    f.debug_reps = 1;
    if (const char* e = getenv("MLRA_DEBUG_FUSE_REPS")) f.debug_reps = std::max(1, atoi(e));
    f.debug_producer_wait = getenv("MLRA_DEBUG_PRODUCER_WAIT") != nullptr;
    if (const char* e = getenv("MLRA_FUSE_PARTS")) {  // dev: "absorb" or "combine" alone
      f.absorb = strstr(e, "absorb") != nullptr;
      f.combine = strstr(e, "combine") != nullptr;
    }
    if (!f.absorb) {
      if (int rc = absorb_impl(q_nope, q_rope, w_uk, q_abs, q_rope_s, B, H, DH, NB, DLAT, DR, score_scale, stream))
        return rc;
    }
    int rc = decode_impl(q_abs, q_rope_s, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR,
                         page_size, max_pages, num_pages, nsplit, stream, false, &f);
    if (rc == MLRA_OK && !f.combine)
      rc = combine_impl(o_part, lse_part, w_uv, out, zbuf, B, H, NB, DLAT, DH, nsplit, alpha, 1, st, false, tp, status);
    if (rc != kNotFusable) return rc;
    if (!f.absorb) return fail(MLRA_ERR_CONFIG, "MLRA_FUSE_PARTS: grid not fusable");
  }
  // K1 then K2 with programmatic dependent launch (K2's TMA producer streams the cache while
  // K1 drains -- the cache was written before K1 started -- and waits on K1 only before
  // reading the queries), then K3 in plain stream order. (K3 launched dependent on K2 measured
  // 5-30 us slower per step: its early CTAs cost more than the overlap gains.)
  const bool pdl = getenv("MLRA_NO_PDL") == nullptr;
  int rc = absorb_impl(q_nope, q_rope, w_uk, q_abs, q_rope_s, B, H, DH, NB, DLAT, DR, score_scale, stream);
  if (rc) return rc;
  const bool late = k3_late(B, H, NB, DLAT, DH, nsplit, w_uv);
  rc = decode_impl(q_abs, q_rope_s, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR, page_size,
                   max_pages, num_pages, nsplit, stream, pdl, nullptr, 1, nullptr, 0, late ? 1 : 0);
  if (rc) return rc;
  return combine_impl(o_part, lse_part, w_uv, out, zbuf, B, H, NB, DLAT, DH, nsplit, alpha, 1, st, late, tp, status);
}

int mlra_gqa_default_splits(int B, int G, int max_seqlen) {
  int sms = mlra_num_sms();
  if (sms <= 0) sms = 148;
  if (B < 1 || G < 1) return 1;
  const int z = G / gqa_nbc(G);
  const int tiles = (max_seqlen + 127) / 128;
  int s = sms / (B * z);
  if (s > tiles) s = tiles;
  if (s > mlra::kMergeMaxSplits) s = mlra::kMergeMaxSplits;
  return s < 1 ? 1 : s;
}

int mlra_gqa_decode_partials(const void* q, const void* pool, const int32_t* block_table, const int32_t* seqlens,
                             float* o_part, float* lse_part, int B, int G, int R, int DH, int page_size, int max_pages,
                             int num_pages, int nsplit, float score_scale, void* stream) {
  return gqa_decode_impl(q, pool, block_table, seqlens, o_part, lse_part, B, G, R, DH, page_size, max_pages, num_pages,
                         nsplit, score_scale, stream);
}

// GQA workspace: [status word | o_part | lse_part], 256-byte aligned.
size_t mlra_gqa_workspace_bytes(int B, int G, int R, int DH, int nsplit) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return 256 + al(size_t(B) * nsplit * G * R * DH * 4) + al(size_t(B) * nsplit * G * R * 4);
}

int mlra_gqa_decode_step(const void* q, const void* pool, const int32_t* block_table, const int32_t* seqlens,
                         float* out, void* workspace, int B, int G, int R, int DH, int page_size, int max_pages,
                         int num_pages, int nsplit, float score_scale, void* stream) {
  if (B <= 0) return MLRA_OK;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int32_t* status = reinterpret_cast<int32_t*>(ws);
  ws += 256;
  float* o_part = reinterpret_cast<float*>(ws);
  ws += al(size_t(B) * nsplit * G * R * DH * 4);
  float* lse_part = reinterpret_cast<float*>(ws);
  int rc = gqa_decode_impl(q, pool, block_table, seqlens, o_part, lse_part, B, G, R, DH, page_size, max_pages,
                           num_pages, nsplit, score_scale, stream);
  if (rc) return rc;
  // split merge; KV head b's query head j is output head b*R + j (out [B, G*R, DH])
  return combine_impl(o_part, lse_part, nullptr, out, nullptr, B, R, G, DH, DH, nsplit, 1.f, 0,
                      static_cast<cudaStream_t>(stream), false, nullptr, status);
}

// ----------------------------------------------------------------------------- K4 (output side)
size_t mlra_outproj_comm_bytes(int B, int D, int world) {
  if (B <= 0 || D <= 0 || world <= 0) return 0;
  const size_t nslabs = size_t(mlra::outproj_nslabs(D));
  return size_t(2) * world * B * D * 4 + size_t(2) * world * nslabs * mlra::kOpMaxKS * 4 + 16;
}

static int outproj_check(int B, int K, int D, int world) {
  if (B <= 0 || B > mlra::kOpMaxB) return fail(MLRA_ERR_SHAPE, "outproj: B=%d outside [1, %d]", B, mlra::kOpMaxB);
  if (K <= 0 || K % 8 != 0 || D <= 0 || D % 8 != 0)
    return fail(MLRA_ERR_SHAPE, "outproj: K=%d and D=%d must be positive multiples of 8", K, D);
  if (world < 1 || world > mlra::kOpMaxRanks)
    return fail(MLRA_ERR_CONFIG, "outproj: world %d outside [1, %d]", world, mlra::kOpMaxRanks);
  return MLRA_OK;
}

static unsigned g_outproj_attr = 0;

size_t mlra_outproj_workspace_bytes(int B, int K) {
  return (B <= 0 || K <= 0) ? 0 : (size_t(B) * K * 2 + 255) / 256 * 256;
}

// K4a (gate + bf16 cast) then K4. Grid of K4: nslabs x KS CTAs per local rank. Real mode:
// clusters of KS CTAs (K slices of a slab), KS = the largest that keeps one wave (every CTA
// resident: a CTA waiting for its slab's flags must not hold back one a peer waits for), K4 a
// programmatic dependent of K4a. Sim mode: KS = 1, one cooperative launch per call.
static int outproj_launch(mlra::OutProjParams& p, const float* const* attn, const float* const* gate,
                          void* const* ws, int nlocal, bool sim, cudaStream_t st) {
  const size_t smem = mlra::outproj_smem();
  auto kern = mlra::outproj_allreduce_kernel;
  if (int rc = set_smem_once(kern, g_outproj_attr, int(smem))) return rc;
  const int n = p.B * p.K;
  for (int r = 0; r < nlocal; ++r) {
    if (attn[r] == nullptr || ws[r] == nullptr || p.w_o[r] == nullptr || p.y[r] == nullptr)
      return fail(MLRA_ERR_CONFIG, "outproj: null tensor pointer (rank slot %d)", r);
    launch_ex(mlra::outproj_gate_kernel, dim3((n / 8 + 255) / 256), dim3(256), 0, st, false, attn[r], gate != nullptr ? gate[r] : nullptr,
                                                                   static_cast<__nv_bfloat16*>(ws[r]), n);
    p.a[r] = static_cast<const __nv_bfloat16*>(ws[r]);
  }
  if (int rc = cuda_check("outproj gate launch")) return rc;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, mlra::kOpThreads, smem);
  p.nslabs = mlra::outproj_nslabs(p.D);
  const int kchunks = (p.K + mlra::kOpKC - 1) / mlra::kOpKC;
  int ks = sim ? 1 : std::max(1, std::min({mlra::kOpMaxKS, kchunks, sms * per_sm / p.nslabs}));
  if (const char* e = getenv("MLRA_DEBUG_OUTPROJ_KS")) ks = std::max(1, std::min(ks, atoi(e)));  // dev override
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  cfg.blockDim = dim3(mlra::kOpThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  for (;; --ks) {
    cfg.gridDim = dim3(p.nslabs * ks, nlocal);
    if (sim) {
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.numAttrs = 1;
      if (p.world > 1 && size_t(cfg.gridDim.x) * nlocal > size_t(sms) * per_sm)
        return fail(MLRA_ERR_CONFIG, "outproj_sim: %d CTAs cannot all be resident (%d SMs x %d)",
                    int(cfg.gridDim.x * nlocal), sms, per_sm);
      break;
    }
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
    int clusters = sms * per_sm;
    if (ks > 1 && cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      clusters = 0;
    }
    if (clusters >= p.nslabs) break;
    if (ks == 1) {
      if (p.world > 1)
        return fail(MLRA_ERR_CONFIG, "outproj: %d slabs cannot all be resident (%d SMs x %d)", p.nslabs, sms, per_sm);
      break;
    }
  }
  p.ks_count = ks;
  p.k_slice = ((p.K + ks - 1) / ks + 63) / 64 * 64;
  if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return cuda_check("outproj launch");
  return cuda_check("outproj launch");
}

int mlra_outproj(const float* attn, const float* gate_pre, const void* w_o, const float* resid, float* y, int B,
                 int K, int D, int rank, int world, void* const* comm, void* workspace, void* stream) {
  if (int rc = outproj_check(B, K, D, world)) return rc;
  if (rank < 0 || rank >= world) return fail(MLRA_ERR_CONFIG, "outproj: rank %d of %d", rank, world);
  if (world > 1 && comm == nullptr)
    return fail(MLRA_ERR_CONFIG, "outproj: world %d needs the communication regions", world);
  mlra::OutProjParams p = {};
  p.w_o[0] = static_cast<const __nv_bfloat16*>(w_o);
  p.y[0] = y;
  p.resid = resid;
  for (int r = 0; r < world && world > 1; ++r) p.comm[r] = static_cast<float*>(comm[r]);
  p.B = B, p.K = K, p.D = D, p.world = world, p.rank0 = rank;
  return outproj_launch(p, &attn, &gate_pre, &workspace, 1, false, static_cast<cudaStream_t>(stream));
}

int mlra_outproj_sim(const float* const* attn, const float* const* gate_pre, const void* const* w_o,
                     const float* resid, float* const* y, int B, int K, int D, int world, void* const* comm,
                     void* const* workspace, void* stream) {
  if (int rc = outproj_check(B, K, D, world)) return rc;
  if (attn == nullptr || w_o == nullptr || y == nullptr || workspace == nullptr || comm == nullptr)
    return fail(MLRA_ERR_CONFIG, "outproj_sim: needs per-rank tensors, workspaces and comm regions");
  mlra::OutProjParams p = {};
  for (int r = 0; r < world; ++r) {
    p.w_o[r] = static_cast<const __nv_bfloat16*>(w_o[r]);
    p.y[r] = y[r];
    p.comm[r] = static_cast<float*>(comm[r]);
  }
  p.resid = resid;
  p.B = B, p.K = K, p.D = D, p.world = world, p.rank0 = 0;
  return outproj_launch(p, attn, gate_pre, workspace, world, true, static_cast<cudaStream_t>(stream));
}

// ----------------------------------------------------------------------------- K5 (peer all-reduce)
size_t mlra_allreduce_comm_bytes(int n, int world) {
  if (n <= 0 || world <= 0) return 0;
  return mlra::ar_region_bytes(n, world);
}

static int allreduce_launch(mlra::AllReduceParams& p, int nlocal, bool sim, cudaStream_t st) {
  if (p.n <= 0) return MLRA_OK;
  if (p.world < 1 || p.world > mlra::kArMaxRanks)
    return fail(MLRA_ERR_CONFIG, "allreduce: world %d outside [1, %d]", p.world, mlra::kArMaxRanks);
  p.nchunks = (p.n + mlra::kArChunk - 1) / mlra::kArChunk;
  if (p.nchunks > mlra::kArFlagSlots) return fail(MLRA_ERR_SHAPE, "allreduce: %d values exceed %d chunks", p.n, mlra::kArFlagSlots);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mlra::allreduce_kernel, mlra::kArThreads, 0);
  if (size_t(p.nchunks) * nlocal > size_t(sms) * per_sm)
    return fail(MLRA_ERR_CONFIG, "allreduce: %d CTAs cannot all be resident (%d SMs x %d)", p.nchunks * nlocal, sms,
                per_sm);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(p.nchunks, nlocal);
  cfg.blockDim = dim3(mlra::kArThreads);
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = sim ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, mlra::allreduce_kernel, p) != cudaSuccess) return cuda_check("allreduce launch");
  return cuda_check("allreduce launch");
}

int mlra_allreduce(const float* x, float* y, int n, int rank, int world, void* const* comm, void* stream) {
  if (world < 1 || rank < 0 || rank >= world) return fail(MLRA_ERR_CONFIG, "allreduce: rank %d of %d", rank, world);
  if (comm == nullptr || x == nullptr || y == nullptr) return fail(MLRA_ERR_CONFIG, "allreduce: null pointer");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) != 0)
    return fail(MLRA_ERR_CONFIG, "allreduce: x and y must be 16-byte aligned");
  mlra::AllReduceParams p = {};
  p.x[0] = x;
  p.y[0] = y;
  for (int r = 0; r < world && r < mlra::kArMaxRanks; ++r) p.comm[r] = static_cast<float*>(comm[r]);
  p.n = n, p.world = world, p.rank0 = rank;
  return allreduce_launch(p, 1, false, static_cast<cudaStream_t>(stream));
}

int mlra_allreduce_sim(const float* const* x, float* const* y, int n, int world, void* const* comm, void* stream) {
  if (world < 1 || world > mlra::kArMaxRanks) return fail(MLRA_ERR_CONFIG, "allreduce_sim: world %d", world);
  if (comm == nullptr || x == nullptr || y == nullptr) return fail(MLRA_ERR_CONFIG, "allreduce_sim: null pointer");
  mlra::AllReduceParams p = {};
  for (int r = 0; r < world; ++r) {
    if (((reinterpret_cast<uintptr_t>(x[r]) | reinterpret_cast<uintptr_t>(y[r])) & 15) != 0)
      return fail(MLRA_ERR_CONFIG, "allreduce_sim: x and y must be 16-byte aligned");
    p.x[r] = x[r];
    p.y[r] = y[r];
    p.comm[r] = static_cast<float*>(comm[r]);
  }
  p.n = n, p.world = world, p.rank0 = 0;
  return allreduce_launch(p, world, true, static_cast<cudaStream_t>(stream));
}

int mlra_comm_alloc(size_t bytes, void** dev_ptr_out) {
  if (bytes == 0 || dev_ptr_out == nullptr) return fail(MLRA_ERR_CONFIG, "comm_alloc: empty request");
  if (cudaMalloc(dev_ptr_out, bytes) != cudaSuccess) return cuda_check("cudaMalloc (comm region)");
  if (cudaMemset(*dev_ptr_out, 0, bytes) != cudaSuccess) return cuda_check("cudaMemset (comm region)");
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_check("comm_alloc sync");
  return MLRA_OK;
}

int mlra_comm_free(void* dev_ptr) {
  if (dev_ptr != nullptr && cudaFree(dev_ptr) != cudaSuccess) return cuda_check("cudaFree (comm region)");
  return MLRA_OK;
}

int mlra_ipc_handle(const void* dev_ptr, void* handle_out) {
  if (dev_ptr == nullptr || handle_out == nullptr) return fail(MLRA_ERR_CONFIG, "ipc_handle: null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handle");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)) != cudaSuccess) return cuda_check("cudaIpcGetMemHandle");
  std::memcpy(handle_out, &h, sizeof h);
  return MLRA_OK;
}

int mlra_ipc_open(const void* handle, void** dev_ptr_out) {
  if (handle == nullptr || dev_ptr_out == nullptr) return fail(MLRA_ERR_CONFIG, "ipc_open: null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  if (cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return cuda_check("cudaIpcOpenMemHandle");
  return MLRA_OK;
}

int mlra_ipc_close(void* dev_ptr) {
  if (dev_ptr == nullptr) return MLRA_OK;
  if (cudaIpcCloseMemHandle(dev_ptr) != cudaSuccess) return cuda_check("cudaIpcCloseMemHandle");
  return MLRA_OK;
}

}  // extern "C"

namespace {
int encode_3d(CUtensorMap* m, const void* base, cuuint64_t d0, cuuint64_t d1, cuuint64_t d2, cuuint64_t s1,
              cuuint64_t s2, cuuint32_t b0, cuuint32_t b1, cuuint32_t b2) {
  auto encode = get_encode();
  if (!encode) return fail(MLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return cr == CUDA_SUCCESS ? MLRA_OK : fail(MLRA_ERR_CONFIG, "cuTensorMapEncodeTiled(3d) failed (%d)", int(cr));
}

template <int DLAT, int DH>
int launch_prefill(const PoolMaps* pm, const void* q_abs, const void* q_rope, const void* w_uv, mlra::PrefillParams& p,
                   int DRq, cudaStream_t st) {
  using L = mlra::PrefillLayout<DLAT, DH>;
  CUtensorMap qm, rm, wm;
  {  // q~ head-major [H, n, NB, DLAT]: 4-D {DLAT, NB, n, H}, box {64, 1, 128, 1}
    auto encode = get_encode();
    cuuint64_t dims[4] = {cuuint64_t(DLAT), cuuint64_t(p.NB), cuuint64_t(p.n), cuuint64_t(p.H)};
    cuuint64_t strides[3] = {cuuint64_t(DLAT) * 2, cuuint64_t(p.NB) * DLAT * 2, cuuint64_t(p.n) * p.NB * DLAT * 2};
    cuuint32_t box[4] = {64, 1, mlra::kPfT, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult cr = encode(&qm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(q_abs), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(MLRA_ERR_CONFIG, "prefill: q~ tensor map failed (%d)", int(cr));
  }
  if (int rc = encode_3d(&rm, q_rope, DRq, p.H, p.n, cuuint64_t(DRq) * 2, cuuint64_t(p.H) * DRq * 2, 64, 1, mlra::kPfT))
    return rc;
  {
    auto encode = get_encode();
    cuuint64_t dims[2] = {cuuint64_t(DH), cuuint64_t(p.H) * p.NB * DLAT};
    cuuint64_t strides[1] = {cuuint64_t(DH) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(DLAT)};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&wm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w_uv), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(MLRA_ERR_CONFIG, "prefill: W^UV tensor map failed (%d)", int(cr));
  }
  auto kern = mlra::prefill_attention_kernel<DLAT, DH>;
  static unsigned done = 0;
  if (int rc = set_smem_once(kern, done, L::kSmem)) return rc;
  const int nqt = (p.n + mlra::kPfT - 1) / mlra::kPfT;
  launch_ex(kern, dim3(nqt * p.H), dim3(mlra::kPfThreads), L::kSmem, st, false, pm->lat, pm->rope, qm, rm, wm, p);
  return cuda_check("prefill_attention launch");
}
}  // namespace

extern "C" int mlra_prefill_attention(const void* q_abs, const void* q_rope, const void* w_uv, const void* pool,
                                      const int32_t* block_table, float* out, int n, int H, int NB, int DLAT, int DH,
                                      int DR, int DRp, int DRq, int page_size, int max_pages, int num_pages,
                                      float alpha, void* stream) {
  if (n <= 0) return MLRA_OK;
  if (H <= 0 || NB < 1 || NB > 4 || DR < 0 || DR > 64 || DRp < DR || DRp % 8 != 0 || DRq < DR || DRq % 8 != 0 ||
      DRq > 64)
    return fail(MLRA_ERR_SHAPE, "prefill_attention: bad dims H=%d NB=%d DR=%d DRp=%d DRq=%d", H, NB, DR, DRp, DRq);
  if (!((DLAT == 128 && DH == 128) || (DLAT == 64 && DH == 64)))
    return fail(MLRA_ERR_CONFIG, "prefill_attention: (DLAT, DH) = (%d, %d) not in {(128,128), (64,64)}", DLAT, DH);
  if (page_size % mlra::kPfT != 0) return fail(MLRA_ERR_CONFIG, "prefill_attention: page_size %d not a multiple of 128", page_size);
  if (long(max_pages) * page_size < n) return fail(MLRA_ERR_CONFIG, "prefill_attention: %d tokens exceed the page table", n);
  const int W = NB * DLAT + DRp;
  const PoolMaps* pm = nullptr;
  if (int rc = get_pool_maps(pool, cuuint64_t(num_pages) * page_size, W, mlra::kPfT, mlra::kPfT, DLAT, NB * DLAT / 64, &pm))
    return rc;
  mlra::PrefillParams p = {};
  p.block_table = block_table;
  p.out = out;
  p.n = n;
  p.H = H;
  p.NB = NB;
  p.DR = DR;
  p.page_size = page_size;
  p.max_pages = max_pages;
  p.alpha = alpha;
  p.rope_col = NB * DLAT;
  if (const char* e = getenv("MLRA_DEBUG_PF_S")) {
    p.dbg_s = reinterpret_cast<float*>(strtoull(e, nullptr, 0));
    p.dbg_cta = getenv("MLRA_DEBUG_PF_CTA") ? atoi(getenv("MLRA_DEBUG_PF_CTA")) : 0;
  }
#ifdef MLRA_PF_WAIT_STATS
  if (const char* e = getenv("MLRA_DEBUG_PF_WAITS")) {  // dev build: per-barrier wait cycles of CTA 0
    unsigned long long* ptr = reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0));
    cudaMemcpyToSymbolAsync(mlra::g_pf_wait_acc, &ptr, sizeof(ptr), 0, cudaMemcpyHostToDevice,
                            static_cast<cudaStream_t>(stream));
  }
#endif
  if (const char* e = getenv("MLRA_DEBUG_PF_PROGRESS")) p.progress = reinterpret_cast<volatile int*>(strtoull(e, nullptr, 0));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (DLAT == 128) return launch_prefill<128, 128>(pm, q_abs, q_rope, w_uv, p, DRq, st);
  return launch_prefill<64, 64>(pm, q_abs, q_rope, w_uv, p, DRq, st);
}

extern "C" int mlra_rows_split(const float* x, int n, int K, int ldx, int norm, float alpha, float eps, void* hi,
                               void* lo, int ldo, void* stream) {
  if (n <= 0) return MLRA_OK;
  if (K <= 0 || ldx < K || ldo < K) return fail(MLRA_ERR_SHAPE, "rows_split: K=%d ldx=%d ldo=%d", K, ldx, ldo);
  if (launch_ex(mlra::rows_split_kernel, dim3(n), dim3(256), 0, static_cast<cudaStream_t>(stream), false, x, K, ldx,
                norm, alpha, eps, static_cast<__nv_bfloat16*>(hi), static_cast<__nv_bfloat16*>(lo), ldo) != cudaSuccess)
    return cuda_check("rows_split launch");
  return cuda_check("rows_split launch");
}

extern "C" int mlra_query_epilogue(const float* y, int n, int ldy, int nq, int H, int dr, int drq, int pos0,
                                   float rope_base, float q_scale, float r_scale, void* q_out, void* r_out,
                                   void* stream) {
  if (n <= 0) return MLRA_OK;
  if (nq < 0 || H <= 0 || dr < 0 || dr % 2 != 0 || dr > 128 || drq < dr || drq % 2 != 0 || ldy < nq + H * dr)
    return fail(MLRA_ERR_SHAPE, "query_epilogue: bad dims nq=%d H=%d dr=%d drq=%d ldy=%d", nq, H, dr, drq, ldy);
  if (launch_ex(mlra::query_epilogue_kernel, dim3(n), dim3(256), 0, static_cast<cudaStream_t>(stream), false, y, ldy,
                nq, H, dr, drq, pos0, rope_base, q_scale, r_scale, static_cast<__nv_bfloat16*>(q_out),
                static_cast<__nv_bfloat16*>(r_out)) != cudaSuccess)
    return cuda_check("query_epilogue launch");
  return cuda_check("query_epilogue launch");
}

// ----------------------------------------------------------------------------- ragged batches
extern "C" int mlra_decode_plan(const int32_t* seqlens, int B, int tile_tokens, int ctas, int nsplit_max,
                                int32_t* plan, int32_t* seq_splits, float* lse_part, int NB, int H, void* stream) {
  if (B <= 0) return MLRA_OK;
  if (tile_tokens <= 0 || ctas < B || ctas > kPlanMaxCtas || nsplit_max < 1 || NB < 1 || H < 1)
    return fail(MLRA_ERR_CONFIG, "decode_plan: B=%d ctas=%d (>= B, <= %d) nsplit_max=%d", B, ctas, kPlanMaxCtas,
                nsplit_max);
  const size_t smem = size_t(2) * B * sizeof(int);
  if (smem > 48 * 1024) return fail(MLRA_ERR_CONFIG, "decode_plan: batch %d too large", B);
  (void)lse_part, (void)NB, (void)H;  // (kept in the signature: the K2 partial layout the plan serves)
  launch_ex(mlra::decode_plan_kernel, dim3(1), dim3(mlra::kPlanThreads), smem, static_cast<cudaStream_t>(stream), false, 
      seqlens, B, tile_tokens, ctas, nsplit_max, plan, seq_splits);
  return cuda_check("decode_plan launch");
}

extern "C" int mlra_decode_step_ragged(const void* q_nope, const void* q_rope, const void* w_uk, const void* w_uv,
                                       const void* pool, const int32_t* block_table, const int32_t* seqlens,
                                       float* out, void* workspace, int B, int H, int DH, int NB, int SUB, int DLS,
                                       int DR, int page_size, int max_pages, int num_pages, int nsplit_max,
                                       float score_scale, float alpha, void* stream) {
  if (B <= 0) return MLRA_OK;
  const int DLAT = SUB * DLS;
  const WsLayout wl = ws_layout(B, H, NB, DLAT, DR, nsplit_max);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  int32_t* status = reinterpret_cast<int32_t*>(ws);
  void* q_abs = ws + wl.q_abs;
  void* q_rope_s = ws + wl.q_rope;
  float* o_part = reinterpret_cast<float*>(ws + wl.o_part);
  float* lse_part = reinterpret_cast<float*>(ws + wl.lse);
  float* zbuf = reinterpret_cast<float*>(ws + wl.zbuf);
  int32_t* plan = reinterpret_cast<int32_t*>(ws + wl.plan);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int hgroups = (H + pick_npad(H, NB, SUB) - 1) / pick_npad(H, NB, SUB);
  const int ctas = std::min(kPlanMaxCtas, std::max(B, num_sms() / hgroups));
  const int T = (SUB == 1) ? 128 : 64;
  int32_t* seq_splits = plan + kPlanMaxCtas * 4;
  if (int rc = mlra_decode_plan(seqlens, B, T, ctas, nsplit_max, plan, seq_splits, lse_part, NB, H, stream)) return rc;
  if (w_uk != nullptr) {
    if (int rc = absorb_impl(q_nope, q_rope, w_uk, q_abs, q_rope_s, B, H, DH, NB, DLAT, DR, score_scale, stream))
      return rc;
  } else {
    q_abs = const_cast<void*>(q_nope);
    q_rope_s = const_cast<void*>(q_rope);
  }
  int rc = decode_impl(q_abs, q_rope_s, pool, block_table, seqlens, o_part, lse_part, B, H, NB, SUB, DLS, DR,
                       page_size, max_pages, num_pages, nsplit_max, stream, w_uk != nullptr && getenv("MLRA_NO_PDL") == nullptr,
                       nullptr, 1, plan, ctas);
  if (rc) return rc;
  return combine_impl(o_part, lse_part, w_uv, out, zbuf, B, H, NB, DLAT, DH, nsplit_max, alpha, 1, st, false, nullptr,
                      status, seq_splits);
}
