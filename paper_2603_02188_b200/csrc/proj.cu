// C ABI of the pre-attention projections (K-1, proj_kernel.cuh; include/mlra_b200.h):
// mlra_proj_down and mlra_proj_query. Validation, the weight's TMA descriptor (cached per
// weight pointer and shape), the split of K over a cluster, and the launch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include "host_common.cuh"
#include "proj_kernel.cuh"

using namespace mlra_host;

namespace {

struct WMap {
  const void* w;
  int K_pad, nslabs;
  CUtensorMap map;
};

// 2-D view {64 columns, nslabs * K_pad rows} of a slab-packed bf16 weight [nslabs][K_pad][64],
// box {64, 64}, 128-byte swizzle (cached per weight pointer and shape)
int get_w_map(const void* w, int K_pad, int nslabs, const CUtensorMap** out) {
  auto encode = get_encode();
  if (!encode) return fail(MLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  thread_local WMap cache[16];
  thread_local int next = 0;
  for (auto& e : cache)
    if (e.w == w && e.K_pad == K_pad && e.nslabs == nslabs) {
      *out = &e.map;
      return MLRA_OK;
    }
  WMap e{w, K_pad, nslabs, {}};
  cuuint64_t dims[2] = {cuuint64_t(mlra::kPjNC), cuuint64_t(K_pad) * nslabs};
  cuuint64_t strides[1] = {cuuint64_t(mlra::kPjNC) * 2};
  cuuint32_t box[2] = {mlra::kPjNC, mlra::kPjBox};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode(&e.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS)
    return fail(MLRA_ERR_CONFIG, "proj: cuTensorMapEncodeTiled failed (%d): K_pad=%d slabs=%d", int(cr), K_pad, nslabs);
  cache[next] = e;
  *out = &cache[next].map;
  next = (next + 1) % 16;
  return MLRA_OK;
}

// K slices per slab: the largest KS <= 8 whose nslabs clusters of KS CTAs are co-resident
// (cudaOccupancyMaxActiveClusters: a cluster lives in one GPC, and GPCs hold different SM
// counts), each slice <= kPjMaxRows rows. Cached per shape.
int pick_ks(int K, int nslabs, int* k_slice) {
  struct Pick { int K, nslabs, dev, ks; };
  thread_local Pick picks[16];
  thread_local int next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const int boxes = (K + mlra::kPjBox - 1) / mlra::kPjBox;
  const int need = (K + mlra::kPjMaxRows - 1) / mlra::kPjMaxRows;
  if (need > mlra::kPjMaxKS) return -1;
  int ks = 0;
  for (auto& e : picks)
    if (e.K == K && e.nslabs == nslabs && e.dev == dev && e.ks > 0) ks = e.ks;
  if (const char* e = getenv("MLRA_DEBUG_PROJ_KS")) ks = std::max(need, std::min(mlra::kPjMaxKS, atoi(e)));
  if (ks == 0) {
    ks = need;
    for (int c = std::min(mlra::kPjMaxKS, boxes); c > need; --c) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nslabs * c);
      cfg.blockDim = dim3(mlra::kPjThreads);
      cfg.dynamicSmemBytes = mlra::proj_smem();
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = c;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, mlra::proj_gemm_kernel, &cfg) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (nc >= nslabs) {
        ks = c;
        break;
      }
    }
    picks[next] = {K, nslabs, dev, ks};
    next = (next + 1) % 16;
  }
  *k_slice = ((boxes + ks - 1) / ks) * mlra::kPjBox;  // slices are whole 64-row boxes (the last shorter)
  return (K + *k_slice - 1) / *k_slice;               // slices actually non-empty
}

int launch_proj(const void* w, mlra::ProjParams& p, cudaStream_t st) {
  static unsigned done = 0;
  if (int rc = set_smem_once(mlra::proj_gemm_kernel, done, int(mlra::proj_smem()))) return rc;
  const int nslabs = (p.N + mlra::kPjNC - 1) / mlra::kPjNC;
  p.K_pad = (p.K + mlra::kPjBox - 1) / mlra::kPjBox * mlra::kPjBox;
  const CUtensorMap* map = nullptr;
  if (int rc = get_w_map(w, p.K_pad, nslabs, &map)) return rc;
  int k_slice = 0;
  const int ks = pick_ks(p.K, nslabs, &k_slice);
  if (ks < 0) return fail(MLRA_ERR_SHAPE, "proj: K=%d exceeds %d x %d rows", p.K, mlra::kPjMaxKS, mlra::kPjMaxRows);
  p.KS = ks;
  p.k_slice = k_slice;
  if (const char* e = getenv("MLRA_DEBUG_PROJ_TRACE")) p.trace = reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nslabs * ks);
  cfg.blockDim = dim3(mlra::kPjThreads);
  cfg.dynamicSmemBytes = mlra::proj_smem();
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  CUtensorMap m = *map;
  const int M = p.M;
  // one launch per 16 rows (the weight stream is the cost; decode batches are <= 16 per group)
  for (int m0 = 0; m0 < M; m0 += mlra::kPjM) {
    mlra::ProjParams q = p;
    q.M = std::min(mlra::kPjM, M - m0);
    q.x = p.x + size_t(m0) * p.ldx;
    if (p.mode == 0) {
      for (int i = 0; i < 3; ++i) {
        const int width = p.seg_end[i] - (i ? p.seg_end[i - 1] : 0);
        if (q.seg_out[i]) q.seg_out[i] = p.seg_out[i] + size_t(m0) * width;
      }
      if (p.ssq_out != nullptr && M > mlra::kPjM)
        return fail(MLRA_ERR_SHAPE, "proj_down: ssq partials need M <= %d (got %d)", mlra::kPjM, M);
    } else {
      if (p.ssq_in != nullptr && M > mlra::kPjM)
        return fail(MLRA_ERR_SHAPE, "proj_query: rmsnorm partials need M <= %d (got %d)", mlra::kPjM, M);
      q.q_out = p.q_out + size_t(m0) * p.nq;
      q.r_out = p.r_out + size_t(m0) * p.H * p.drp;
      q.pos = p.pos + m0;
    }
    if (cudaLaunchKernelEx(&cfg, mlra::proj_gemm_kernel, m, q) != cudaSuccess) return cuda_check("proj launch");
  }
  return cuda_check("proj launch");
}

}  // namespace

extern "C" {

int mlra_proj_down(const float* x, const void* w, int M, int K, int n_q, int n_kv, int n_kr, float* c_q_raw,
                   float* kv_raw, float* kr_raw, float* ssq, void* stream) {
  if (M <= 0) return MLRA_OK;
  const int n_used = n_q + n_kv + n_kr, N = n_used;
  if (K <= 0 || n_q < 0 || n_kv < 0 || n_kr < 0 || n_used <= 0)
    return fail(MLRA_ERR_SHAPE, "proj_down: bad dims K=%d n_q=%d n_kv=%d n_kr=%d", K, n_q, n_kv, n_kr);
  if ((reinterpret_cast<uintptr_t>(w) & 15) != 0) return fail(MLRA_ERR_CONFIG, "proj_down: w must be 16-byte aligned");
  mlra::ProjParams p = {};
  p.x = x;
  p.ldx = K;
  p.M = M;
  p.K = K;
  p.N = N;
  p.mode = 0;
  p.seg_out[0] = c_q_raw;
  p.seg_out[1] = kv_raw;
  p.seg_out[2] = kr_raw;
  p.seg_end[0] = n_q;
  p.seg_end[1] = n_q + n_kv;
  p.seg_end[2] = n_used;
  p.ssq_out = ssq;
  p.ssq_cols = ssq != nullptr ? n_q : 0;
  return launch_proj(w, p, static_cast<cudaStream_t>(stream));
}

int mlra_proj_query(const float* c_q_raw, const float* ssq, float alpha_q, float eps, const void* w, int M, int K,
                    int nq, int H, int dr, int drp, const int32_t* pos, int pos_delta, float rope_base, float q_scale, float r_scale,
                    void* q_out, void* r_out, void* stream) {
  if (M <= 0) return MLRA_OK;
  if (K <= 0 || nq <= 0 || nq % 2 != 0 || H <= 0 || dr < 0 || dr % 2 != 0 || dr > 64 || drp < dr)
    return fail(MLRA_ERR_SHAPE, "proj_query: bad dims K=%d nq=%d H=%d dr=%d drp=%d", K, nq, H, dr, drp);
  const int N = nq + H * dr;
  if ((reinterpret_cast<uintptr_t>(w) & 15) != 0) return fail(MLRA_ERR_CONFIG, "proj_query: w must be 16-byte aligned");
  if (dr > 0 && (r_out == nullptr || pos == nullptr)) return fail(MLRA_ERR_CONFIG, "proj_query: rope output needs r_out and pos");
  mlra::ProjParams p = {};
  p.x = c_q_raw;
  p.ldx = K;
  p.ssq_in = ssq;
  p.norm_parts = (K + mlra::kPjNC - 1) / mlra::kPjNC;
  p.norm_alpha = alpha_q;
  p.eps = eps;
  p.M = M;
  p.K = K;
  p.N = N;
  p.mode = 1;
  p.q_out = static_cast<__nv_bfloat16*>(q_out);
  p.r_out = static_cast<__nv_bfloat16*>(r_out);
  p.nq = nq;
  p.H = H;
  p.dr = dr > 0 ? dr : 2;
  p.drp = drp > 0 ? drp : 2;
  p.pos = pos;
  p.pos_delta = pos_delta;
  p.rope_base = rope_base;
  for (int l = 0; l < dr / 2; ++l) p.theta[l] = pow(double(rope_base), -2.0 * l / dr);
  p.q_scale = q_scale;
  p.r_scale = r_scale;
  return launch_proj(w, p, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
