// Host-side helpers shared by the translation units of libmlra_b200.so: error reporting,
// launch wrappers, and the K2 launcher template (its instantiations are compiled in the
// decode_inst_*.cu units so the build runs them in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include "../../include/mlra_b200.h"
#include "decode_kernel.cuh"

namespace mlra_host {

extern thread_local char g_err[512];  // defined in capi.cu

inline int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

inline int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MLRA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return MLRA_OK;
}

// Launch with (pdl = true) programmatic stream serialization: the kernel may start before its
// predecessor on the stream finishes and must griddepcontrol.wait before consuming its output.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
template <typename K>
int set_smem_once(K kern, unsigned& done_mask, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 32 && (done_mask & (1u << dev))) return MLRA_OK;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return cuda_check("cudaFuncSetAttribute");
  if (dev < 32) done_mask |= 1u << dev;
  return MLRA_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

inline int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

constexpr int kSmemBudget = 232448;  // 227 KB opt-in dynamic smem (the kernel has no static smem)
constexpr int kNotFusable = 1;       // launch_decode: the fused step cannot run this grid (caller falls back)

// K2 launch: ring depths from the smem budget, then one launch of grid (nsplit, B, head_groups).
// With p.fused the grid must be co-resident (one CTA per SM, grid <= #SMs) and the K3 units'
// staging must fit in the (then idle) ring; otherwise nothing is launched and kNotFusable is
// returned.
template <int T, int NPAD, int DLS, int NB, bool GQA = false>
int launch_decode(const CUtensorMap& lat_map, const CUtensorMap& rope_map, mlra::DecodeParams p, int head_groups,
                  cudaStream_t stream) {
  using L = mlra::DecodeLayout<T, NPAD, DLS>;
  const int q_chunks = NB * p.SUB * (DLS / 64) + 1;
  auto fixed = [&](int p_slots) { return q_chunks * L::kQChunkBytes + p_slots * L::kPBytes + L::kScratchBytes; };
  auto fits = [&](int lat, int rope, int ps) { return L::smem_bytes(NB, p.SUB, lat, rope, ps) <= kSmemBudget; };
  int rope_slots = 0, lat_slots = 0, p_slots = 2;
  if (GQA) {
    // K and V sub-blocks share one ring; no rope part
    lat_slots = (kSmemBudget - fixed(2)) / L::kLatBytes;
    if (lat_slots < 3) return fail(MLRA_ERR_CONFIG, "gqa decode: ring of %d slots < 3", lat_slots);
  } else if (NB > 1) {
    // Several branches per tile share one rope tile (consumed by the tile's first QK): one
    // rope slot suffices; latent depth is what keeps HBM busy (5 slots with a single P
    // buffer beat 4 with two).
    if (fits(5, 1, 1)) { lat_slots = 5; rope_slots = 1; p_slots = 1; }
    else { rope_slots = 2; lat_slots = (kSmemBudget - fixed(2) - 2 * L::kRopeBytes) / L::kLatBytes; }
  } else if (p.SUB == 1) {
    // one branch: every round consumes a latent and a rope sub-block -> equal ring depths
    for (int d = 6; d >= 2; --d)
      if (fits(d, d, 2)) { lat_slots = rope_slots = d; break; }
  } else {
    // multi-block latent (MLA, 64-token tiles): 2*SUB resident + 1 in flight at least
    rope_slots = T == 64 ? 3 : 2;
    for (;; --rope_slots) {
      lat_slots = (kSmemBudget - fixed(2) - rope_slots * L::kRopeBytes) / L::kLatBytes;
      if (lat_slots >= 2 * p.SUB + 2 || rope_slots == 2) break;
    }
  }
  if (!GQA && lat_slots < 2 * p.SUB + 1)
    return fail(MLRA_ERR_CONFIG, "decode: latent ring of %d slots cannot hold 2*SUB+1=%d sub-blocks", lat_slots,
                2 * p.SUB + 1);
  if (lat_slots > mlra::kMaxLat) lat_slots = mlra::kMaxLat;
  if (rope_slots > mlra::kMaxRope) rope_slots = mlra::kMaxRope;
  if (const char* e = getenv("MLRA_DEBUG_RING")) {  // dev: "lat,rope,p"
    int a = 0, b = 0, c = 0;
    if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && fits(a, b, c)) { lat_slots = a; rope_slots = b; p_slots = c; }
  }
  p.lat_slots = lat_slots;
  p.rope_slots = rope_slots;
  p.p_slots = p_slots;
  const int smem = L::smem_bytes(NB, p.SUB, lat_slots, rope_slots, p_slots);
  if (smem > kSmemBudget) return fail(MLRA_ERR_CONFIG, "decode: smem %d exceeds budget", smem);
  auto kern = mlra::mlra_decode_kernel<T, NPAD, DLS, NB, GQA>;
  static unsigned attr_done = 0;  // per instantiation, one bit per device
  if (int rc = set_smem_once(kern, attr_done, kSmemBudget)) return rc;
  if (p.fused == 2) {
    // cluster step: the nsplit CTAs of a sequence form one cluster; every cluster resident at once
    const bool dbg = getenv("MLRA_DEBUG_FUSE") != nullptr;
    if (GQA || NB != 1 || head_groups != 1 || p.nsplit > 16 || p.nsplit < 2) {
      if (dbg) fprintf(stderr, "cluster step: shape not eligible (NB=%d hgroups=%d nsplit=%d)\n", NB, head_groups, p.nsplit);
      return kNotFusable;
    }
    const int heads = mlra::cluster_heads_per_cta(p.H, p.nsplit);
    if (mlra::cluster_epilogue_bytes(NPAD, p.SUB * DLS, p.fz.DH, heads) >
        size_t(lat_slots) * L::kLatBytes + size_t(rope_slots) * L::kRopeBytes) {
      if (dbg) fprintf(stderr, "cluster step: epilogue %zu B > ring %zu B\n",
                       mlra::cluster_epilogue_bytes(NPAD, p.SUB * DLS, p.fz.DH, heads),
                       size_t(lat_slots) * L::kLatBytes + size_t(rope_slots) * L::kRopeBytes);
      return kNotFusable;
    }
    static unsigned np_done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 32 || !(np_done & (1u << dev))) {
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return cuda_check("cudaFuncSetAttribute(non-portable cluster)");
      if (dev < 32) np_done |= 1u << dev;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.B, 1);
    cfg.blockDim = dim3(mlra::kNumThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.nsplit;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
      if (dbg) fprintf(stderr, "cluster step: occupancy query failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      cudaGetLastError();
      return kNotFusable;
    }
    if (dbg) fprintf(stderr, "cluster step: %d clusters of %d resident, %d needed\n", clusters, p.nsplit, p.B);
    if (clusters < p.B) return kNotFusable;  // one wave (the TP sum waits on every rank's clusters)
    p.hgroups = 1;
    p.fz.npad = NPAD;
    if (cudaLaunchKernelEx(&cfg, kern, lat_map, rope_map, p) != cudaSuccess)
      return cuda_check("mlra_decode_kernel (cluster step) launch");
    return cuda_check("mlra_decode_kernel (cluster step) launch");
  }
  if (p.fused) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, mlra::kNumThreads, smem);
    const long grid = long(p.nsplit) * p.B * head_groups;
    if (grid > long(num_sms()) * per_sm ||
        mlra::combine_smem_bytes(p.fz.DH, p.fz.DLAT) > size_t(lat_slots) * L::kLatBytes ||
        (p.fz.absorb && mlra::absorb_smem_bytes(p.fz.DH) > size_t(q_chunks) * L::kQChunkBytes + size_t(p_slots) * L::kPBytes))
      return kNotFusable;
    p.hgroups = head_groups;
    p.fz.npad = NPAD;
    p.fz.hgroups = head_groups;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = p.plan != nullptr ? dim3(p.plan_ctas, 1, head_groups) : dim3(p.nsplit, p.B, head_groups);
  cfg.blockDim = dim3(mlra::kNumThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, lat_map, rope_map, p) != cudaSuccess)
    return cuda_check("mlra_decode_kernel launch");
  return cuda_check("mlra_decode_kernel launch");
}

#define MLRA_DECODE_INSTANCES(X)                                                                  \
  X(128, 16, 128, 1, false) X(128, 32, 128, 1, false) X(128, 64, 128, 1, false)                  \
  X(128, 16, 128, 2, false) X(128, 32, 128, 2, false) X(128, 64, 128, 2, false)                  \
  X(128, 16, 128, 4, false) X(128, 32, 128, 4, false)                                            \
  X(64, 16, 128, 1, false) X(64, 32, 128, 1, false) X(64, 64, 128, 1, false)                     \
  X(128, 16, 64, 1, false) X(128, 32, 64, 1, false) X(128, 64, 64, 1, false)                     \
  X(128, 16, 64, 2, false) X(128, 32, 64, 2, false) X(128, 64, 64, 2, false)                     \
  X(128, 16, 64, 4, false) X(128, 32, 64, 4, false)                                              \
  X(64, 16, 64, 1, false) X(64, 32, 64, 1, false) X(64, 64, 64, 1, false)                        \
  X(128, 16, 128, 1, true) X(128, 16, 128, 2, true) X(128, 16, 128, 4, true)                     \
  X(128, 16, 64, 1, true) X(128, 16, 64, 2, true) X(128, 16, 64, 4, true)

#define MLRA_EXTERN_DECODE(T, NP, D, NB, G)                                                              \
  extern template int launch_decode<T, NP, D, NB, G>(const CUtensorMap&, const CUtensorMap&, mlra::DecodeParams, \
                                                     int, cudaStream_t);
#define MLRA_INSTANTIATE_DECODE(T, NP, D, NB, G)                                                  \
  template int launch_decode<T, NP, D, NB, G>(const CUtensorMap&, const CUtensorMap&, mlra::DecodeParams, int, \
                                              cudaStream_t);

}  // namespace mlra_host
