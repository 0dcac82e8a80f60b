// K2 instantiations: 64-token tiles for multi-block latents (MLA, GLA-2 TP1).
// (One translation unit per group so the library builds in parallel; see host_common.cuh.)
#include "host_common.cuh"

namespace mlra_host {
MLRA_INSTANTIATE_DECODE(64, 16, 128, 1, false) MLRA_INSTANTIATE_DECODE(64, 32, 128, 1, false) MLRA_INSTANTIATE_DECODE(64, 64, 128, 1, false)
MLRA_INSTANTIATE_DECODE(64, 16, 64, 1, false) MLRA_INSTANTIATE_DECODE(64, 32, 64, 1, false) MLRA_INSTANTIATE_DECODE(64, 64, 64, 1, false)
}  // namespace mlra_host
