// K2 instantiations: 128-token tiles, 64-wide latent sub-blocks (small head widths).
// (One translation unit per group so the library builds in parallel; see host_common.cuh.)
#include "host_common.cuh"

namespace mlra_host {
MLRA_INSTANTIATE_DECODE(128, 16, 64, 1, false) MLRA_INSTANTIATE_DECODE(128, 32, 64, 1, false) MLRA_INSTANTIATE_DECODE(128, 64, 64, 1, false)
MLRA_INSTANTIATE_DECODE(128, 16, 64, 2, false) MLRA_INSTANTIATE_DECODE(128, 32, 64, 2, false) MLRA_INSTANTIATE_DECODE(128, 64, 64, 2, false)
MLRA_INSTANTIATE_DECODE(128, 16, 64, 4, false) MLRA_INSTANTIATE_DECODE(128, 32, 64, 4, false)
}  // namespace mlra_host
