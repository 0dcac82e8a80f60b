// K2 instantiations: 128-token tiles, 128-wide latent sub-blocks (2.9B MLRA-4 / MLRA-2, TP1..TP4).
// (One translation unit per group so the library builds in parallel; see host_common.cuh.)
#include "host_common.cuh"

namespace mlra_host {
MLRA_INSTANTIATE_DECODE(128, 16, 128, 1, false) MLRA_INSTANTIATE_DECODE(128, 32, 128, 1, false) MLRA_INSTANTIATE_DECODE(128, 64, 128, 1, false)
MLRA_INSTANTIATE_DECODE(128, 16, 128, 2, false) MLRA_INSTANTIATE_DECODE(128, 32, 128, 2, false) MLRA_INSTANTIATE_DECODE(128, 64, 128, 2, false)
MLRA_INSTANTIATE_DECODE(128, 16, 128, 4, false) MLRA_INSTANTIATE_DECODE(128, 32, 128, 4, false)
}  // namespace mlra_host
