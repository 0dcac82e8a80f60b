// K2 instantiations: the GQA comparison variant.
// (One translation unit per group so the library builds in parallel; see host_common.cuh.)
#include "host_common.cuh"

namespace mlra_host {
MLRA_INSTANTIATE_DECODE(128, 16, 128, 1, true) MLRA_INSTANTIATE_DECODE(128, 16, 128, 2, true) MLRA_INSTANTIATE_DECODE(128, 16, 128, 4, true)
MLRA_INSTANTIATE_DECODE(128, 16, 64, 1, true) MLRA_INSTANTIATE_DECODE(128, 16, 64, 2, true) MLRA_INSTANTIATE_DECODE(128, 16, 64, 4, true)
}  // namespace mlra_host
