// WCOJ kernel instances of mode kMaterialize (one translation unit per mode so
// the build compiles the instances in parallel).
#include "wcoj_launch.cuh"

namespace srdl {
template void launch<kMaterialize>(const srdl_plan *, const srdl_exec *, const srdl_spec *, cudaStream_t);
}  // namespace srdl
