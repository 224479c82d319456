// WCOJ kernel instances of mode kSpec (one translation unit per mode so
// the build compiles the instances in parallel).
#include "wcoj_launch.cuh"

namespace srdl {
template void launch<kSpec>(const srdl_plan *, const srdl_exec *, const srdl_spec *, cudaStream_t);
}  // namespace srdl
