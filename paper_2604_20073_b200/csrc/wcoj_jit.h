// Per-plan WCOJ kernels compiled at run time (wcoj_jit.cu).
#pragma once

#include "common.cuh"

namespace srdl {

// The kernel specialised for the shape of plan P in MODE (wcoj_kernel.cuh
// instantiated with a generated constant shape), compiled with NVRTC on
// first use and cached per shape (in process and on disk), or nullptr when
// the JIT is disabled (SRDL_JIT=0) or unavailable — the caller then runs the
// generic instance of the plan's class. Thread-safe.
const void *jit_kernel(const srdl_plan *P, int mode);

}  // namespace srdl
