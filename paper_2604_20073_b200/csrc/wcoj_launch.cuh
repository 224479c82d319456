// Kernel instances and launch of one MODE (included by wcoj_mode{0,1,2}.cu):
// the generic kernels per plan class (shape read from the descriptor) and
// the dispatch to the per-plan kernel compiled at run time (wcoj_jit.cu).
#pragma once

#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "wcoj_jit.h"
#include "wcoj_kernel.cuh"

namespace srdl {

template <int MODE, int KIND>
__global__ void __launch_bounds__(kJoinWarps * 32, kMinBlocks)
    wcoj_kernel(const __grid_constant__ srdl_plan P, const __grid_constant__ srdl_exec X,
                const __grid_constant__ srdl_spec Q) {
    wcoj_body<MODE, KIND, DynShape>(P, X, Q);
}

static inline uint32_t env_u32(const char *name, uint32_t dflt) {
    const char *v = getenv(name);
    return v && *v ? (uint32_t)strtoul(v, nullptr, 10) : dflt;
}

static int plan_kind(const srdl_plan *P) {
    // SRDL_WCOJ_GENERAL=1 routes every plan through the general instance
    // (tests cover both; also an A/B knob for the specialisation)
    if (env_u32("SRDL_WCOJ_GENERAL", 0)) return kGeneral;
    return plan_class(P->depth, P->nmid);
}

static size_t block_bytes(const srdl_plan *P) {
    const uint32_t NL = P->nspec[P->depth - 1] ? P->nspec[P->depth - 1] : 1;
    return warp_bytes(P->depth, P->natoms, NL, P->nmid) * kJoinWarps;
}

// One full wave of resident blocks (the plan's shared-memory footprint and
// the register budget decide how many fit per SM); slices are fetched
// dynamically, so more blocks would only queue. The slice geometry
// (X->nwarps, nslices, min_units) comes from the caller and is identical
// for the count and the materialize launch; the grid is only how many warps
// fetch those slices, so it never feeds into the slicing.
// (memoised per kernel, shared-memory size and device: the occupancy query
// is a driver call on every one of ~1,000 launches per DOOP fixpoint)
static unsigned wave_blocks(const void *fn, size_t bytes) {
    struct Key {
        const void *fn;
        size_t bytes;
        int dev;
        bool operator==(const Key &o) const { return fn == o.fn && bytes == o.bytes && dev == o.dev; }
    };
    struct KeyHash {
        size_t operator()(const Key &k) const {
            return std::hash<const void *>()(k.fn) ^ (k.bytes * 0x9e3779b97f4a7c15ull) ^ (size_t)k.dev;
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, unsigned, KeyHash> memo;
    int dev = 0;
    SRDL_CUDA(cudaGetDevice(&dev));
    const Key key{fn, bytes, dev};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
    }
    int per_sm = 0;
    SRDL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kJoinWarps * 32, bytes));
    if (per_sm < 1) per_sm = 1;
    const unsigned blocks = (unsigned)(per_sm * sm_count());
    std::lock_guard<std::mutex> lock(mu);
    memo[key] = blocks;
    return blocks;
}

template <int MODE, int KIND>
static void launch_kind(const srdl_plan *P, const srdl_exec *X, const srdl_spec *Q, cudaStream_t s) {
    const size_t bytes = block_bytes(P);
    static uint64_t raised = 0;
    if (first_use_on_device(&raised)) {  // allow up to the full 227 KB of dynamic shared memory
        SRDL_CUDA(cudaFuncSetAttribute(wcoj_kernel<MODE, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
    }
    SRDL_REQUIRE(bytes <= 227 * 1024, "join state of %zu bytes per block exceeds shared memory", bytes);
    const unsigned blocks = wave_blocks((const void *)wcoj_kernel<MODE, KIND>, bytes);
    wcoj_kernel<MODE, KIND><<<blocks, kJoinWarps * 32, bytes, s>>>(*P, *X, *Q);
}

template <int MODE>
void launch(const srdl_plan *P, const srdl_exec *X, const srdl_spec *Q, cudaStream_t s) {
    srdl_spec none{};
    if (!Q) Q = &none;
    const size_t bytes = block_bytes(P);
    SRDL_REQUIRE(bytes <= 227 * 1024, "join state of %zu bytes per block exceeds shared memory", bytes);
    // the plan's own kernel (compiled once per plan shape) when available
    if (!env_u32("SRDL_WCOJ_GENERAL", 0)) {
        const void *fn = jit_kernel(P, MODE);
        if (fn) {
            const unsigned blocks = wave_blocks(fn, bytes);
            void *args[] = {(void *)P, (void *)X, (void *)Q};
            SRDL_CUDA(cudaLaunchKernel(fn, dim3(blocks), dim3(kJoinWarps * 32), args, bytes, s));
            return;
        }
    }
    switch (plan_kind(P)) {
        case kShallow:
            launch_kind<MODE, kShallow>(P, X, Q, s);
            break;
        case kDepth3:
            launch_kind<MODE, kDepth3>(P, X, Q, s);
            break;
        case kDepth4Mid:
            launch_kind<MODE, kDepth4Mid>(P, X, Q, s);
            break;
        default:
            launch_kind<MODE, kGeneral>(P, X, Q, s);
    }
}

}  // namespace srdl
