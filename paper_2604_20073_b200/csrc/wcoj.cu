// Host side of the WCOJ join (paper Alg. 1 phases 2-3, Alg. 2; reference
// executor.count_pass / materialize_pass, executor.py:439-485): the generic
// kernel instances (one per plan class, the plan shape read from the
// descriptor), the per-plan kernels compiled at run time (wcoj_jit.cu), the
// launch geometry, the arena gather, and the C ABI. The device code is in
// wcoj_kernel.cuh.
#include <stdlib.h>

#include "wcoj_kernel.cuh"

namespace srdl {

// the launch of one mode: generic instances + per-plan kernels
// (wcoj_launch.cuh, instantiated in wcoj_mode{0,1,2}.cu, one TU per mode so
// the build compiles them in parallel)
template <int MODE>
void launch(const srdl_plan *P, const srdl_exec *X, const srdl_spec *Q, cudaStream_t s);
extern template void launch<kCount>(const srdl_plan *, const srdl_exec *, const srdl_spec *, cudaStream_t);
extern template void launch<kMaterialize>(const srdl_plan *, const srdl_exec *, const srdl_spec *, cudaStream_t);
extern template void launch<kSpec>(const srdl_plan *, const srdl_exec *, const srdl_spec *, cudaStream_t);

// Warp per slice: copy the slice's chunk chain to its exact output offset.
__global__ void __launch_bounds__(256) gather_kernel(const srdl_exec X, const srdl_spec Q, uint32_t arity,
                                                     uint32_t nslices) {
    const uint32_t l = lane_id();
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    // only the slices the count walk used can hold tuples
    const uint64_t T = X.nkeys ? X.prefix[X.nkeys - 1] : 0;
    const uint32_t used = (uint32_t)slices_used(X, T);
    if (nslices > used) nslices = used;
    for (uint32_t sl = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sl < nslices; sl += warps) {
        const uint64_t n = X.slice_counts[sl];
        if (n == 0 || Q.slice_spill[sl]) continue;
        uint64_t off = X.slice_offsets[sl];
        uint32_t c = Q.slice_first[sl];
        uint64_t left = n;
        while (true) {
            const uint32_t take = left < Q.chunk ? (uint32_t)left : Q.chunk;
            const uint64_t src = (uint64_t)c * Q.chunk;
            // the next link is loaded before the copy so its latency overlaps
            const uint32_t nxt = left > take ? __ldg(Q.chunk_next + c) : 0u;
            for (uint32_t h = 0; h < arity; ++h) {
                const uint32_t *__restrict__ in = Q.cols[h] + src;
                uint32_t *__restrict__ out = X.out[h] + off;
                // four loads in flight per lane before the stores
                for (uint32_t i = l; i < take; i += 128) {
                    uint32_t v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = i + 32 * u < take ? __ldcs(in + i + 32 * u) : 0u;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (i + 32 * u < take) __stcs(out + i + 32 * u, v[u]);
                }
            }
            left -= take;
            off += take;
            if (left == 0) break;
            c = nxt;
        }
    }
}

// Count prologue (one launch instead of four or five memsets over the whole
// slice capacity): zero the slice ticket and the arena cursor / spill count,
// compute the number of slices this launch uses (slices_used of the root
// work total) into *used, and zero only those slices' counts and spill
// flags — every reader (scan, gather, materialize) stops at the same bound.
__global__ void __launch_bounds__(256) count_prologue(const srdl_exec X, const srdl_spec Q, int spec,
                                                      uint64_t *used_out) {
    const uint64_t T = X.nkeys ? X.prefix[X.nkeys - 1] : 0;
    const uint64_t used = slices_used(X, T);
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i0 == 0) {
        *X.ticket = 0;
        *used_out = used;
        if (spec) {
            *Q.cursor = 0;
            *Q.spills = 0;
        }
    }
    for (uint64_t i = i0; i < used; i += (uint64_t)gridDim.x * blockDim.x) {
        X.slice_counts[i] = 0;
        if (spec) Q.slice_spill[i] = 0;
    }
}

static void count_prologue_launch(const srdl_exec *X, const srdl_spec *Q, uint64_t *used, cudaStream_t s) {
    const unsigned blocks = (unsigned)((X->nslices + 255) / 256 < (uint64_t)sm_count() * 4
                                           ? (X->nslices + 255) / 256 : (uint64_t)sm_count() * 4);
    srdl_spec none{};
    count_prologue<<<blocks, 256, 0, s>>>(*X, Q ? *Q : none, Q != nullptr, used);
    SRDL_CHECK_LAUNCH();
}

static void check_spec(const srdl_plan *P, const srdl_spec *Q) {
    SRDL_REQUIRE(Q != nullptr, "a speculative arena is required");
    SRDL_REQUIRE(Q->chunk >= 32 && (Q->chunk & (Q->chunk - 1)) == 0, "chunk %u: power of two >= 32", Q->chunk);
    SRDL_REQUIRE(Q->cursor && Q->spills && Q->slice_first && Q->slice_spill, "arena bookkeeping arrays missing");
    SRDL_REQUIRE(Q->nchunks == 0 || Q->chunk_next, "chunk links missing");
    for (uint32_t h = 0; h < P->head_arity && Q->nchunks; ++h)
        SRDL_REQUIRE(Q->cols[h] != nullptr, "arena column %u missing", h);
}

static void check_plan(const srdl_plan *P, const srdl_exec *X) {
    SRDL_REQUIRE(P->depth >= 1 && P->depth <= SRDL_MAX_LEVELS, "plan depth %u unsupported", P->depth);
    SRDL_REQUIRE(P->natoms >= 1 && P->natoms <= SRDL_MAX_ATOMS, "plan has %u atoms", P->natoms);
    SRDL_REQUIRE(P->head_arity <= SRDL_MAX_HEAD, "head arity %u", P->head_arity);
    SRDL_REQUIRE(P->nspec[P->depth - 1] <= SRDL_MAX_LEAF_SPECS, "leaf level has %u sources (max %d)",
                 P->nspec[P->depth - 1], SRDL_MAX_LEAF_SPECS);
    SRDL_REQUIRE(X->nwarps >= 1 && X->nslices >= 1, "nwarps and nslices must be >= 1");
    SRDL_REQUIRE(X->ticket != nullptr, "a slice ticket counter is required");
    SRDL_REQUIRE(X->min_units >= 1, "min_units must be >= 1");
}

}  // namespace srdl

using namespace srdl;

extern "C" {

int srdl_wcoj_count(const srdl_plan *plan, const srdl_exec *ex, void *stream) {
    return guarded([&] {
        check_plan(plan, ex);
        cudaStream_t s = (cudaStream_t)stream;
        Scratch used(sizeof(uint64_t), s);
        count_prologue_launch(ex, nullptr, used.as<uint64_t>(), s);
        launch<kCount>(plan, ex, nullptr, s);
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u64_bounded(ex->slice_counts, ex->slice_offsets, ex->nslices, used.as<uint64_t>(),
                                   ex->total, s);
    });
}

int srdl_wcoj_count_spec(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec, void *stream) {
    return guarded([&] {
        check_plan(plan, ex);
        check_spec(plan, spec);
        cudaStream_t s = (cudaStream_t)stream;
        Scratch used(sizeof(uint64_t), s);
        count_prologue_launch(ex, spec, used.as<uint64_t>(), s);
        launch<kSpec>(plan, ex, spec, s);
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u64_bounded(ex->slice_counts, ex->slice_offsets, ex->nslices, used.as<uint64_t>(),
                                   ex->total, s);
    });
}

int srdl_wcoj_gather(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec, void *stream) {
    return guarded([&] {
        check_plan(plan, ex);
        check_spec(plan, spec);
        const unsigned blocks = (unsigned)(sm_count() * 8);
        gather_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*ex, *spec, plan->head_arity, ex->nslices);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_wcoj_materialize_spilled(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec,
                                  void *stream) {
    return guarded([&] {
        check_plan(plan, ex);
        check_spec(plan, spec);
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_CUDA(cudaMemsetAsync(ex->ticket, 0, sizeof(uint32_t), s));
        launch<kMaterialize>(plan, ex, spec, s);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_wcoj_materialize(const srdl_plan *plan, const srdl_exec *ex, void *stream) {
    return guarded([&] {
        check_plan(plan, ex);
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_CUDA(cudaMemsetAsync(ex->ticket, 0, sizeof(uint32_t), s));
        launch<kMaterialize>(plan, ex, nullptr, s);
        SRDL_CHECK_LAUNCH();
    });
}

}  // extern "C"
