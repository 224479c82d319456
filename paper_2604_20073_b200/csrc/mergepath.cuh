// Merge path over sorted row sets (Green, McColl & Bader, "GPU merge path").
// Thread t owns output diagonals [t*kMergeItems, (t+1)*kMergeItems) of the
// stable merge of A and B (A first on ties): one binary search finds where
// its window starts, then it merges sequentially. Linear total work and
// near-coalesced reads, used for
//   * the head/body flush and head merges (merge of disjoint sets), and
//   * the anti-join of compute_delta (membership of every staged row in a
//     full segment), replacing per-row binary searches.
#pragma once

#include "common.cuh"

namespace srdl {

constexpr int kMergeItems = 32;

// Rows of a segment read as packed keys (same layout as the staged keys).
struct PackedRows {
    Cols c;
    uint32_t arity, bits;
    __device__ __forceinline__ uint64_t operator[](uint64_t j) const {
        uint64_t k = 0;
        for (uint32_t q = 0; q < arity; ++q) k = (k << bits) | __ldg(c.c[q] + j);
        return k;
    }
};

// number of A elements among the first d outputs (A[i] <= B[j] takes A)
template <class LE>
__device__ __forceinline__ uint64_t mp_split(uint64_t d, uint64_t na, uint64_t nb, const LE &le) {
    uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (le(mid, d - 1 - mid))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Merge two sorted row sets (ties: A first) into out.
static __global__ void mp_merge_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity, MutCols out) {
    const uint64_t n = na + nb;
    auto le = [&](uint64_t i, uint64_t j) { return row_cmp(A, i, B, j, arity) <= 0; };
    for (uint64_t d0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kMergeItems; d0 < n;
         d0 += (uint64_t)gridDim.x * blockDim.x * kMergeItems) {
        uint64_t i = mp_split(d0, na, nb, le), j = d0 - i;
        const uint64_t end = d0 + kMergeItems < n ? d0 + kMergeItems : n;
        for (uint64_t d = d0; d < end; ++d) {
            const bool take_a = j >= nb || (i < na && le(i, j));
            const Cols &src = take_a ? A : B;
            const uint64_t row = take_a ? i++ : j++;
            for (uint32_t c = 0; c < arity; ++c) out.c[c][d] = __ldg(src.c[c] + row);
        }
    }
}

// keep[i] = 0 for every staged key present in the packed segment B.
static __global__ void mp_diff_keys(const uint64_t *__restrict__ keys, uint64_t na, PackedRows B, uint64_t nb,
                             uint32_t *__restrict__ keep) {
    const uint64_t n = na + nb;
    auto le = [&](uint64_t i, uint64_t j) { return keys[i] <= B[j]; };
    for (uint64_t d0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kMergeItems; d0 < n;
         d0 += (uint64_t)gridDim.x * blockDim.x * kMergeItems) {
        uint64_t i = mp_split(d0, na, nb, le), j = d0 - i;
        const uint64_t end = d0 + kMergeItems < n ? d0 + kMergeItems : n;
        uint64_t bj = j < nb ? B[j] : ~0ull;
        for (uint64_t d = d0; d < end; ++d) {
            if (i < na && (j >= nb || keys[i] <= bj)) {
                if (j < nb && keys[i] == bj) keep[i] = 0;
                ++i;
            } else {
                ++j;
                bj = j < nb ? B[j] : ~0ull;
            }
        }
    }
}

// keep[i] = 0 for every staged row of A present in segment B (row compare).
static __global__ void mp_diff_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity,
                             uint32_t *__restrict__ keep) {
    const uint64_t n = na + nb;
    auto le = [&](uint64_t i, uint64_t j) { return row_cmp(A, i, B, j, arity) <= 0; };
    for (uint64_t d0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * kMergeItems; d0 < n;
         d0 += (uint64_t)gridDim.x * blockDim.x * kMergeItems) {
        uint64_t i = mp_split(d0, na, nb, le), j = d0 - i;
        const uint64_t end = d0 + kMergeItems < n ? d0 + kMergeItems : n;
        for (uint64_t d = d0; d < end; ++d) {
            int c = (i < na && j < nb) ? row_cmp(A, i, B, j, arity) : (i < na ? -1 : 1);
            if (c <= 0) {
                if (c == 0) keep[i] = 0;
                ++i;
            } else {
                ++j;
            }
        }
    }
}

inline unsigned mp_grid(uint64_t n) {
    uint64_t threads = (n + kMergeItems - 1) / kMergeItems;
    return stride_grid(threads);
}

}  // namespace srdl
