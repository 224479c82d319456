// Merge path over sorted row sets (Green, McColl & Bader, "GPU merge path"),
// block-tiled. Block b owns output diagonals [b*kMT, (b+1)*kMT) of the
// stable merge of A and B (A first on ties): thread 0 finds where the tile
// starts and ends in A with two binary searches, the block loads both input
// tiles into shared memory with coalesced reads, and each thread merges
// kMI consecutive outputs from shared memory. Linear work, one global read
// of every input element, coalesced writes. Used for
//   * the head/body flush and head merges (merge of disjoint row sets), and
//   * the anti-join of compute_delta (membership of every staged row in a
//     full segment), replacing per-row binary searches.
#pragma once

#include "common.cuh"

namespace srdl {

constexpr int kMI = 4;                 // outputs per thread
constexpr int kMT = kThreads * kMI;    // outputs per block tile (1024)
constexpr int kMTS = kMT + 1;          // tile stride: + one B sentinel past the tile

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

// Tile splits for every block, computed by a separate fully parallel
// kernel (one thread per tile boundary): splits[t] = A elements among the
// first t*kMT outputs, t in [0, tiles].
template <class LE>
__device__ __forceinline__ void split_all(uint64_t na, uint64_t nb, const LE &le, uint64_t *splits) {
    const uint64_t n = na + nb, tiles = (n + kMT - 1) / kMT;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t <= tiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = t * kMT < n ? t * kMT : n;
        splits[t] = mp_split(d, na, nb, le);
    }
}

static __global__ void mp_splits_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity,
                                      uint64_t *splits) {
    split_all(na, nb, [&](uint64_t i, uint64_t j) { return row_cmp(A, i, B, j, arity) <= 0; }, splits);
}



// Tile bounds of this block from the precomputed splits.
__device__ __forceinline__ void tile_bounds(uint64_t na, uint64_t nb, const uint64_t *splits,
                                            uint64_t *sh) {
    if (threadIdx.x == 0) {
        const uint64_t n = na + nb, d0 = (uint64_t)blockIdx.x * kMT;
        sh[0] = splits[blockIdx.x];
        sh[1] = splits[blockIdx.x + 1];
        sh[2] = d0;
        sh[3] = d0 + kMT < n ? d0 + kMT : n;
    }
    __syncthreads();
}

// smem layout for row tiles: column c of tile row k at s[c * kMTS + k];
// A rows at [0, ta), B rows at [ta, ta + tb), and for the anti-join the B
// row following the tile at ta + tb (a staged row equal to it is the last A
// element before the tile boundary and must still be recognised)
__device__ __forceinline__ int smem_row_cmp(const uint32_t *s, uint32_t x, uint32_t y, uint32_t arity) {
    for (uint32_t c = 0; c < arity; ++c) {
        const uint32_t u = s[c * kMTS + x], v = s[c * kMTS + y];
        if (u != v) return u < v ? -1 : 1;
    }
    return 0;
}

// Merge two sorted row sets (ties: A first) into out. Dynamic smem: arity*kMTS*4.
static __global__ void __launch_bounds__(kThreads)
    mp_merge_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity, const uint64_t *splits,
                  MutCols out) {
    extern __shared__ uint32_t tile[];
    __shared__ uint64_t sh[4];
    tile_bounds(na, nb, splits, sh);
    const uint64_t a0 = sh[0], a1 = sh[1], d0 = sh[2], d1 = sh[3];
    const uint32_t ta = (uint32_t)(a1 - a0), tb = (uint32_t)((d1 - d0) - ta);
    const uint64_t b0 = d0 - a0;
    for (uint32_t c = 0; c < arity; ++c) {
        for (uint32_t k = threadIdx.x; k < ta + tb; k += kThreads)
            tile[c * kMTS + k] = k < ta ? __ldg(A.c[c] + a0 + k) : __ldg(B.c[c] + b0 + (k - ta));
    }
    __syncthreads();
    const uint32_t k0 = threadIdx.x * kMI < ta + tb ? threadIdx.x * kMI : ta + tb;  // idle: empty range
    // split of this thread's diagonal inside the tile
    uint32_t lo = k0 > tb ? k0 - tb : 0, hi = k0 < ta ? k0 : ta;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (smem_row_cmp(tile, mid, ta + (k0 - 1 - mid), arity) <= 0)
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = k0 - lo;
    const uint32_t kend = k0 + kMI < ta + tb ? k0 + kMI : ta + tb;
    uint32_t src[kMI];
    for (uint32_t k = k0; k < kend; ++k) {
        const bool take_a = j >= tb || (i < ta && smem_row_cmp(tile, i, ta + j, arity) <= 0);
        src[k - k0] = take_a ? i++ : ta + j++;
    }
    // stage the merged tile column by column in shared memory (the source
    // slots are overwritten only after every thread picked its rows), then
    // store each column with coalesced writes
    uint32_t vals[kMI];
    for (uint32_t c = 0; c < arity; ++c) {
        for (uint32_t k = k0; k < kend; ++k) vals[k - k0] = tile[c * kMTS + src[k - k0]];
        __syncthreads();
        for (uint32_t k = k0; k < kend; ++k) tile[c * kMTS + k] = vals[k - k0];
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < ta + tb; k += kThreads) out.c[c][d0 + k] = tile[c * kMTS + k];
    }
}

// keep[i] = 0 for every staged key present in the packed segment B.
static __global__ void __launch_bounds__(kThreads)
    mp_diff_keys(const uint64_t *__restrict__ keys, uint64_t na, PackedRows B, uint64_t nb,
                 const uint64_t *splits, uint32_t *__restrict__ keep) {
    __shared__ uint64_t tile[kMTS];
    __shared__ uint64_t sh[4];
    tile_bounds(na, nb, splits, sh);
    const uint64_t a0 = sh[0], a1 = sh[1], d0 = sh[2], d1 = sh[3];
    const uint32_t ta = (uint32_t)(a1 - a0), tb = (uint32_t)((d1 - d0) - ta);
    const uint64_t b0 = d0 - a0;
    for (uint32_t k = threadIdx.x; k <= ta + tb; k += kThreads) {
        if (k < ta)
            tile[k] = keys[a0 + k];
        else if (k < ta + tb || b0 + tb < nb)
            tile[k] = B[b0 + k - ta];  // k == ta + tb: sentinel B row after the tile
        else
            tile[k] = ~0ull;
    }
    __syncthreads();
    const uint32_t k0 = threadIdx.x * kMI;
    if (k0 >= ta + tb) return;
    uint32_t lo = k0 > tb ? k0 - tb : 0, hi = k0 < ta ? k0 : ta;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (tile[mid] <= tile[ta + (k0 - 1 - mid)])
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = k0 - lo;
    const uint32_t kend = k0 + kMI < ta + tb ? k0 + kMI : ta + tb;
    for (uint32_t k = k0; k < kend; ++k) {
        if (i < ta && (j >= tb || tile[i] <= tile[ta + j])) {
            if (tile[i] == tile[ta + j]) keep[a0 + i] = 0;  // j <= tb: sentinel included
            ++i;
        } else {
            ++j;
        }
    }
}

// keep[i] = 0 for every staged row of A present in segment B (row compare).
// Dynamic smem: arity*kMTS*4.
static __global__ void __launch_bounds__(kThreads)
    mp_diff_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity, const uint64_t *splits,
                 uint32_t *__restrict__ keep) {
    extern __shared__ uint32_t tile[];
    __shared__ uint64_t sh[4];
    tile_bounds(na, nb, splits, sh);
    const uint64_t a0 = sh[0], a1 = sh[1], d0 = sh[2], d1 = sh[3];
    const uint32_t ta = (uint32_t)(a1 - a0), tb = (uint32_t)((d1 - d0) - ta);
    const uint64_t b0 = d0 - a0;
    const bool sentinel = b0 + tb < nb;
    for (uint32_t c = 0; c < arity; ++c) {
        for (uint32_t k = threadIdx.x; k < ta + tb + (sentinel ? 1u : 0u); k += kThreads)
            tile[c * kMTS + k] = k < ta ? __ldg(A.c[c] + a0 + k) : __ldg(B.c[c] + b0 + (k - ta));
    }
    __syncthreads();
    const uint32_t k0 = threadIdx.x * kMI;
    if (k0 >= ta + tb) return;
    uint32_t lo = k0 > tb ? k0 - tb : 0, hi = k0 < ta ? k0 : ta;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (smem_row_cmp(tile, mid, ta + (k0 - 1 - mid), arity) <= 0)
            lo = mid + 1;
        else
            hi = mid;
    }
    uint32_t i = lo, j = k0 - lo;
    const uint32_t kend = k0 + kMI < ta + tb ? k0 + kMI : ta + tb;
    for (uint32_t k = k0; k < kend; ++k) {
        if (i < ta && (j >= tb || smem_row_cmp(tile, i, ta + j, arity) <= 0)) {
            // A step: member if equal to the current B row (j == tb is the
            // sentinel row after the tile, when there is one)
            if ((j < tb || sentinel) && smem_row_cmp(tile, i, ta + j, arity) == 0) keep[a0 + i] = 0;
            ++i;
        } else {
            ++j;
        }
    }
}

static __global__ void mp_splits_keys(const uint64_t *__restrict__ keys, uint64_t na, PackedRows B,
                                      uint64_t nb, uint64_t *splits) {
    split_all(na, nb, [&](uint64_t i, uint64_t j) { return keys[i] <= B[j]; }, splits);
}

inline unsigned mp_grid(uint64_t n) { return grid_for(n, kMT); }
inline uint64_t mp_tiles(uint64_t n) { return (n + kMT - 1) / kMT; }
inline size_t mp_smem(uint32_t arity) { return (size_t)arity * kMTS * sizeof(uint32_t); }

}  // namespace srdl
