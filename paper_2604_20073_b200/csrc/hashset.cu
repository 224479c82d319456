// Compute Delta through a device hash set of the full relation (paper Fig. 1
// "Compute Delta"; reference storage.compute_delta, storage.py:311-324:
// sort_dedup(new) minus full).
//
// The staged output of an iteration is several times larger than the delta
// it yields (TC: 493 M staged rows for 98.6 M new ones over a fixpoint):
// sorting all of it and then anti-joining against the sorted full relation
// pays radix passes for rows that are already known. Here every staged row
// (packed into one 64-bit key) first probes an open-addressing hash set of
// the full relation's keys — one 32-byte sector per probe — and only the
// rows not found are compacted, radix-sorted and deduplicated. The set is
// maintained incrementally: each iteration's delta is inserted after the
// merge, so its cost is proportional to the delta, not to the relation.
//
// Layout: `slots` holds 2^log2cap u64 keys, kEmpty marks a free slot; keys
// are rows packed column 0 first with `bits` bits per column (the layout of
// the radix sort), so they are < 2^(arity*bits) <= 2^64 - 1 and never equal
// kEmpty. Linear probing from a multiplicative hash.
#include "common.cuh"

namespace srdl {

constexpr uint64_t kEmpty = ~0ull;

__device__ __forceinline__ uint64_t hslot(uint64_t k, uint32_t log2cap) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return k >> (64 - log2cap);
}

__device__ __forceinline__ uint64_t pack_row_at(const Cols &c, uint64_t i, uint32_t arity, uint32_t bits) {
    uint64_t k = 0;
    for (uint32_t q = 0; q < arity; ++q) k = (k << bits) | __ldg(c.c[q] + i);
    return k;
}

__global__ void hset_insert_rows(Cols rows, uint32_t arity, uint32_t bits, uint64_t n, uint64_t *slots,
                                 uint32_t log2cap) {
    const uint64_t mask = (1ull << log2cap) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = pack_row_at(rows, i, arity, bits);
        uint64_t h = hslot(k, log2cap);
        while (true) {
            const unsigned long long prev =
                atomicCAS((unsigned long long *)(slots + h), (unsigned long long)kEmpty, (unsigned long long)k);
            if (prev == kEmpty || prev == k) break;
            h = (h + 1) & mask;
        }
    }
}

// keys of the staged rows not in the set, compacted (order not kept: the
// survivors are radix-sorted next); *nkeep counts them
__global__ void hset_filter_rows(Cols rows, uint32_t arity, uint32_t bits, uint64_t n, const uint64_t *__restrict__ slots,
                                 uint32_t log2cap, uint64_t *__restrict__ keys, uint32_t *__restrict__ nkeep) {
    const uint64_t mask = (1ull << log2cap) - 1;
    const uint32_t l = threadIdx.x & 31;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < n; base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        bool keep = false;
        uint64_t k = 0;
        if (i < n) {
            k = pack_row_at(rows, i, arity, bits);
            uint64_t h = hslot(k, log2cap);
            while (true) {
                const uint64_t v = __ldg(slots + h);
                if (v == k) break;
                if (v == kEmpty) {
                    keep = true;
                    break;
                }
                h = (h + 1) & mask;
            }
        }
        // warp-aggregated compaction: one atomic per warp
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        uint32_t at = 0;
        if (l == 0 && m) at = atomicAdd(nkeep, (uint32_t)__popc(m));
        at = __shfl_sync(0xffffffffu, at, 0);
        if (keep) keys[at + __popc(m & ((1u << l) - 1u))] = k;
    }
}

__global__ void flag_distinct(const uint64_t *__restrict__ keys, uint64_t n, uint32_t *__restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        keep[i] = (i == 0) || __ldg(keys + i - 1) != __ldg(keys + i);
}

__global__ void unpack_kept(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ keep,
                            const uint32_t *__restrict__ pos, uint64_t n, uint32_t arity, uint32_t bits,
                            MutCols out) {
    const uint64_t mask = bits >= 32 ? 0xffffffffull : ((1ull << bits) - 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        uint64_t k = keys[i];
        const uint32_t p = pos[i];
        for (int c = (int)arity - 1; c >= 0; --c) {
            out.c[c][p] = (uint32_t)(k & mask);
            k >>= bits;
        }
    }
}

}  // namespace srdl

using namespace srdl;

extern "C" {

int srdl_hset_insert(uint64_t *slots, uint32_t log2cap, const uint32_t *const *cols, uint32_t arity, uint64_t n,
                     uint32_t bits, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(log2cap >= 4 && log2cap <= 40, "hash set capacity 2^%u", log2cap);
        SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS && bits >= 1 && arity * bits <= 63,
                     "hash set keys: %u columns of %u bits", arity, bits);
        if (n == 0) return;
        hset_insert_rows<<<stride_grid(n), kThreads, 0, (cudaStream_t)stream>>>(make_cols(cols, arity), arity, bits,
                                                                              n, slots, log2cap);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_hset_filter(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits, const uint64_t *slots,
                     uint32_t log2cap, uint64_t *keys_out, uint32_t *count_dev, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(log2cap >= 4 && log2cap <= 40, "hash set capacity 2^%u", log2cap);
        SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS && bits >= 1 && arity * bits <= 63,
                     "hash set keys: %u columns of %u bits", arity, bits);
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_CUDA(cudaMemsetAsync(count_dev, 0, sizeof(uint32_t), s));
        if (n == 0) return;
        SRDL_REQUIRE(n < (1ull << 32), "hset_filter: %llu rows exceeds 2^32", (unsigned long long)n);
        hset_filter_rows<<<stride_grid(n), kThreads, 0, s>>>(make_cols(cols, arity), arity, bits, n, slots, log2cap,
                                                            keys_out, count_dev);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_sort_unique_keys(uint64_t *keys, uint64_t m, uint32_t arity, uint32_t bits, uint32_t *const *out,
                          uint32_t *count_dev, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS && bits >= 1 && arity * bits <= 64,
                     "keys: %u columns of %u bits", arity, bits);
        cudaStream_t s = (cudaStream_t)stream;
        if (m == 0) {
            SRDL_CUDA(cudaMemsetAsync(count_dev, 0, sizeof(uint32_t), s));
            return;
        }
        SRDL_REQUIRE(m < (1ull << 32), "sort_unique_keys: %llu keys exceeds 2^32", (unsigned long long)m);
        radix_sort(keys, nullptr, m, arity * bits, s);
        Scratch keep(m * sizeof(uint32_t), s), pos(m * sizeof(uint32_t), s);
        const unsigned g = stride_grid(m);
        flag_distinct<<<g, kThreads, 0, s>>>(keys, m, keep.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u32(keep.as<uint32_t>(), pos.as<uint32_t>(), m, count_dev, s);
        unpack_kept<<<g, kThreads, 0, s>>>(keys, keep.as<uint32_t>(), pos.as<uint32_t>(), m, arity, bits,
                                           make_mut(out, arity));
        SRDL_CHECK_LAUNCH();
    });
}

}  // extern "C"
