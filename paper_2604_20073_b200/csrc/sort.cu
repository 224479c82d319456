// Delta maintenance, part 1: LSD radix sort of packed tuples, unique, and the
// anti-join against the full relation (paper Fig. 1 "Compute Delta" /
// "Build Index"; reference storage.compute_delta, storage.py:311, and
// rowops.sort_dedup, rowops.py:60).
//
// Tuples of `arity` u32 ids with `bits` significant bits each are packed
// into u64 keys, column 0 most significant, so the numeric order of keys is
// the lexicographic order of rows. When arity*bits > 64 the columns are
// split into chunks of at most 64 bits, sorted least-significant chunk first
// with a stable radix sort carrying a row permutation.
#include "common.cuh"
#include "mergepath.cuh"

namespace srdl {

constexpr int kRadixBits = 8;
constexpr int kBins = 1 << kRadixBits;
constexpr int kWarps = kThreads / 32;
constexpr int kWarpChunk = 32 * kItems;
constexpr int kMaxPasses = 8;  // 64-bit keys
#ifndef SRDL_SORT_BACKOFF_DEFAULT
#define SRDL_SORT_BACKOFF_DEFAULT 0
#endif
#ifndef SRDL_SORT_ITEMS_DEFAULT
#define SRDL_SORT_ITEMS_DEFAULT 16
#endif
constexpr int kDefaultSortItems = SRDL_SORT_ITEMS_DEFAULT;


// Onesweep LSD radix sort (decoupled look-back, Merrill & Garland's single-
// pass prefix scan applied per digit): one histogram pass over the keys
// counts the digits of every pass at once; each pass then reads and writes
// every key exactly once — a tile ranks its keys, publishes its per-digit
// counts, looks back over the preceding tiles' published counts for its
// global offsets and scatters. Per pass: 8 B read + 8 B written per key
// (+ 4 + 4 B of row permutation), instead of the 8 + 8 + 8 B of a separate
// histogram read, and one launch instead of three.

// ghist[p * kBins + d] += number of keys whose pass-p digit is d
__global__ void __launch_bounds__(kThreads)
    radix_hist_all(const uint64_t *__restrict__ keys, uint64_t n, int passes, int lo_bit,
                   uint32_t *__restrict__ ghist, const int *__restrict__ unsorted) {
    if (unsorted && *unsorted == 0) return;  // input already in order: the sort is skipped
    __shared__ uint32_t h[kMaxPasses][kBins];
    for (int i = threadIdx.x; i < kMaxPasses * kBins; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    // four independent loads per thread and round (memory-level parallelism)
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < n; base += 4 * stride) {
        uint64_t k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) k[u] = base + u * stride < n ? __ldcs(keys + base + u * stride) : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (base + u * stride >= n) break;
            for (int p = 0; p < passes; ++p)
                atomicAdd(&h[p][(k[u] >> (lo_bit + p * kRadixBits)) & (kBins - 1)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kBins; i += kThreads) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(ghist + i, v);
    }
}

// per pass: exclusive scan of the digit counts (one warp per pass)
__global__ void radix_digit_starts(uint32_t *hist, int passes, const int *__restrict__ unsorted) {
    if (unsorted && *unsorted == 0) return;
    const int p = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (p >= passes) return;
    uint32_t *h = hist + p * kBins;
    uint32_t carry = 0;
    for (int base = 0; base < kBins; base += 32) {
        const uint32_t v = h[base + l];
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (l >= o) incl += y;
        }
        h[base + l] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// look-back status word per (tile, digit): flag in the top two bits, the
// pass's epoch in bits 32-61, the count in bits 0-31 (n < 2^32). The words
// persist across passes and sorts (onesweep_status): a word of an earlier
// pass carries another epoch and reads as "not published", so no pass
// clears them first.
constexpr uint64_t kFlagAgg = 1ull << 62;  // this tile's own count is published
constexpr uint64_t kFlagInc = 2ull << 62;  // inclusive prefix through this tile
constexpr uint64_t kValMask = 0xffffffffull;
constexpr uint64_t kEpochMask = (1ull << 30) - 1;

// Lanes of the warp holding the same digit as this lane (invalid lanes,
// digit kBins, group among themselves): one ballot per digit bit instead of
// __match_any_sync, which stalled the ranking loop (short_scoreboard 60 %).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, bool ok) {
    uint32_t peers = __ballot_sync(0xffffffffu, ok);
    if (!ok) peers = ~peers;
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
        const uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? m : ~m;
    }
    return peers;
}

// ITEMS keys per thread, a tile of kThreads * ITEMS keys. 16 items: 128
// registers, 2 blocks (25 % of the warp slots) per SM; 8 items: 4 blocks.
// ncu (TC, 113 M keys per pass, 16 items): issue-bound at 25 % occupancy
// (issue active 48 %, DRAM 20 % of peak, 169 instructions per key).
template <int ITEMS>
constexpr int onesweep_min_blocks() {
    return ITEMS >= 16 ? 2 : 4;
}

template <bool HAS_VALS, int ITEMS>
constexpr size_t onesweep_smem() {
    return (size_t)kThreads * ITEMS * 8 + (HAS_VALS ? (size_t)kThreads * ITEMS * 4 : 0) +
           (size_t)kWarps * kBins * 4 + (size_t)kBins * 8 + 64 * 4 + 16;
}

template <bool HAS_VALS, int ITEMS>
__global__ void __launch_bounds__(kThreads, onesweep_min_blocks<ITEMS>())
    onesweep_pass(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vals, uint64_t n, int shift,
                  const uint32_t *__restrict__ starts, uint64_t *status, uint64_t epoch, uint32_t *tile_ticket,
                  uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out,
                  const int *__restrict__ unsorted, uint32_t backoff_ns) {
    if (unsorted && *unsorted == 0) return;
    constexpr int kI = ITEMS;
    constexpr uint32_t kT = (uint32_t)kThreads * ITEMS;  // keys per tile
    extern __shared__ __align__(16) unsigned char sm[];
    uint64_t *skeys = (uint64_t *)sm;
    uint32_t *svals = (uint32_t *)(sm + (size_t)kT * 8);
    uint32_t(*cnt)[kBins] = (uint32_t(*)[kBins])(sm + (size_t)kT * 8 + (HAS_VALS ? (size_t)kT * 4 : 0));
    int64_t *gbase = (int64_t *)((unsigned char *)cnt + (size_t)kWarps * kBins * 4);
    uint32_t *wsum = (uint32_t *)(gbase + kBins);  // [kWarps] scan carries
    uint32_t *tile_slot = wsum + 64;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    // tiles are numbered in the order blocks start, so every tile a block
    // looks back on has started (forward progress of the look-back)
    if (threadIdx.x == 0) *tile_slot = atomicAdd(tile_ticket, 1u);
    for (int i = threadIdx.x; i < kWarps * kBins; i += kThreads) (&cnt[0][0])[i] = 0;
    __syncthreads();
    const uint64_t tile = *tile_slot;
    uint64_t k[kI];
    uint32_t v[kI];
    uint32_t rank[kI];
    const uint32_t lt = (1u << l) - 1u;
    // all of the thread's keys in flight at once (the ranking loop below
    // serialises on shared memory; loading inside it left one global load
    // outstanding per warp: 45 % of stall samples on the key's first use)
#pragma unroll
    for (int r = 0; r < kI; ++r) {
        const uint64_t i = (tile * kT + (uint64_t)w * (32 * kI) + r * 32 + l);
        k[r] = i < n ? __ldcs(keys + i) : 0;
        if (HAS_VALS) v[r] = i < n ? __ldcs(vals + i) : 0;
    }
#pragma unroll
    for (int r = 0; r < kI; ++r) {
        const uint64_t i = (tile * kT + (uint64_t)w * (32 * kI) + r * 32 + l);
        const bool ok = i < n;
        const uint32_t d = ok ? (uint32_t)((k[r] >> shift) & (kBins - 1)) : (uint32_t)kBins;
        const uint32_t peers = digit_peers(d, ok);
        uint32_t before = 0;
        if (ok) before = cnt[w][d];
        __syncwarp();
        if (ok && (peers & lt) == 0) cnt[w][d] = before + __popc(peers);
        __syncwarp();
        rank[r] = before + __popc(peers & lt);
    }
    __syncthreads();
    // digit d (one per thread, kThreads == kBins): per-warp exclusive offsets
    // within the digit, the tile's digit total, a block scan of the totals
    static_assert(kThreads == kBins, "one thread per digit");
    const int d = threadIdx.x;
    uint32_t total = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
        const uint32_t c = cnt[q][d];
        cnt[q][d] = total;
        total += c;
    }
    // publish this tile's count, then look back for the digit's prefix
    uint64_t *st = status + tile * kBins + d;
    const uint64_t stamp = epoch << 32;
    if (tile == 0) {
        *(volatile uint64_t *)st = kFlagInc | stamp | total;
    } else {
        *(volatile uint64_t *)st = kFlagAgg | stamp | total;
    }
    uint64_t excl = 0;
    if (tile > 0) {
        // windowed look-back: kLook predecessors loaded at once (independent
        // loads), consumed newest first until an inclusive prefix; a window
        // restarts at the first tile that has not published yet. A serial
        // walk made the first wave's look-backs chains of hundreds of
        // dependent L2 round trips.
        constexpr int kLook = 8;
        int64_t t = (int64_t)tile - 1;
        while (true) {
            uint64_t sw[kLook];
#pragma unroll
            for (int j = 0; j < kLook; ++j)
                sw[j] = t - j >= 0 ? *(volatile uint64_t *)(status + (uint64_t)(t - j) * kBins + d)
                                   : (kFlagInc | stamp);  // before tile 0: an empty inclusive prefix
            int j = 0;
            bool done = false;
#pragma unroll
            for (int q = 0; q < kLook; ++q) {
                if (done || j != q) continue;
                // not published in this pass yet (an older epoch): retry from here
                if (((sw[q] >> 32) & kEpochMask) != epoch || (sw[q] >> 62) == 0) continue;
                excl += sw[q] & kValMask;
                ++j;
                done = (sw[q] & kFlagInc) != 0;
            }
            if (done) break;
            t -= j;
            // no predecessor published since the last window: back off
            // instead of re-issuing the window loads (spinning tiles take
            // issue slots from the co-resident tile's ranking)
            if (j == 0 && backoff_ns) __nanosleep(backoff_ns);
        }
        *(volatile uint64_t *)st = kFlagInc | stamp | (excl + total);
    }
    uint32_t incl = total;  // block-wide inclusive scan of the digit totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
    }
    if (l == 31) wsum[w] = incl;
    __syncthreads();
    uint32_t carry = 0;
    for (int q = 0; q < w; ++q) carry += wsum[q];
    const uint32_t local_start = carry + incl - total;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) cnt[q][d] += local_start;
    gbase[d] = (int64_t)starts[d] + (int64_t)excl - (int64_t)local_start;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kI; ++r) {
        const uint64_t i = (tile * kT + (uint64_t)w * (32 * kI) + r * 32 + l);
        if (i < n) {
            const uint32_t dd = (uint32_t)((k[r] >> shift) & (kBins - 1));
            const uint32_t lpos = cnt[w][dd] + rank[r];
            skeys[lpos] = k[r];
            if (HAS_VALS) svals[lpos] = v[r];
        }
    }
    __syncthreads();
    const uint64_t base = tile * kT;
    const uint32_t here = n - base < (uint64_t)kT ? (uint32_t)(n - base) : (uint32_t)kT;
    for (uint32_t i = threadIdx.x; i < here; i += kThreads) {
        const uint64_t key = skeys[i];
        const uint32_t dd = (uint32_t)((key >> shift) & (kBins - 1));
        const uint64_t pos = (uint64_t)(gbase[dd] + (int64_t)i);
        keys_out[pos] = key;
        if (HAS_VALS) vals_out[pos] = svals[i];
    }
}

template <class T>
__global__ void copy_if_unsorted(T *__restrict__ dst, const T *__restrict__ src, uint64_t n,
                                 const int *__restrict__ unsorted) {
    if (unsorted && *unsorted == 0) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// keys per thread of the onesweep passes: SRDL_SORT_ITEMS=8|16 (A/B knob)
static int sort_items() {
    static int items = [] {
        const char *v = getenv("SRDL_SORT_ITEMS");
        const int x = v && *v ? atoi(v) : kDefaultSortItems;
        return x == 8 ? 8 : 16;
    }();
    return items;
}

// look-back back-off of the onesweep passes in ns (SRDL_SORT_BACKOFF; A/B knob)
static uint32_t sort_backoff_ns() {
    static uint32_t ns = [] {
        const char *v = getenv("SRDL_SORT_BACKOFF");
        return v && *v ? (uint32_t)atoi(v) : (uint32_t)SRDL_SORT_BACKOFF_DEFAULT;
    }();
    return ns;
}

// `unsorted` (optional device flag): when it reads 0 every pass returns at
// once and the keys stay in place, so a caller can skip sorting already
// ordered input without a host round trip.
void radix_sort(uint64_t *keys, uint32_t *vals, uint64_t n, uint32_t bits, cudaStream_t s,
                const int *unsorted, uint32_t lo_bit) {
    if (n <= 1 || bits == 0) return;
    SRDL_REQUIRE(n < (1ull << 32), "radix_sort: %llu rows exceeds the 32-bit rank space",
                 (unsigned long long)n);
    const int passes = (int)((bits + kRadixBits - 1) / kRadixBits);
    SRDL_REQUIRE(passes <= kMaxPasses, "radix_sort: %u bits", bits);
    static uint64_t raised = 0;
    if (first_use_on_device(&raised)) {  // the reorder tile needs more than the 48 KB default
        SRDL_CUDA(cudaFuncSetAttribute(onesweep_pass<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)onesweep_smem<true, 16>()));
        SRDL_CUDA(cudaFuncSetAttribute(onesweep_pass<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)onesweep_smem<false, 16>()));
        SRDL_CUDA(cudaFuncSetAttribute(onesweep_pass<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)onesweep_smem<true, 8>()));
        SRDL_CUDA(cudaFuncSetAttribute(onesweep_pass<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)onesweep_smem<false, 8>()));
    }
    const int items = sort_items();
    const uint32_t backoff = sort_backoff_ns();
    const uint64_t tiles = (n + (uint64_t)kThreads * items - 1) / ((uint64_t)kThreads * items);
    Scratch kalt(n * sizeof(uint64_t), s);
    Scratch valt(vals ? n * sizeof(uint32_t) : 16, s);
    // digit counts of every pass and one tile ticket per pass (zeroed once);
    // the look-back status of every (tile, digit) is the stream's persistent
    // epoch-stamped buffer (never cleared; a fresh epoch per pass)
    const size_t hist_bytes = (size_t)kMaxPasses * kBins * sizeof(uint32_t);
    const size_t ticket_bytes = (size_t)kMaxPasses * sizeof(uint32_t);
    Scratch meta(hist_bytes + ticket_bytes, s);
    uint32_t *hist = meta.as<uint32_t>();
    uint32_t *tickets = hist + kMaxPasses * kBins;
    SRDL_CUDA(cudaMemsetAsync(hist, 0, hist_bytes + ticket_bytes, s));
    SRDL_REQUIRE(lo_bit + bits <= 64, "radix_sort: bits [%u, %u) outside the key", lo_bit, lo_bit + bits);
    radix_hist_all<<<stride_grid(n), kThreads, 0, s>>>(keys, n, passes, (int)lo_bit, hist, unsorted);
    SRDL_CHECK_LAUNCH();
    radix_digit_starts<<<1, 32 * kMaxPasses, 0, s>>>(hist, passes, unsorted);
    SRDL_CHECK_LAUNCH();
    uint64_t *kin = keys, *kout = kalt.as<uint64_t>();
    uint32_t *vin = vals, *vout = vals ? valt.as<uint32_t>() : nullptr;
    for (int p = 0; p < passes; ++p) {
        const int shift = (int)lo_bit + p * kRadixBits;
        uint32_t epoch = 0;
        uint64_t *status = onesweep_status(s, (size_t)tiles * kBins, &epoch);
        if (items == 8) {
            if (vals)
                onesweep_pass<true, 8><<<(unsigned)tiles, kThreads, onesweep_smem<true, 8>(), s>>>(
                    kin, vin, n, shift, hist + p * kBins, status, epoch, tickets + p, kout, vout, unsorted, backoff);
            else
                onesweep_pass<false, 8><<<(unsigned)tiles, kThreads, onesweep_smem<false, 8>(), s>>>(
                    kin, nullptr, n, shift, hist + p * kBins, status, epoch, tickets + p, kout, nullptr, unsorted, backoff);
        } else {
            if (vals)
                onesweep_pass<true, 16><<<(unsigned)tiles, kThreads, onesweep_smem<true, 16>(), s>>>(
                    kin, vin, n, shift, hist + p * kBins, status, epoch, tickets + p, kout, vout, unsorted, backoff);
            else
                onesweep_pass<false, 16><<<(unsigned)tiles, kThreads, onesweep_smem<false, 16>(), s>>>(
                    kin, nullptr, n, shift, hist + p * kBins, status, epoch, tickets + p, kout, nullptr, unsorted, backoff);
        }
        SRDL_CHECK_LAUNCH();
        std::swap(kin, kout);
        std::swap(vin, vout);
    }
    if (kin != keys) {
        if (unsorted) {  // skipped passes left the keys in place
            copy_if_unsorted<<<stride_grid(n), kThreads, 0, s>>>(keys, kin, n, unsorted);
            SRDL_CHECK_LAUNCH();
            if (vals) {
                copy_if_unsorted<<<stride_grid(n), kThreads, 0, s>>>(vals, vin, n, unsorted);
                SRDL_CHECK_LAUNCH();
            }
        } else {
            SRDL_CUDA(cudaMemcpyAsync(keys, kin, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
            if (vals)
                SRDL_CUDA(cudaMemcpyAsync(vals, vin, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        }
    }
}

// ----------------------------------------------------------- pack / unpack

struct Chunk {
    uint32_t first, count;  // columns [first, first+count)
};

// Elementwise kernels below keep kIlp independent loads in flight per
// thread (a grid-stride loop with one load per round is capped near 2-3 TB/s
// by the ~300 K resident threads of the device, Little's law).
constexpr int kIlp = 4;

__global__ void pack_keys(Cols cols, Chunk ch, uint32_t bits, const uint32_t *__restrict__ perm,
                          uint64_t n, uint64_t *__restrict__ keys) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < n; base += kIlp * stride) {
        uint64_t row[kIlp], k[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const uint64_t i = base + u * stride;
            row[u] = i < n ? (perm ? __ldg(perm + i) : i) : 0;
            k[u] = 0;
        }
        for (uint32_t c = 0; c < ch.count; ++c) {
            const uint32_t *col = cols.c[ch.first + c];
#pragma unroll
            for (int u = 0; u < kIlp; ++u)
                if (base + u * stride < n) k[u] = (k[u] << bits) | __ldg(col + row[u]);
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u)
            if (base + u * stride < n) keys[base + u * stride] = k[u];
    }
}

__global__ void iota_u32(uint32_t *p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

// pack row j of a sorted segment with the same layout as the staged keys
__device__ __forceinline__ uint64_t pack_row(const Cols &c, uint64_t j, uint32_t arity,
                                             uint32_t bits) {
    uint64_t k = 0;
    for (uint32_t q = 0; q < arity; ++q) k = (k << bits) | __ldg(c.c[q] + j);
    return k;
}

constexpr int kMaxDiffSegs = 8;  // head, body + earlier chunks of a large staging buffer

struct Segs {
    Cols seg[kMaxDiffSegs];
    uint64_t rows[kMaxDiffSegs];
    uint32_t nseg;
};

// keep[i] = first of its run of equal keys (membership in the full
// segments is removed afterwards by the merge-path anti-join)
__global__ void flag_keys(const uint64_t *__restrict__ keys, uint64_t n, uint32_t *__restrict__ keep) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < n; base += kIlp * stride) {
        uint64_t a[kIlp], b[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const uint64_t i = base + u * stride;
            b[u] = i < n ? __ldg(keys + i) : 0;
            a[u] = i < n && i > 0 ? __ldg(keys + i - 1) : ~b[u];
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u)
            if (base + u * stride < n) keep[base + u * stride] = a[u] != b[u];
    }
}

__global__ void scatter_unpack(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ keep,
                               const uint32_t *__restrict__ pos, uint64_t n, uint32_t arity,
                               uint32_t bits, MutCols out) {
    const uint64_t mask = bits >= 32 ? 0xffffffffull : ((1ull << bits) - 1);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; base < n; base += kIlp * stride) {
        uint32_t kp[kIlp], p[kIlp];
        uint64_t k[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            const uint64_t i = base + u * stride;
            kp[u] = i < n ? __ldg(keep + i) : 0;
            k[u] = i < n ? __ldg(keys + i) : 0;
            p[u] = i < n ? __ldg(pos + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
            if (!kp[u]) continue;
            uint64_t x = k[u];
            for (int c = (int)arity - 1; c >= 0; --c) {
                out.c[c][p[u]] = (uint32_t)(x & mask);
                x >>= bits;
            }
        }
    }
}

// general path (arity*bits > 64 or presorted input): run starts of sorted rows
__global__ void flag_rows(Cols rows, uint64_t n, uint32_t arity, uint32_t *__restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        keep[i] = (i == 0) || row_cmp(rows, i - 1, rows, i, arity) != 0;
}

// Per-row binary search anti-join, for a small staged set against a large
// segment (the merge path would stream the whole segment).
__global__ void bs_diff_keys(const uint64_t *__restrict__ keys, uint64_t n, PackedRows B, uint64_t nb,
                             uint32_t *__restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        const uint64_t k = keys[i];
        uint64_t lo = 0, hi = nb;
        while (lo < hi) {
            uint64_t mid = lo + ((hi - lo) >> 1);
            if (B[mid] < k) lo = mid + 1; else hi = mid;
        }
        if (lo < nb && B[lo] == k) keep[i] = 0;
    }
}

__global__ void bs_diff_rows(Cols A, uint64_t n, Cols B, uint64_t nb, uint32_t arity,
                             uint32_t *__restrict__ keep) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        const uint64_t pos = row_bound(B, 0, nb, A, i, arity, false);
        if (pos < nb && row_cmp(B, pos, A, i, arity) == 0) keep[i] = 0;
    }
}

// binary search when the segment is this many times larger than the staged set
constexpr uint64_t kSearchRatio = 24;

static void anti_join_keys(const uint64_t *keys, uint64_t n, const Segs &S, uint32_t arity,
                           uint32_t bits, uint32_t *keep, cudaStream_t s) {
    for (uint32_t q = 0; q < S.nseg; ++q) {
        PackedRows B{S.seg[q], arity, bits};
        if (S.rows[q] > kSearchRatio * n) {
            bs_diff_keys<<<stride_grid(n), kThreads, 0, s>>>(keys, n, B, S.rows[q], keep);
            SRDL_CHECK_LAUNCH();
            continue;
        }
        const uint64_t m = n + S.rows[q];
        Scratch splits((mp_tiles(m) + 1) * sizeof(uint64_t), s);
        mp_splits_keys<<<stride_grid(mp_tiles(m) + 1), kThreads, 0, s>>>(keys, n, B, S.rows[q],
                                                                        splits.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        mp_diff_keys<<<mp_grid(m), kThreads, 0, s>>>(keys, n, B, S.rows[q], splits.as<uint64_t>(), keep);
        SRDL_CHECK_LAUNCH();
    }
}

static void anti_join_rows(const Cols &rows, uint64_t n, const Segs &S, uint32_t arity,
                           uint32_t *keep, cudaStream_t s) {
    for (uint32_t q = 0; q < S.nseg; ++q) {
        if (S.rows[q] > kSearchRatio * n) {
            bs_diff_rows<<<stride_grid(n), kThreads, 0, s>>>(rows, n, S.seg[q], S.rows[q], arity, keep);
            SRDL_CHECK_LAUNCH();
            continue;
        }
        const uint64_t m = n + S.rows[q];
        Scratch splits((mp_tiles(m) + 1) * sizeof(uint64_t), s);
        mp_splits_rows<<<stride_grid(mp_tiles(m) + 1), kThreads, 0, s>>>(rows, n, S.seg[q], S.rows[q],
                                                                        arity, splits.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        mp_diff_rows<<<mp_grid(m), kThreads, mp_smem(arity), s>>>(rows, n, S.seg[q], S.rows[q], arity,
                                                                  splits.as<uint64_t>(), keep);
        SRDL_CHECK_LAUNCH();
    }
}

__global__ void scatter_rows(Cols rows, const uint32_t *__restrict__ keep,
                             const uint32_t *__restrict__ pos, uint64_t n, uint32_t arity,
                             MutCols out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        uint32_t p = pos[i];
        for (uint32_t c = 0; c < arity; ++c) out.c[c][p] = __ldg(rows.c[c] + i);
    }
}

__global__ void gather_cols(Cols cols, uint32_t arity, const uint32_t *__restrict__ idx, uint64_t n,
                            MutCols out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t r = idx[i];
        for (uint32_t c = 0; c < arity; ++c) out.c[c][i] = __ldg(cols.c[c] + r);
    }
}

// every packed key back to `arity` columns of `bits` bits (no dedup)
__global__ void unpack_all(const uint64_t *__restrict__ keys, uint64_t n, uint32_t arity, uint32_t bits,
                           MutCols out) {
    const uint64_t mask = bits >= 32 ? 0xffffffffull : ((1ull << bits) - 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = keys[i];
        for (int c = (int)arity - 1; c >= 0; --c) {
            out.c[c][i] = (uint32_t)(k & mask);
            k >>= bits;
        }
    }
}

// bad = 1 if some row is greater than (strict: not less than) its successor.
// Unsorted input is the common case (staged join output): one atomic per
// warp that sees an inversion, and every warp stops once the flag is set
// (a per-thread atomic on the same word serialised millions of them).
__global__ void check_sorted(Cols rows, uint64_t n, uint32_t arity, int strict, int *bad) {
    const int limit = strict ? 0 : 1;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base + 1 < n; base += stride) {
        if (*(volatile int *)bad) return;  // warp-uniform
        const uint64_t i = base + threadIdx.x;
        const bool inv = i + 1 < n && row_cmp(rows, i, rows, i + 1, arity) >= limit;
        const uint32_t m = __ballot_sync(0xffffffffu, inv);
        if (m) {
            if (lane_id() == 0) atomicExch(bad, 1);
            return;
        }
    }
}

static bool rows_sorted(const Cols &rows, uint64_t n, uint32_t arity, bool strict, cudaStream_t s) {
    if (n <= 1) return true;
    Scratch bad(sizeof(int), s);
    SRDL_CUDA(cudaMemsetAsync(bad.as<int>(), 0, sizeof(int), s));
    check_sorted<<<stride_grid(n), kThreads, 0, s>>>(rows, n, arity, strict ? 1 : 0, bad.as<int>());
    SRDL_CHECK_LAUNCH();
    int h = 0;
    SRDL_CUDA(cudaMemcpyAsync(&h, bad.as<int>(), sizeof(int), cudaMemcpyDeviceToHost, s));
    SRDL_CUDA(cudaStreamSynchronize(s));
    return h == 0;
}

// Sort + unique + anti-join; the heart of compute_delta.
// Inputs up to this many rows decide "already sorted?" on the device (the
// radix passes skip themselves) instead of with a host round trip; larger
// inputs take the host branch, where the sorted fast path avoids the key
// packing altogether and one round trip is noise.
constexpr uint64_t kDeviceBranchRows = 1ull << 22;

static uint64_t sort_unique_minus(const uint32_t *const *cols, uint32_t arity, uint64_t n,
                                  uint32_t bits, const Segs &S, uint32_t *const *out,
                                  cudaStream_t s, bool want_count = true,
                                  uint32_t *count_dev = nullptr) {
    SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS, "arity %u outside [1, %d]", arity,
                 SRDL_MAX_COLS);
    SRDL_REQUIRE(bits >= 1 && bits <= 32, "bits %u outside [1, 32]", bits);
    if (n == 0) return 0;
    SRDL_REQUIRE(n < (1ull << 32), "sort: %llu rows exceeds 2^32", (unsigned long long)n);
    Cols in = make_cols(cols, arity);
    MutCols dst = make_mut(out, arity);
    const unsigned g = stride_grid(n);
    Scratch keys(n * sizeof(uint64_t), s);
    Scratch keep(n * sizeof(uint32_t), s);
    Scratch total(sizeof(uint32_t) * 2, s);
    const uint32_t per_chunk = 64 / bits;
    const bool device_branch = n <= kDeviceBranchRows || count_dev != nullptr;
    Scratch unsorted(sizeof(int), s);
    const int *uns = nullptr;
    if (device_branch) {
        SRDL_CUDA(cudaMemsetAsync(unsorted.as<int>(), 0, sizeof(int), s));
        check_sorted<<<stride_grid(n), kThreads, 0, s>>>(in, n, arity, 0, unsorted.as<int>());
        SRDL_CHECK_LAUNCH();
        uns = unsorted.as<int>();
    }
    if (!device_branch && rows_sorted(in, n, arity, false, s)) {
        // staged rows already in index order (e.g. WCOJ output enumerated in
        // variable order): unique + anti-join without sorting
        flag_rows<<<g, kThreads, 0, s>>>(in, n, arity, keep.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        anti_join_rows(in, n, S, arity, keep.as<uint32_t>(), s);
        Scratch pos(n * sizeof(uint32_t), s);
        exclusive_scan_u32(keep.as<uint32_t>(), pos.as<uint32_t>(), n, total.as<uint32_t>(), s);
        scatter_rows<<<g, kThreads, 0, s>>>(in, keep.as<uint32_t>(), pos.as<uint32_t>(), n, arity, dst);
        SRDL_CHECK_LAUNCH();
    } else if (arity <= per_chunk) {
        pack_keys<<<g, kThreads, 0, s>>>(in, Chunk{0, arity}, bits, nullptr, n, keys.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        radix_sort(keys.as<uint64_t>(), nullptr, n, arity * bits, s, uns);
        flag_keys<<<g, kThreads, 0, s>>>(keys.as<uint64_t>(), n, keep.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        anti_join_keys(keys.as<uint64_t>(), n, S, arity, bits, keep.as<uint32_t>(), s);
        Scratch pos(n * sizeof(uint32_t), s);
        exclusive_scan_u32(keep.as<uint32_t>(), pos.as<uint32_t>(), n, total.as<uint32_t>(), s);
        scatter_unpack<<<g, kThreads, 0, s>>>(keys.as<uint64_t>(), keep.as<uint32_t>(),
                                              pos.as<uint32_t>(), n, arity, bits, dst);
        SRDL_CHECK_LAUNCH();
    } else {
        Scratch perm(n * sizeof(uint32_t), s);
        iota_u32<<<g, kThreads, 0, s>>>(perm.as<uint32_t>(), n);
        SRDL_CHECK_LAUNCH();
        // least significant chunk first; chunks end at the last column
        int end = (int)arity;
        while (end > 0) {
            int first = end - (int)per_chunk;
            if (first < 0) first = 0;
            Chunk ch{(uint32_t)first, (uint32_t)(end - first)};
            pack_keys<<<g, kThreads, 0, s>>>(in, ch, bits, perm.as<uint32_t>(), n,
                                             keys.as<uint64_t>());
            SRDL_CHECK_LAUNCH();
            radix_sort(keys.as<uint64_t>(), perm.as<uint32_t>(), n, ch.count * bits, s, uns);
            end = first;
        }
        Scratch sorted(n * sizeof(uint32_t) * arity, s);
        MutCols tmp{};
        Cols tmpc{};
        for (uint32_t c = 0; c < arity; ++c) {
            tmp.c[c] = sorted.as<uint32_t>() + c * n;
            tmpc.c[c] = tmp.c[c];
        }
        gather_cols<<<g, kThreads, 0, s>>>(in, arity, perm.as<uint32_t>(), n, tmp);
        SRDL_CHECK_LAUNCH();
        flag_rows<<<g, kThreads, 0, s>>>(tmpc, n, arity, keep.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        anti_join_rows(tmpc, n, S, arity, keep.as<uint32_t>(), s);
        Scratch pos(n * sizeof(uint32_t), s);
        exclusive_scan_u32(keep.as<uint32_t>(), pos.as<uint32_t>(), n, total.as<uint32_t>(), s);
        scatter_rows<<<g, kThreads, 0, s>>>(tmpc, keep.as<uint32_t>(), pos.as<uint32_t>(), n, arity,
                                            dst);
        SRDL_CHECK_LAUNCH();
    }
    if (count_dev) {  // asynchronous: the count stays on the device
        SRDL_CUDA(cudaMemcpyAsync(count_dev, total.as<uint32_t>(), sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        return n;
    }
    if (!want_count) return n;  // caller guarantees distinct rows: no round trip
    uint32_t cnt = 0;
    SRDL_CUDA(cudaMemcpyAsync(&cnt, total.as<uint32_t>(), sizeof(cnt), cudaMemcpyDeviceToHost, s));
    SRDL_CUDA(cudaStreamSynchronize(s));
    return cnt;
}

}  // namespace srdl

using namespace srdl;

extern "C" {

int srdl_sort_dedup(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                    uint32_t *const *out, uint64_t *n_out, void *stream) {
    return guarded([&] {
        Segs none{};
        none.nseg = 0;
        const uint64_t got = sort_unique_minus(cols, arity, n, bits, none, out, (cudaStream_t)stream,
                                               n_out != nullptr);
        if (n_out) *n_out = got;
    });
}

int srdl_compute_delta(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                       const uint32_t *const *const *seg_cols, const uint64_t *seg_rows,
                       uint32_t nseg, uint32_t *const *out, uint64_t *n_out, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(nseg <= kMaxDiffSegs, "at most %d full segments", kMaxDiffSegs);
        Segs S{};
        S.nseg = 0;
        for (uint32_t q = 0; q < nseg; ++q) {
            if (seg_rows[q] == 0) continue;
            S.seg[S.nseg] = make_cols(seg_cols[q], arity);
            S.rows[S.nseg] = seg_rows[q];
            S.nseg++;
        }
        *n_out = sort_unique_minus(cols, arity, n, bits, S, out, (cudaStream_t)stream);
    });
}

int srdl_compute_delta_async(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                             const uint32_t *const *const *seg_cols, const uint64_t *seg_rows,
                             uint32_t nseg, uint32_t *const *out, uint32_t *count_dev, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(nseg <= kMaxDiffSegs, "at most %d full segments", kMaxDiffSegs);
        SRDL_REQUIRE(count_dev != nullptr, "compute_delta_async needs a device count slot");
        cudaStream_t s = (cudaStream_t)stream;
        if (n == 0) {
            SRDL_CUDA(cudaMemsetAsync(count_dev, 0, sizeof(uint32_t), s));
            return;
        }
        Segs S{};
        S.nseg = 0;
        for (uint32_t q = 0; q < nseg; ++q) {
            if (seg_rows[q] == 0) continue;
            S.seg[S.nseg] = make_cols(seg_cols[q], arity);
            S.rows[S.nseg] = seg_rows[q];
            S.nseg++;
        }
        sort_unique_minus(cols, arity, n, bits, S, out, s, false, count_dev);
    });
}

int srdl_sort_reorder(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits, uint32_t nkey,
                      uint32_t *const *out, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS, "arity %u outside [1, %d]", arity, SRDL_MAX_COLS);
        SRDL_REQUIRE(nkey >= 1 && nkey <= arity && bits >= 1 && bits <= 32 && nkey * bits <= 64,
                     "sort_reorder: %u key columns of %u bits", nkey, bits);
        if (n == 0) return;
        SRDL_REQUIRE(n < (1ull << 32), "sort: %llu rows exceeds 2^32", (unsigned long long)n);
        cudaStream_t s = (cudaStream_t)stream;
        const Cols in = make_cols(cols, arity);
        const MutCols dst = make_mut(out, arity);
        const unsigned g = stride_grid(n);
        Scratch keys(n * sizeof(uint64_t), s);
        if (arity == 2 && nkey == 1) {
            // both columns ride in one key (column 0 in the high word); only
            // the high word's significant bits are sorted, stably
            pack_keys<<<g, kThreads, 0, s>>>(in, Chunk{0, 2}, 32, nullptr, n, keys.as<uint64_t>());
            SRDL_CHECK_LAUNCH();
            radix_sort(keys.as<uint64_t>(), nullptr, n, bits, s, nullptr, 32);
            unpack_all<<<g, kThreads, 0, s>>>(keys.as<uint64_t>(), n, 2, 32, dst);
            SRDL_CHECK_LAUNCH();
            return;
        }
        // key columns packed, a stable sort carries the row permutation, all
        // columns gathered through it
        Scratch perm(n * sizeof(uint32_t), s);
        pack_keys<<<g, kThreads, 0, s>>>(in, Chunk{0, nkey}, bits, nullptr, n, keys.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        iota_u32<<<g, kThreads, 0, s>>>(perm.as<uint32_t>(), n);
        SRDL_CHECK_LAUNCH();
        radix_sort(keys.as<uint64_t>(), perm.as<uint32_t>(), n, nkey * bits, s);
        gather_cols<<<g, kThreads, 0, s>>>(in, arity, perm.as<uint32_t>(), n, dst);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_is_sorted_strict(const uint32_t *const *cols, uint32_t arity, uint64_t n, int *ok,
                          void *stream) {
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        *ok = 1;
        if (n <= 1) return;
        *ok = rows_sorted(make_cols(cols, arity), n, arity, true, s) ? 1 : 0;
    });
}

int srdl_gather(const uint32_t *const *cols, uint32_t arity, const uint32_t *idx, uint64_t n,
                uint32_t *const *out, void *stream) {
    return guarded([&] {
        if (n == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        gather_cols<<<stride_grid(n), kThreads, 0, s>>>(make_cols(cols, arity), arity, idx, n,
                                                        make_mut(out, arity));
        SRDL_CHECK_LAUNCH();
    });
}

}  // extern "C"
