// Delta maintenance, part 2, and the root histogram pipeline:
//  - rank merge of disjoint sorted row sets (head/body merge, Fig. 1 "Merge";
//    reference ColumnarRelation.merge_delta, storage.py:272)
//  - run-length histograms of a sorted key column and their incremental
//    union (reference Histogram.over_column / updated, storage.py:48-76)
//  - per-plan root work space: d2 lookup + prefix of outer_deg * d2
//    (reference executor.build_partition, executor.py:246-274; paper Alg. 1)
//  - constant-prefix narrowing (reference executor.prepare, executor.py:188)
//  - the synthetic R-MAT generator used by the benchmarks.
#include "common.cuh"
#include "mergepath.cuh"

namespace srdl {

// out[i + |{b < a_i}|] = a_i ; out[j + |{a < b_j}|] = b_j  (disjoint inputs)
__global__ void rank_merge_rows(Cols A, uint64_t na, Cols B, uint64_t nb, uint32_t arity,
                                MutCols out) {
    const uint64_t n = na + nb;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t dst;
        const Cols *src;
        uint64_t row;
        if (t < na) {
            row = t;
            src = &A;
            dst = t + row_bound(B, 0, nb, A, row, arity, false);
        } else {
            row = t - na;
            src = &B;
            dst = row + row_bound(A, 0, na, B, row, arity, false);
        }
        for (uint32_t c = 0; c < arity; ++c) out.c[c][dst] = __ldg(src->c[c] + row);
    }
}

__global__ void run_flags(const uint32_t *__restrict__ col, uint64_t n, uint32_t *__restrict__ f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        f[i] = (i == 0) || col[i] != col[i - 1];
}

__global__ void run_starts(const uint32_t *__restrict__ col, const uint32_t *__restrict__ f,
                           const uint32_t *__restrict__ pos, uint64_t n, uint32_t *__restrict__ keys,
                           uint32_t *__restrict__ starts) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (f[i]) {
            keys[pos[i]] = col[i];
            starts[pos[i]] = (uint32_t)i;
        }
    }
}

__global__ void run_lengths(const uint32_t *__restrict__ starts, const uint32_t *__restrict__ kdev,
                            uint64_t n, uint32_t *__restrict__ deg, uint64_t *__restrict__ deg64) {
    const uint64_t K = *kdev;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < K;
         k += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t end = k + 1 < K ? starts[k + 1] : n;
        uint32_t d = (uint32_t)(end - starts[k]);
        deg[k] = d;
        deg64[k] = d;
    }
}

// merged (key, degree) lists with ties kept adjacent (A before B)
__global__ void rank_merge_hist(const uint32_t *__restrict__ ka, const uint32_t *__restrict__ da,
                                uint64_t na, const uint32_t *__restrict__ kb,
                                const uint32_t *__restrict__ db, uint64_t nb,
                                uint32_t *__restrict__ mk, uint32_t *__restrict__ md) {
    const uint64_t n = na + nb;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (t < na) {
            uint32_t k = ka[t];
            uint64_t lo = 0, hi = nb;
            while (lo < hi) {
                uint64_t m = (lo + hi) >> 1;
                if (kb[m] < k) lo = m + 1; else hi = m;
            }
            mk[t + lo] = k;
            md[t + lo] = da[t];
        } else {
            uint64_t j = t - na;
            uint32_t k = kb[j];
            uint64_t lo = 0, hi = na;
            while (lo < hi) {
                uint64_t m = (lo + hi) >> 1;
                if (ka[m] <= k) lo = m + 1; else hi = m;
            }
            mk[j + lo] = k;
            md[j + lo] = db[j];
        }
    }
}

__global__ void combine_pairs(const uint32_t *__restrict__ mk, const uint32_t *__restrict__ md,
                              const uint32_t *__restrict__ f, const uint32_t *__restrict__ pos,
                              uint64_t n, uint32_t *__restrict__ keys, uint32_t *__restrict__ deg,
                              uint64_t *__restrict__ deg64) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!f[i]) continue;
        uint32_t d = md[i];
        if (i + 1 < n && mk[i + 1] == mk[i]) d += md[i + 1];
        keys[pos[i]] = mk[i];
        deg[pos[i]] = d;
        deg64[pos[i]] = d;
    }
}

__global__ void root_work_kernel(const uint32_t *__restrict__ okeys, const uint32_t *__restrict__ odeg,
                                 const uint64_t *__restrict__ oprefix, uint64_t nk,
                                 const uint32_t *__restrict__ ikeys, const uint32_t *__restrict__ ideg,
                                 const uint64_t *__restrict__ iprefix, uint64_t nik, int has_inner,
                                 uint32_t *__restrict__ d2, uint64_t *__restrict__ work,
                                 uint32_t *__restrict__ outer_lo, uint32_t *__restrict__ inner_lo) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = 1, ilo = 0;
        if (has_inner) {
            uint32_t k = okeys[i];
            uint64_t lo = 0, hi = nik;
            while (lo < hi) {
                uint64_t m = (lo + hi) >> 1;
                if (ikeys[m] < k) lo = m + 1; else hi = m;
            }
            const bool found = lo < nik && ikeys[lo] == k;
            d = found ? ideg[lo] : 0u;
            if (found && iprefix) ilo = (uint32_t)(iprefix[lo] - ideg[lo]);
        }
        d2[i] = d;
        work[i] = (uint64_t)odeg[i] * d;
        if (outer_lo) outer_lo[i] = (uint32_t)(oprefix[i] - odeg[i]);
        if (inner_lo) inner_lo[i] = ilo;
    }
}

__global__ void narrow_prefix_kernel(Cols cols, uint64_t n, const uint32_t *__restrict__ vals,
                                     uint32_t nv, uint64_t *__restrict__ range) {
    uint64_t lo = 0, hi = n;
    for (uint32_t c = 0; c < nv && lo < hi; ++c) {
        const uint32_t *col = cols.c[c];
        uint32_t v = vals[c];
        uint64_t a = lo, b = hi;
        while (a < b) {
            uint64_t m = (a + b) >> 1;
            if (col[m] < v) a = m + 1; else b = m;
        }
        uint64_t e = a, f = hi;
        while (e < f) {
            uint64_t m = (e + f) >> 1;
            if (col[m] <= v) e = m + 1; else f = m;
        }
        lo = a;
        hi = e;
    }
    if (lo > hi) hi = lo;
    range[0] = lo;
    range[1] = hi;
}

// CSR offsets of a sorted key list over the id space [0, n_ids]: off[v] =
// rows with key < v. Each thread owns kIdsPerThread consecutive ids, finds
// the first key >= its first id by one binary search and walks forward, so
// the work is O(n_ids + nk) plus one search per tile (instead of one search
// per id); consecutive threads write consecutive 64-byte runs.
constexpr uint32_t kIdsPerThread = 16;

__global__ void dense_offsets_kernel(const uint32_t *__restrict__ keys,
                                     const uint64_t *__restrict__ prefix, uint64_t nk,
                                     uint32_t n_ids, uint32_t *__restrict__ off) {
    const uint64_t ntiles = ((uint64_t)n_ids + kIdsPerThread) / kIdsPerThread;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ntiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v0 = t * kIdsPerThread;
        uint64_t lo = 0, hi = nk;  // first key >= v0
        while (lo < hi) {
            const uint64_t m = (lo + hi) >> 1;
            if (__ldg(keys + m) < v0) lo = m + 1; else hi = m;
        }
        uint32_t vals[kIdsPerThread];
#pragma unroll
        for (uint32_t j = 0; j < kIdsPerThread; ++j) {
            const uint64_t v = v0 + j;
            while (lo < nk && __ldg(keys + lo) < v) ++lo;
            vals[j] = lo ? (uint32_t)__ldg(prefix + lo - 1) : 0u;
        }
        if (v0 + kIdsPerThread <= (uint64_t)n_ids + 1) {
            uint4 *dst = reinterpret_cast<uint4 *>(off + v0);  // off is 16-byte aligned (allocator)
#pragma unroll
            for (uint32_t j = 0; j < kIdsPerThread / 4; ++j)
                dst[j] = make_uint4(vals[4 * j], vals[4 * j + 1], vals[4 * j + 2], vals[4 * j + 3]);
        } else {
            for (uint32_t j = 0; v0 + j <= (uint64_t)n_ids; ++j) off[v0 + j] = vals[j];
        }
    }
}

__device__ __forceinline__ uint32_t owner_of(uint32_t v, uint32_t world) {
    return ((uint32_t)(v * 2654435761u) >> 8) % world;
}

__global__ void owner_flags(const uint32_t *__restrict__ col, uint64_t n, uint32_t world, uint32_t rank,
                            uint32_t *__restrict__ f) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        f[i] = owner_of(col[i], world) == rank;
}

__global__ void scatter_flagged(Cols in, uint32_t arity, const uint32_t *__restrict__ f,
                                const uint32_t *__restrict__ pos, uint64_t n, uint64_t base, MutCols out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!f[i]) continue;
        for (uint32_t c = 0; c < arity; ++c) out.c[c][base + pos[i]] = __ldg(in.c[c] + i);
    }
}

__global__ void root_own_kernel(const uint32_t *__restrict__ keys, uint64_t nk,
                                const uint32_t *__restrict__ odeg, const uint32_t *__restrict__ d2,
                                uint32_t world, uint32_t rank, uint64_t *__restrict__ work) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nk;
         i += (uint64_t)gridDim.x * blockDim.x)
        work[i] = owner_of(keys[i], world) == rank ? (uint64_t)odeg[i] * d2[i] : 0;
}

// counter-based RNG: splitmix64 finaliser over (seed, edge, level)
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

__global__ void rmat_kernel(uint32_t scale, uint64_t m, float a, float b, float c, uint64_t seed,
                            uint32_t *__restrict__ src, uint32_t *__restrict__ dst) {
    const float ab = a + b, abc = a + b + c;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t u = 0, v = 0;
        uint64_t state = mix64(seed * 0x9e3779b97f4a7c15ull + e);
        for (uint32_t lvl = 0; lvl < scale; ++lvl) {
            state = mix64(state + 0x9e3779b97f4a7c15ull);
            float r = (float)(state >> 40) * (1.0f / 16777216.0f);
            uint32_t sb = r >= ab;
            uint32_t db = (r >= a && r < ab) || r >= abc;
            u |= sb << lvl;
            v |= db << lvl;
        }
        src[e] = u;
        dst[e] = v;
    }
}

// ---- device-sized variants (lengths read from device memory): the delta
// histogram and its union with the full histogram run back to back with a
// single host readback at the end (srdl_histogram_union)

// rank_merge_hist with |B| = *nb_dev; t runs over the capacity na + nb_cap
__global__ void rank_merge_hist_dev(const uint32_t *__restrict__ ka, const uint32_t *__restrict__ da,
                                    uint64_t na, const uint32_t *__restrict__ kb,
                                    const uint32_t *__restrict__ db, const uint32_t *__restrict__ nb_dev,
                                    uint64_t cap, uint32_t *__restrict__ mk, uint32_t *__restrict__ md) {
    const uint64_t nb = *nb_dev;
    const uint64_t n = na + nb;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n && t < cap;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (t < na) {
            const uint32_t k = ka[t];
            uint64_t lo = 0, hi = nb;
            while (lo < hi) {
                const uint64_t m = (lo + hi) >> 1;
                if (kb[m] < k) lo = m + 1; else hi = m;
            }
            mk[t + lo] = k;
            md[t + lo] = da[t];
        } else {
            const uint64_t j = t - na;
            const uint32_t k = kb[j];
            uint64_t lo = 0, hi = na;
            while (lo < hi) {
                const uint64_t m = (lo + hi) >> 1;
                if (ka[m] <= k) lo = m + 1; else hi = m;
            }
            mk[j + lo] = k;
            md[j + lo] = db[j];
        }
    }
}

// run flags over the first na + *nb_dev entries, zero up to the capacity
__global__ void run_flags_dev(const uint32_t *__restrict__ col, uint64_t na, const uint32_t *__restrict__ nb_dev,
                              uint64_t cap, uint32_t *__restrict__ f) {
    const uint64_t n = na + *nb_dev;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
         i += (uint64_t)gridDim.x * blockDim.x)
        f[i] = i < n && ((i == 0) || col[i] != col[i - 1]);
}

__global__ void combine_pairs_dev(const uint32_t *__restrict__ mk, const uint32_t *__restrict__ md,
                                  const uint32_t *__restrict__ f, const uint32_t *__restrict__ pos,
                                  uint64_t na, const uint32_t *__restrict__ nb_dev, uint32_t *__restrict__ keys,
                                  uint32_t *__restrict__ deg, uint64_t *__restrict__ deg64) {
    const uint64_t n = na + *nb_dev;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!f[i]) continue;
        uint32_t d = md[i];
        if (i + 1 < n && mk[i + 1] == mk[i]) d += md[i + 1];
        keys[pos[i]] = mk[i];
        deg[pos[i]] = d;
        deg64[pos[i]] = d;
    }
}

__global__ void fence_kernel(const uint32_t *__restrict__ keys, uint64_t m, uint32_t *__restrict__ fence) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        fence[i] = keys[i * SRDL_FENCE];
}

static uint64_t histogram_impl(const uint32_t *col, uint64_t n, uint32_t *keys, uint32_t *degrees,
                               uint64_t *prefix, cudaStream_t s) {
    if (n == 0) return 0;
    SRDL_REQUIRE(n < (1ull << 32), "histogram: column longer than 2^32");
    const unsigned g = stride_grid(n);
    Scratch f(n * sizeof(uint32_t), s), pos(n * sizeof(uint32_t), s), starts(n * sizeof(uint32_t), s);
    Scratch k(sizeof(uint32_t) * 2, s), deg64(n * sizeof(uint64_t), s);
    run_flags<<<g, kThreads, 0, s>>>(col, n, f.as<uint32_t>());
    SRDL_CHECK_LAUNCH();
    exclusive_scan_u32(f.as<uint32_t>(), pos.as<uint32_t>(), n, k.as<uint32_t>(), s);
    run_starts<<<g, kThreads, 0, s>>>(col, f.as<uint32_t>(), pos.as<uint32_t>(), n, keys,
                                      starts.as<uint32_t>());
    SRDL_CHECK_LAUNCH();
    run_lengths<<<g, kThreads, 0, s>>>(starts.as<uint32_t>(), k.as<uint32_t>(), n, degrees,
                                       deg64.as<uint64_t>());
    SRDL_CHECK_LAUNCH();
    uint32_t K = 0;
    SRDL_CUDA(cudaMemcpyAsync(&K, k.as<uint32_t>(), sizeof(K), cudaMemcpyDeviceToHost, s));
    SRDL_CUDA(cudaStreamSynchronize(s));
    inclusive_scan_u64(deg64.as<uint64_t>(), prefix, K, s);
    return K;
}

// max over the columns of a row set (atomicMax of per-warp maxima)
__global__ void max_rows(Cols cols, uint32_t arity, uint64_t n, uint32_t *__restrict__ out) {
    uint32_t m = 0;
    for (uint32_t c = 0; c < arity; ++c)
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
             i += (uint64_t)gridDim.x * blockDim.x)
            m = max(m, __ldg(cols.c[c] + i));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ---- packed exchange buffers (multi-GPU all-to-all, dist.py)

__global__ void owner_keys(const uint32_t *__restrict__ col, uint64_t n, uint32_t world,
                           uint64_t *__restrict__ keys, uint32_t *__restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        keys[i] = owner_of(__ldg(col + i), world);
        idx[i] = (uint32_t)i;
    }
}

// counts[r] = rows owned by rank r (keys sorted by owner)
__global__ void owner_counts(const uint64_t *__restrict__ keys, uint64_t n, uint32_t world,
                             uint64_t *__restrict__ counts) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= world) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {  // first key >= r
        const uint64_t m = (lo + hi) >> 1;
        if (keys[m] < r) lo = m + 1; else hi = m;
    }
    uint64_t a = lo;
    hi = n;
    while (lo < hi) {  // first key > r
        const uint64_t m = (lo + hi) >> 1;
        if (keys[m] <= r) lo = m + 1; else hi = m;
    }
    counts[r] = lo - a;
}

// send[i * arity + c] = cols[c][idx[i]]: row-major rows, grouped by owner
__global__ void pack_rows(Cols cols, uint32_t arity, const uint32_t *__restrict__ idx, uint64_t n,
                          uint32_t *__restrict__ send) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = __ldg(idx + i);
        for (uint32_t c = 0; c < arity; ++c) send[i * arity + c] = __ldg(cols.c[c] + r);
    }
}

__global__ void unpack_rows(const uint32_t *__restrict__ recv, uint32_t arity, uint64_t n, MutCols out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        for (uint32_t c = 0; c < arity; ++c) out.c[c][i] = __ldg(recv + i * arity + c);
}

}  // namespace srdl

using namespace srdl;

static void histogram_union_impl(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                                 uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix,
                                 uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint64_t *kd_out,
                                 uint64_t *ku_out, uint32_t *k_dev, cudaStream_t s);


extern "C" {


int srdl_merge(const uint32_t *const *a, uint64_t na, const uint32_t *const *b, uint64_t nb,
               uint32_t arity, uint32_t *const *out, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(arity >= 1 && arity <= SRDL_MAX_COLS, "arity %u out of range", arity);
        const uint64_t n = na + nb;
        if (n == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        Cols A = na ? make_cols(a, arity) : Cols{};
        Cols B = nb ? make_cols(b, arity) : Cols{};
        Scratch splits((mp_tiles(n) + 1) * sizeof(uint64_t), s);
        mp_splits_rows<<<stride_grid(mp_tiles(n) + 1), kThreads, 0, s>>>(A, na, B, nb, arity,
                                                                        splits.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        mp_merge_rows<<<mp_grid(n), kThreads, mp_smem(arity), s>>>(A, na, B, nb, arity,
                                                                   splits.as<uint64_t>(), make_mut(out, arity));
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_histogram(const uint32_t *col, uint64_t n, uint32_t *keys, uint32_t *degrees,
                   uint64_t *prefix, uint64_t *k_out, void *stream) {
    return guarded([&] { *k_out = histogram_impl(col, n, keys, degrees, prefix, (cudaStream_t)stream); });
}

int srdl_histogram_merge(const uint32_t *ka, const uint32_t *da, uint64_t na, const uint32_t *kb,
                         const uint32_t *db, uint64_t nb, uint32_t *keys, uint32_t *degrees,
                         uint64_t *prefix, uint64_t *k_out, void *stream) {
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        const uint64_t n = na + nb;
        *k_out = 0;
        if (n == 0) return;
        const unsigned g = stride_grid(n);
        Scratch mk(n * sizeof(uint32_t), s), md(n * sizeof(uint32_t), s);
        Scratch f(n * sizeof(uint32_t), s), pos(n * sizeof(uint32_t), s);
        Scratch k(sizeof(uint32_t) * 2, s), deg64(n * sizeof(uint64_t), s);
        rank_merge_hist<<<g, kThreads, 0, s>>>(ka, da, na, kb, db, nb, mk.as<uint32_t>(),
                                               md.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        run_flags<<<g, kThreads, 0, s>>>(mk.as<uint32_t>(), n, f.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u32(f.as<uint32_t>(), pos.as<uint32_t>(), n, k.as<uint32_t>(), s);
        combine_pairs<<<g, kThreads, 0, s>>>(mk.as<uint32_t>(), md.as<uint32_t>(), f.as<uint32_t>(),
                                             pos.as<uint32_t>(), n, keys, degrees,
                                             deg64.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        uint32_t K = 0;
        SRDL_CUDA(cudaMemcpyAsync(&K, k.as<uint32_t>(), sizeof(K), cudaMemcpyDeviceToHost, s));
        SRDL_CUDA(cudaStreamSynchronize(s));
        inclusive_scan_u64(deg64.as<uint64_t>(), prefix, K, s);
        *k_out = K;
    });
}

int srdl_histogram_union(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                         uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix, uint64_t *kd_out,
                         uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint64_t *ku_out, void *stream) {
    return guarded([&] {
        *kd_out = 0;
        *ku_out = 0;
        histogram_union_impl(col, n, fkeys, fdeg, nf, dkeys, ddeg, dprefix, ukeys, udeg, uprefix, kd_out, ku_out,
                             nullptr, (cudaStream_t)stream);
    });
}

int srdl_histogram_union_async(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                               uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix,
                               uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint32_t *k_dev,
                               void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(k_dev != nullptr, "histogram_union_async needs two device count slots");
        cudaStream_t s = (cudaStream_t)stream;
        if (n == 0) {
            SRDL_CUDA(cudaMemsetAsync(k_dev, 0, 2 * sizeof(uint32_t), s));
            return;
        }
        histogram_union_impl(col, n, fkeys, fdeg, nf, dkeys, ddeg, dprefix, ukeys, udeg, uprefix, nullptr, nullptr,
                             k_dev, s);
    });
}

}  // extern "C"

static void histogram_union_impl(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                                 uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix,
                                 uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint64_t *kd_out,
                                 uint64_t *ku_out, uint32_t *k_dev, cudaStream_t s) {
    {
        if (n == 0) return;
        SRDL_REQUIRE(n + nf < (1ull << 32), "histogram_union: %llu keys exceed 2^32",
                     (unsigned long long)(n + nf));
        const uint64_t cap = n + nf;
        const unsigned g = stride_grid(n), gu = stride_grid(cap);
        Scratch f(cap * sizeof(uint32_t), s), pos(cap * sizeof(uint32_t), s), starts(n * sizeof(uint32_t), s);
        Scratch k(sizeof(uint32_t) * 4, s), deg64(cap * sizeof(uint64_t), s);
        uint32_t *kd = k.as<uint32_t>(), *ku = kd + 2;
        // delta histogram (keys/degrees of the sorted column), sized on device
        run_flags<<<g, kThreads, 0, s>>>(col, n, f.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u32(f.as<uint32_t>(), pos.as<uint32_t>(), n, kd, s);
        run_starts<<<g, kThreads, 0, s>>>(col, f.as<uint32_t>(), pos.as<uint32_t>(), n, dkeys,
                                          starts.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        SRDL_CUDA(cudaMemsetAsync(deg64.as<uint64_t>(), 0, n * sizeof(uint64_t), s));
        run_lengths<<<g, kThreads, 0, s>>>(starts.as<uint32_t>(), kd, n, ddeg, deg64.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        inclusive_scan_u64(deg64.as<uint64_t>(), dprefix, n, s);  // entries >= K_d repeat the total
        // union with the existing histogram (equal keys summed)
        Scratch mk(cap * sizeof(uint32_t), s), md(cap * sizeof(uint32_t), s);
        rank_merge_hist_dev<<<gu, kThreads, 0, s>>>(fkeys, fdeg, nf, dkeys, ddeg, kd, cap, mk.as<uint32_t>(),
                                                    md.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        run_flags_dev<<<gu, kThreads, 0, s>>>(mk.as<uint32_t>(), nf, kd, cap, f.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        exclusive_scan_u32(f.as<uint32_t>(), pos.as<uint32_t>(), cap, ku, s);
        SRDL_CUDA(cudaMemsetAsync(deg64.as<uint64_t>(), 0, cap * sizeof(uint64_t), s));
        combine_pairs_dev<<<gu, kThreads, 0, s>>>(mk.as<uint32_t>(), md.as<uint32_t>(), f.as<uint32_t>(),
                                                  pos.as<uint32_t>(), nf, kd, ukeys, udeg, deg64.as<uint64_t>());
        SRDL_CHECK_LAUNCH();
        inclusive_scan_u64(deg64.as<uint64_t>(), uprefix, cap, s);
        if (k_dev) {  // asynchronous: (K_delta, K_union) stay on the device
            SRDL_CUDA(cudaMemcpyAsync(k_dev, kd, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            SRDL_CUDA(cudaMemcpyAsync(k_dev + 1, ku, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
            return;
        }
        uint32_t h[4] = {0, 0, 0, 0};
        SRDL_CUDA(cudaMemcpyAsync(h, kd, sizeof(h), cudaMemcpyDeviceToHost, s));
        SRDL_CUDA(cudaStreamSynchronize(s));
        *kd_out = h[0];
        *ku_out = h[2];
    }
}

extern "C" {

int srdl_max_id(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t *max_dev, void *stream) {
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_CUDA(cudaMemsetAsync(max_dev, 0, sizeof(uint32_t), s));
        if (n == 0) return;
        max_rows<<<stride_grid(n), kThreads, 0, s>>>(make_cols(cols, arity), arity, n, max_dev);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_key_fence(const uint32_t *keys, uint64_t n, uint32_t *fence, void *stream) {
    return guarded([&] {
        const uint64_t m = (n + SRDL_FENCE - 1) / SRDL_FENCE;
        if (m == 0) return;
        fence_kernel<<<stride_grid(m), kThreads, 0, (cudaStream_t)stream>>>(keys, m, fence);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_narrow_prefix(const uint32_t *const *cols, uint64_t n, const uint32_t *values,
                       uint32_t nvalues, uint64_t *lo, uint64_t *hi, void *stream) {
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_REQUIRE(nvalues <= SRDL_MAX_COLS, "too many constant columns");
        Scratch dv(sizeof(uint32_t) * SRDL_MAX_COLS + 2 * sizeof(uint64_t), s);
        uint32_t *vals = dv.as<uint32_t>();
        uint64_t *range = reinterpret_cast<uint64_t *>(vals + SRDL_MAX_COLS);
        SRDL_CUDA(cudaMemcpyAsync(vals, values, nvalues * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        narrow_prefix_kernel<<<1, 1, 0, s>>>(make_cols(cols, nvalues), n, vals, nvalues, range);
        SRDL_CHECK_LAUNCH();
        uint64_t h[2];
        SRDL_CUDA(cudaMemcpyAsync(h, range, sizeof(h), cudaMemcpyDeviceToHost, s));
        SRDL_CUDA(cudaStreamSynchronize(s));
        *lo = h[0];
        *hi = h[1];
    });
}

int srdl_root_work(const uint32_t *okeys, const uint32_t *odeg, const uint64_t *oprefix,
                   uint64_t nk, const uint32_t *ikeys, const uint32_t *ideg,
                   const uint64_t *iprefix, uint64_t nik, int has_inner, uint32_t *d2,
                   uint64_t *prefix, uint32_t *outer_lo, uint32_t *inner_lo, void *stream) {
    return guarded([&] {
        if (nk == 0) return;
        SRDL_REQUIRE(!outer_lo || oprefix, "outer_lo needs the outer prefix");
        SRDL_REQUIRE(!inner_lo || iprefix, "inner_lo needs the inner prefix");
        cudaStream_t s = (cudaStream_t)stream;
        root_work_kernel<<<stride_grid(nk), kThreads, 0, s>>>(okeys, odeg, oprefix, nk, ikeys, ideg,
                                                              iprefix, nik, has_inner, d2, prefix,
                                                              outer_lo, inner_lo);
        SRDL_CHECK_LAUNCH();
        inclusive_scan_u64(prefix, prefix, nk, s);
    });
}

int srdl_dense_offsets(const uint32_t *keys, const uint64_t *prefix, uint64_t nkeys,
                       uint32_t n_ids, uint32_t *off, void *stream) {
    return guarded([&] {
        cudaStream_t s = (cudaStream_t)stream;
        SRDL_REQUIRE(((uintptr_t)off & 15) == 0, "dense offsets buffer must be 16-byte aligned");
        dense_offsets_kernel<<<stride_grid(((uint64_t)n_ids + kIdsPerThread) / kIdsPerThread), kThreads, 0, s>>>(
            keys, prefix, nkeys, n_ids, off);
        SRDL_CHECK_LAUNCH();
    });
}

// rows owned by one rank, appended at `base` of out; returns the count
static uint64_t route_one(const Cols &in, uint32_t arity, uint64_t n, uint32_t key_col, uint32_t world,
                          uint32_t rank, const MutCols &out, uint64_t base, cudaStream_t s) {
    const unsigned g = stride_grid(n);
    Scratch f(n * sizeof(uint32_t), s), pos(n * sizeof(uint32_t), s), total(sizeof(uint32_t) * 2, s);
    owner_flags<<<g, kThreads, 0, s>>>(in.c[key_col], n, world, rank, f.as<uint32_t>());
    SRDL_CHECK_LAUNCH();
    exclusive_scan_u32(f.as<uint32_t>(), pos.as<uint32_t>(), n, total.as<uint32_t>(), s);
    scatter_flagged<<<g, kThreads, 0, s>>>(in, arity, f.as<uint32_t>(), pos.as<uint32_t>(), n, base, out);
    SRDL_CHECK_LAUNCH();
    uint32_t cnt = 0;
    SRDL_CUDA(cudaMemcpyAsync(&cnt, total.as<uint32_t>(), sizeof(cnt), cudaMemcpyDeviceToHost, s));
    SRDL_CUDA(cudaStreamSynchronize(s));
    return cnt;
}

int srdl_route_pack(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                    uint32_t world, uint32_t *send, uint64_t *counts_dev, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(world >= 1 && world <= 256 && key_col < arity && arity <= SRDL_MAX_COLS,
                     "bad routing arguments");
        SRDL_REQUIRE(n < (1ull << 32), "route: too many rows");
        cudaStream_t s = (cudaStream_t)stream;
        if (n == 0) {
            SRDL_CUDA(cudaMemsetAsync(counts_dev, 0, world * sizeof(uint64_t), s));
            return;
        }
        Scratch keys(n * sizeof(uint64_t), s), idx(n * sizeof(uint32_t), s);
        owner_keys<<<stride_grid(n), kThreads, 0, s>>>(cols[key_col], n, world, keys.as<uint64_t>(),
                                                       idx.as<uint32_t>());
        SRDL_CHECK_LAUNCH();
        // one stable radix pass on the owner (8 bits): rows grouped by rank,
        // in their original order within a rank
        radix_sort(keys.as<uint64_t>(), idx.as<uint32_t>(), n, 8, s);
        owner_counts<<<(world + 255) / 256, 256, 0, s>>>(keys.as<uint64_t>(), n, world, counts_dev);
        SRDL_CHECK_LAUNCH();
        pack_rows<<<stride_grid(n), kThreads, 0, s>>>(make_cols(cols, arity), arity, idx.as<uint32_t>(), n, send);
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_unpack_rows(const uint32_t *recv, uint32_t arity, uint64_t n, uint32_t *const *out, void *stream) {
    return guarded([&] {
        if (n == 0) return;
        unpack_rows<<<stride_grid(n), kThreads, 0, (cudaStream_t)stream>>>(recv, arity, n, make_mut(out, arity));
        SRDL_CHECK_LAUNCH();
    });
}

int srdl_route_rows(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                    uint32_t world, uint32_t *const *out, uint64_t *counts, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(world >= 1 && key_col < arity, "bad routing arguments");
        SRDL_REQUIRE(n < (1ull << 32), "route: too many rows");
        cudaStream_t s = (cudaStream_t)stream;
        uint64_t base = 0;
        for (uint32_t r = 0; r < world; ++r) {
            counts[r] = n ? route_one(make_cols(cols, arity), arity, n, key_col, world, r,
                                      make_mut(out, arity), base, s) : 0;
            base += counts[r];
        }
    });
}

int srdl_filter_owned(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                      uint32_t world, uint32_t rank, uint32_t *const *out, uint64_t *n_out,
                      void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(world >= 1 && rank < world && key_col < arity, "bad filter arguments");
        SRDL_REQUIRE(n < (1ull << 32), "filter: too many rows");
        *n_out = n ? route_one(make_cols(cols, arity), arity, n, key_col, world, rank,
                               make_mut(out, arity), 0, (cudaStream_t)stream) : 0;
    });
}

int srdl_root_own(const uint32_t *keys, uint64_t nk, const uint32_t *odeg, const uint32_t *d2,
                  uint32_t world, uint32_t rank, uint64_t *prefix, void *stream) {
    return guarded([&] {
        if (nk == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        root_own_kernel<<<stride_grid(nk), kThreads, 0, s>>>(keys, nk, odeg, d2, world, rank, prefix);
        SRDL_CHECK_LAUNCH();
        inclusive_scan_u64(prefix, prefix, nk, s);
    });
}

int srdl_gen_rmat(uint32_t scale, uint64_t nedges, float a, float b, float c, uint64_t seed,
                  uint32_t *src, uint32_t *dst, void *stream) {
    return guarded([&] {
        SRDL_REQUIRE(scale >= 1 && scale <= 32, "scale %u outside [1, 32]", scale);
        if (nedges == 0) return;
        cudaStream_t s = (cudaStream_t)stream;
        rmat_kernel<<<stride_grid(nedges), kThreads, 0, s>>>(scale, nedges, a, b, c, seed, src, dst);
        SRDL_CHECK_LAUNCH();
    });
}

}  // extern "C"
