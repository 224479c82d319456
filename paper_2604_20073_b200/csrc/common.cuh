// Shared plumbing for libsrdl: error reporting, stream-ordered scratch,
// launch geometry and small device helpers. Target: sm_100a (B200).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "srdl.h"

namespace srdl {

// ------------------------------------------------------------------ errors

void set_error(const char *fmt, ...);

struct Fail {
    int code;
};

#define SRDL_CUDA(expr)                                                                   \
    do {                                                                                  \
        cudaError_t err_ = (expr);                                                        \
        if (err_ != cudaSuccess) {                                                        \
            ::srdl::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                  \
                              cudaGetErrorString(err_));                                  \
            throw ::srdl::Fail{SRDL_ERR_CUDA};                                            \
        }                                                                                 \
    } while (0)

// every kernel launch in the library is followed by this check, which also
// feeds srdl_launch_count() (the benchmark's gpu_launches figure)
void note_launch();
#define SRDL_CHECK_LAUNCH()          \
    do {                             \
        ::srdl::note_launch();       \
        SRDL_CUDA(cudaGetLastError()); \
    } while (0)

#define SRDL_REQUIRE(cond, ...)                                                           \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            ::srdl::set_error(__VA_ARGS__);                                               \
            throw ::srdl::Fail{SRDL_ERR_ARG};                                             \
        }                                                                                 \
    } while (0)

// Wrap a C-ABI body: exceptions become return codes.
template <class F>
int guarded(F &&f) {
    try {
        f();
        return SRDL_OK;
    } catch (const Fail &e) {
        return e.code;
    } catch (...) {
        set_error("unexpected C++ exception");
        return SRDL_ERR_INTERNAL;
    }
}

// --------------------------------------------------------- scratch memory

// Stream-ordered scratch buffer from the stack arena of (device, stream,
// host thread) in scan.cu: strictly nested inside one C-ABI call.
class Scratch {
  public:
    Scratch(size_t bytes, cudaStream_t s);
    ~Scratch();
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    template <class T>
    T *as() const {
        return reinterpret_cast<T *>(ptr_);
    }

  private:
    void *ptr_ = nullptr;
    cudaStream_t stream_;
    int dev_ = 0;
    size_t bytes_ = 0;
    size_t block_ = 0;
};

int sm_count();  // of the current device (cached per device)

// true the first time it is called for the current device with this mask
// (per-device one-time setup such as cudaFuncSetAttribute)
bool first_use_on_device(uint64_t *mask);

// Host-visible read of a device scalar (synchronises the stream).
uint64_t read_u64(const uint64_t *dev, cudaStream_t s);

// ----------------------------------------------------------------- launch

constexpr int kThreads = 256;
constexpr int kItems = 16;  // items per thread for tiled kernels
constexpr int kTile = kThreads * kItems;

inline unsigned grid_for(uint64_t n, int per_block) {
    uint64_t g = (n + per_block - 1) / per_block;
    return (unsigned)(g == 0 ? 1 : g);
}

// grid-stride launch size: a few waves over the SMs
inline unsigned stride_grid(uint64_t n, int threads = kThreads) {
    uint64_t need = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)sm_count() * 8;
    if (need > cap) need = cap;
    return (unsigned)(need == 0 ? 1 : need);
}

// Column-pointer bundle passed by value to kernels.
struct Cols {
    const uint32_t *c[SRDL_MAX_COLS];
};
struct MutCols {
    uint32_t *c[SRDL_MAX_COLS];
};

inline Cols make_cols(const uint32_t *const *p, uint32_t arity) {
    Cols k{};
    for (uint32_t i = 0; i < arity; ++i) k.c[i] = p[i];
    return k;
}
inline MutCols make_mut(uint32_t *const *p, uint32_t arity) {
    MutCols k{};
    for (uint32_t i = 0; i < arity; ++i) k.c[i] = p[i];
    return k;
}

// ---------------------------------------------------------- device helpers

// lexicographic compare of row i of A with row j of B: -1, 0, 1
__device__ __forceinline__ int row_cmp(const Cols &A, uint64_t i, const Cols &B, uint64_t j,
                                       uint32_t arity) {
    for (uint32_t c = 0; c < arity; ++c) {
        uint32_t x = __ldg(A.c[c] + i), y = __ldg(B.c[c] + j);
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// first index in [lo, hi) of sorted rows B whose row is >= (strict=false) or
// > (strict=true) row i of A
__device__ __forceinline__ uint64_t row_bound(const Cols &B, uint64_t lo, uint64_t hi,
                                              const Cols &A, uint64_t i, uint32_t arity,
                                              bool strict) {
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        int c = row_cmp(B, mid, A, i, arity);
        if (c < 0 || (strict && c == 0))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

}  // namespace srdl

// Scan primitives (scan.cu)
namespace srdl {
// exclusive scan of n values; writes out[n] and optionally the total to
// total_dev (device pointer, may be null). in and out may alias.
void exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *total_dev,
                        cudaStream_t s);
// the same over the first min(n, *bound) values, bound a device word (the
// count is produced by an earlier kernel of the stream; no host round trip)
void exclusive_scan_u64_bounded(const uint64_t *in, uint64_t *out, uint64_t n, const uint64_t *bound,
                                uint64_t *total_dev, cudaStream_t s);
void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, uint32_t *total_dev,
                        cudaStream_t s);
// the onesweep passes' (tile, digit) look-back words, persistent per
// (device, stream, thread) and never cleared: every pass gets a fresh epoch
// (1 .. kOnesweepEpochs - 1) that its words carry in bits 32-61
constexpr uint32_t kOnesweepEpochs = 1u << 30;
uint64_t *onesweep_status(cudaStream_t s, size_t words, uint32_t *epoch);
void inclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, cudaStream_t s);
// stable radix sort of keys (and optional 32-bit values) on key bits
// [lo_bit, lo_bit + bits); results land back in keys/vals.
void radix_sort(uint64_t *keys, uint32_t *vals, uint64_t n, uint32_t bits, cudaStream_t s,
                const int *unsorted = nullptr, uint32_t lo_bit = 0);
}  // namespace srdl
