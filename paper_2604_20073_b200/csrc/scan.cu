// Device-wide scans (reduce-then-scan, warp-striped tiles), error plumbing,
// stream-ordered scratch. Used by every counting / compaction step of the
// two-phase pipeline (Alg. 1 "offsets <- PrefixSum(tc)").
#include <stdarg.h>

#include <atomic>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace srdl {

// ------------------------------------------------------------------ errors

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launches() { return g_launches.load(std::memory_order_relaxed); }

// ----------------------------------------------------------------- scratch

// Scratch memory comes from a stack arena per (device, stream, host thread):
// every Scratch lives inside one C-ABI call (RAII, strictly nested), so
// allocation is a pointer bump and release a pop. Kernels of a later call
// from the same thread on the same stream run after the earlier call's
// kernels (stream order), so reusing the bytes is safe. Keying by thread as
// well keeps the stack discipline when several host threads share a stream
// (the legacy default stream, one stream pool for all engines): their calls
// interleave, but each thread's allocations stay nested in its own arena.
// Keying by device keeps a second GPU's scratch on that GPU. Blocks are
// cudaMalloc'ed when a stack outgrows its current block and kept for the
// process — no driver call per scratch buffer (cudaMallocAsync was measured
// to stall for ~0.5 s now and then under torch's expandable segments).
namespace {

struct Block {
    char *base;
    size_t size, used;
};

struct StreamArena {
    std::vector<Block> blocks;  // blocks[0..top] in use as a stack
    size_t top = 0;
};

struct ArenaKey {
    int dev;
    cudaStream_t stream;
    std::thread::id thread;
    bool operator==(const ArenaKey &o) const { return dev == o.dev && stream == o.stream && thread == o.thread; }
};

struct ArenaKeyHash {
    size_t operator()(const ArenaKey &k) const {
        return std::hash<void *>()((void *)k.stream) * 31u + std::hash<std::thread::id>()(k.thread) * 7u +
               (size_t)k.dev;
    }
};

std::mutex g_arena_mu;
std::unordered_map<ArenaKey, StreamArena, ArenaKeyHash> g_arenas;

constexpr size_t kAlign = 256;
constexpr size_t kMinBlock = size_t(64) << 20;

ArenaKey arena_key(cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    return ArenaKey{dev, s, std::this_thread::get_id()};
}

}  // namespace

Scratch::Scratch(size_t bytes, cudaStream_t s) : stream_(s) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + kAlign - 1) & ~(kAlign - 1);
    const ArenaKey key = arena_key(s);
    dev_ = key.dev;
    std::lock_guard<std::mutex> lock(g_arena_mu);
    StreamArena &A = g_arenas[key];
    // current block, else the next existing block with room, else a new one
    while (A.top < A.blocks.size() && A.blocks[A.top].size - A.blocks[A.top].used < bytes) {
        if (A.blocks[A.top].used == 0 && A.top + 1 >= A.blocks.size()) break;
        ++A.top;
    }
    if (A.top >= A.blocks.size() || A.blocks[A.top].size - A.blocks[A.top].used < bytes) {
        size_t want = bytes > kMinBlock ? bytes : kMinBlock;
        if (!A.blocks.empty() && want < 2 * A.blocks.back().size) want = 2 * A.blocks.back().size;
        if (want < bytes) want = bytes;
        void *p = nullptr;
        SRDL_CUDA(cudaMalloc(&p, want));
        A.blocks.push_back(Block{(char *)p, want, 0});
        A.top = A.blocks.size() - 1;
    }
    Block &b = A.blocks[A.top];
    ptr_ = b.base + b.used;
    bytes_ = bytes;
    block_ = A.top;
    b.used += bytes;
}

Scratch::~Scratch() {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    StreamArena &A = g_arenas[ArenaKey{dev_, stream_, std::this_thread::get_id()}];
    Block &b = A.blocks[block_];
    if ((char *)ptr_ + bytes_ != b.base + b.used) {
        // not the newest allocation of its block: the stack discipline was
        // broken (a Scratch moved across threads). Keep the bytes reserved
        // rather than hand live memory out again; the block is reclaimed
        // once everything above it is released.
        set_error("scratch arena released out of order (kept reserved)");
        return;
    }
    b.used -= bytes_;
    while (A.top > 0 && A.blocks[A.top].used == 0) --A.top;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

bool first_use_on_device(uint64_t *mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    std::lock_guard<std::mutex> lock(g_arena_mu);
    if (*mask & bit) return false;
    *mask |= bit;
    return true;
}

uint64_t read_u64(const uint64_t *dev, cudaStream_t s) {
    uint64_t v = 0;
    SRDL_CUDA(cudaMemcpyAsync(&v, dev, sizeof(v), cudaMemcpyDeviceToHost, s));
    SRDL_CUDA(cudaStreamSynchronize(s));
    return v;
}

// ------------------------------------------------------------------- scans

// Tile = 8 warps x 16 rounds x 32 lanes; element (w, r, l) is at
// tile_base + w*512 + r*32 + l, so each warp owns a contiguous chunk and
// every round is a coalesced 32-wide access.
constexpr int kWarps = kThreads / 32;
constexpr int kWarpChunk = 32 * kItems;

template <class T>
__global__ void __launch_bounds__(kThreads) tile_reduce(const T *__restrict__ in, uint64_t n,
                                                        T *__restrict__ partial) {
    __shared__ T wsum[kWarps];
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    T acc = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        uint64_t i = base + (uint64_t)w * kWarpChunk + r * 32 + l;
        if (i < n) acc += in[i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (l == 0) wsum[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int k = 0; k < kWarps; ++k) t += wsum[k];
        partial[blockIdx.x] = t;
    }
}

// Exclusive scan of one tile with an incoming block offset.
template <class T, bool EXCLUSIVE>
__global__ void __launch_bounds__(kThreads) tile_scan(const T *__restrict__ in, T *__restrict__ out,
                                                      uint64_t n, const T *__restrict__ offsets,
                                                      T *__restrict__ total) {
    __shared__ T wsum[kWarps];
    __shared__ T wbase[kWarps];
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    T v[kItems];
    T carry = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        uint64_t i = base + (uint64_t)w * kWarpChunk + r * 32 + l;
        T x = i < n ? in[i] : T(0);
        T s = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += y;
        }
        v[r] = carry + (EXCLUSIVE ? s - x : s);
        carry += __shfl_sync(0xffffffffu, s, 31);
    }
    if (l == 0) wsum[w] = carry;
    __syncthreads();
    if (threadIdx.x == 0) {
        T run = offsets ? offsets[blockIdx.x] : T(0);
        for (int k = 0; k < kWarps; ++k) {
            wbase[k] = run;
            run += wsum[k];
        }
        if (total && blockIdx.x == gridDim.x - 1) *total = run;
    }
    __syncthreads();
    const T add = wbase[w];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        uint64_t i = base + (uint64_t)w * kWarpChunk + r * 32 + l;
        if (i < n) out[i] = v[r] + add;
    }
}

template <class T>
__global__ void write_zero(T *p) {
    *p = 0;
}

// Single-pass scan (chained scan with decoupled look-back, Merrill &
// Garland): tile t scans its 4096 elements, publishes its aggregate, warp 0
// looks back over the preceding tiles' published aggregates / inclusive
// prefixes 32 at a time, and the tile writes its outputs — one launch
// instead of reduce + scan-of-partials + scan. The status words carry a
// per-call epoch, so the persistent status buffer (per device / stream /
// thread) is never cleared: a stale word from an earlier call has a smaller
// epoch and reads as "not published".
constexpr uint64_t kStAgg = 1, kStInc = 2;

template <class T>
__device__ __forceinline__ T wsum_total(const T *wsum) {
    T t = 0;
    for (int k = 0; k < kWarps; ++k) t += wsum[k];
    return t;
}

template <class T, bool EXCLUSIVE>
__global__ void __launch_bounds__(kThreads)
    chained_scan(const T *__restrict__ in, T *__restrict__ out, uint64_t n, T *__restrict__ total,
                 uint64_t *status, uint64_t *value, uint64_t cap, uint64_t epoch,
                 const uint64_t *__restrict__ bound) {
    __shared__ T wsum[kWarps];
    __shared__ T wbase[kWarps];
    __shared__ uint64_t tile_excl;
    const uint64_t tile = blockIdx.x;  // blocks are dispatched in index order
    const uint64_t base = tile * kTile;
    // bound (device word, optional): scan only [0, min(n, *bound)); tiles
    // past it return before publishing (no later tile looks back on them)
    if (bound) {
        const uint64_t b = *bound;
        if (b < n) n = b;
        if (n == 0) {
            if (total && tile == 0 && threadIdx.x == 0) *total = 0;
            return;
        }
        if (base >= n) return;
    }
    const uint64_t last_tile = (n - 1) / kTile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    T x[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const uint64_t i = base + (uint64_t)w * kWarpChunk + r * 32 + l;
        x[r] = i < n ? in[i] : T(0);
    }
    T v[kItems];
    T carry = 0;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        T s = x[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += y;
        }
        v[r] = carry + (EXCLUSIVE ? s - x[r] : s);
        carry += __shfl_sync(0xffffffffu, s, 31);
    }
    if (l == 0) wsum[w] = carry;
    __syncthreads();
    if (w == 0) {
        T agg = 0;
        if (l == 0) {
            T run = 0;
            for (int k = 0; k < kWarps; ++k) {
                wbase[k] = run;
                run += wsum[k];
            }
            agg = run;
            // aggregate and inclusive prefix live in separate words (value[t]
            // and value[cap + t]): a reader that saw "aggregate" must not read
            // a word the tile has meanwhile overwritten with its inclusive sum
            value[tile] = (uint64_t)run;
            if (tile == 0) value[cap + tile] = (uint64_t)run;
            __threadfence();
            *(volatile uint64_t *)(status + tile) = (epoch << 2) | (tile == 0 ? kStInc : kStAgg);
        }
        agg = __shfl_sync(0xffffffffu, agg, 0);
        uint64_t excl = 0;
        if (tile > 0) {
            // look back 32 tiles at a time: lane j inspects tile t - j
            int64_t t = (int64_t)tile - 1;
            while (true) {
                const int64_t mine = t - l;
                uint64_t st = 0, val = 0;
                if (mine >= 0) {
                    do {
                        st = *(volatile uint64_t *)(status + mine);
                    } while ((st >> 2) != epoch);
                    __threadfence();
                    val = *(volatile uint64_t *)(value + ((st & 3) == kStInc ? cap : 0) + mine);
                } else {
                    st = (epoch << 2) | kStInc;  // before tile 0: empty inclusive prefix
                }
                const uint32_t inc = __ballot_sync(0xffffffffu, (st & 3) == kStInc);
                const int first = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive tile
                uint64_t part = l <= first ? val : 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (inc) break;
                t -= 32;
            }
            if (l == 0) {
                value[cap + tile] = excl + (uint64_t)agg;
                __threadfence();
                *(volatile uint64_t *)(status + tile) = (epoch << 2) | kStInc;
            }
        }
        if (l == 0) tile_excl = excl;
    }
    __syncthreads();
    const T add = wbase[w] + (T)tile_excl;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const uint64_t i = base + (uint64_t)w * kWarpChunk + r * 32 + l;
        if (i < n) out[i] = v[r] + add;
    }
    if (total && tile == last_tile && threadIdx.x == 0) *total = (T)(tile_excl + wsum_total(wsum));
}

namespace {

// persistent look-back status of one (device, stream, thread): grown, never cleared
struct ScanState {
    uint64_t *status = nullptr, *value = nullptr;
    size_t cap = 0;
    uint64_t epoch = 0;
};

std::mutex g_scan_mu;
std::unordered_map<ArenaKey, ScanState, ArenaKeyHash> g_scan;

ScanState &scan_state(cudaStream_t s, size_t tiles) {
    const ArenaKey key = arena_key(s);
    std::lock_guard<std::mutex> lock(g_scan_mu);
    ScanState &st = g_scan[key];
    if (st.cap < tiles) {
        // the old buffers may still be read by queued scans of this stream:
        // they are leaked rather than freed (a few growth steps per process)
        size_t cap = st.cap ? st.cap : 1024;
        while (cap < tiles) cap *= 2;
        SRDL_CUDA(cudaMalloc(&st.status, cap * sizeof(uint64_t)));
        SRDL_CUDA(cudaMalloc(&st.value, 2 * cap * sizeof(uint64_t)));  // aggregates, inclusive prefixes
        SRDL_CUDA(cudaMemsetAsync(st.status, 0, cap * sizeof(uint64_t), s));  // epoch 0 = never published
        st.cap = cap;
    }
    return st;
}

// persistent per-(tile, digit) look-back status of the onesweep radix passes
// (sort.cu), per (device, stream, thread); epoch-stamped like the scan's
struct SortStatus {
    uint64_t *words = nullptr;
    size_t cap = 0;
    uint32_t epoch = 0;
};
std::unordered_map<ArenaKey, SortStatus, ArenaKeyHash> g_sort_status;

}  // namespace

uint64_t *onesweep_status(cudaStream_t s, size_t words, uint32_t *epoch) {
    const ArenaKey key = arena_key(s);
    std::lock_guard<std::mutex> lock(g_scan_mu);
    SortStatus &st = g_sort_status[key];
    if (st.cap < words) {
        // old buffers may still be read by queued passes of this stream: leaked
        size_t cap = st.cap ? st.cap : (size_t)1 << 16;
        while (cap < words) cap *= 2;
        SRDL_CUDA(cudaMalloc(&st.words, cap * sizeof(uint64_t)));
        SRDL_CUDA(cudaMemsetAsync(st.words, 0, cap * sizeof(uint64_t), s));  // epoch 0: never published
        st.cap = cap;
        st.epoch = 0;
    }
    if (++st.epoch >= kOnesweepEpochs) {  // the 30-bit epoch wrapped: start over from a clear buffer
        SRDL_CUDA(cudaMemsetAsync(st.words, 0, st.cap * sizeof(uint64_t), s));
        st.epoch = 1;
    }
    *epoch = st.epoch;
    return st.words;
}

template <class T, bool EXCLUSIVE>
static void scan_impl(const T *in, T *out, uint64_t n, T *total, cudaStream_t s, const uint64_t *bound = nullptr) {
    if (n && bound) {  // the element count is only known on the device: the chained kernel always
        const uint64_t blocks = (n + kTile - 1) / kTile;
        ScanState &st = scan_state(s, blocks);
        const uint64_t epoch = ++st.epoch;
        chained_scan<T, EXCLUSIVE><<<(unsigned)blocks, kThreads, 0, s>>>(in, out, n, total, st.status, st.value,
                                                                           st.cap, epoch, bound);
        SRDL_CHECK_LAUNCH();
        return;
    }
    if (n == 0) {
        if (total) {
            write_zero<T><<<1, 1, 0, s>>>(total);
            SRDL_CHECK_LAUNCH();
        }
        return;
    }
    const uint64_t blocks = (n + kTile - 1) / kTile;
    if (blocks == 1) {
        tile_scan<T, EXCLUSIVE><<<1, kThreads, 0, s>>>(in, out, n, nullptr, total);
        SRDL_CHECK_LAUNCH();
        return;
    }
    ScanState &st = scan_state(s, blocks);
    const uint64_t epoch = ++st.epoch;
    chained_scan<T, EXCLUSIVE><<<(unsigned)blocks, kThreads, 0, s>>>(in, out, n, total, st.status, st.value, st.cap,
                                                                       epoch, nullptr);
    SRDL_CHECK_LAUNCH();
}

void exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *total,
                        cudaStream_t s) {
    scan_impl<uint64_t, true>(in, out, n, total, s);
}
void exclusive_scan_u64_bounded(const uint64_t *in, uint64_t *out, uint64_t n, const uint64_t *bound,
                                uint64_t *total, cudaStream_t s) {
    scan_impl<uint64_t, true>(in, out, n, total, s, bound);
}
void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, uint32_t *total,
                        cudaStream_t s) {
    scan_impl<uint32_t, true>(in, out, n, total, s);
}
void inclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, cudaStream_t s) {
    scan_impl<uint64_t, false>(in, out, n, nullptr, s);
}

}  // namespace srdl

extern "C" {

int srdl_version(void) { return SRDL_VERSION; }

// Device-wide scans (the two-phase allocation's offsets, reference
// executor.py:516-524 np.cumsum of the per-slice counts), exposed for tests.
int srdl_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, int exclusive, uint32_t *total, void *stream) {
    return srdl::guarded([&] {
        SRDL_REQUIRE(exclusive || total == nullptr, "an inclusive scan has no separate total");
        if (exclusive)
            srdl::exclusive_scan_u32(in, out, n, total, (cudaStream_t)stream);
        else
            srdl::scan_impl<uint32_t, false>(in, out, n, nullptr, (cudaStream_t)stream);
    });
}

int srdl_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, int exclusive, uint64_t *total, void *stream) {
    return srdl::guarded([&] {
        SRDL_REQUIRE(exclusive || total == nullptr, "an inclusive scan has no separate total");
        if (exclusive)
            srdl::exclusive_scan_u64(in, out, n, total, (cudaStream_t)stream);
        else
            srdl::inclusive_scan_u64(in, out, n, (cudaStream_t)stream);
    });
}

uint64_t srdl_launch_count(void) { return srdl::launches(); }

// Stream ordering for the fork-join phases of the stream schedule: work
// launched on `waiter` after this call starts after everything launched on
// `signaler` before it. One record + wait on an event from a per-(device,
// thread) ring; a wait captures the event's state when it is enqueued, so
// re-recording a ring slot later never affects it. torch's Stream.wait_stream
// costs ~7 us of Python per call, thousands of times per fixpoint.
int srdl_stream_wait(void *waiter, void *signaler) {
    return srdl::guarded([&] {
        constexpr int kRing = 64;
        struct Ring {
            int device = -1;
            cudaEvent_t ev[kRing] = {};
            unsigned next = 0;
        };
        static thread_local Ring rings[16];
        int d = 0;
        SRDL_CUDA(cudaGetDevice(&d));
        SRDL_REQUIRE(d >= 0 && d < 16, "device %d", d);
        Ring &r = rings[d];
        if (r.device != d) {
            for (auto &e : r.ev) SRDL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            r.device = d;
        }
        cudaEvent_t e = r.ev[r.next++ % kRing];
        SRDL_CUDA(cudaEventRecord(e, (cudaStream_t)signaler));
        SRDL_CUDA(cudaStreamWaitEvent((cudaStream_t)waiter, e, 0));
    });
}

const char *srdl_last_error(void) { return srdl::g_err; }

int srdl_sm_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        srdl::set_error("no CUDA device visible");
        return SRDL_ERR_CUDA;
    }
    return srdl::sm_count();
}

}  // extern "C"
