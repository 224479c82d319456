// Histogram-guided, warp-cooperative worst-case-optimal join (paper Alg. 1
// phases 2-3 and Alg. 2; reference executor.count_pass / materialize_pass /
// _run_slice / _root_setup / _descend, executor.py:342-485) — the device
// code, templated on the plan's SHAPE.
//
// The shape of a plan (its depth, atoms, which atom binds which index
// columns at which level, negations, the head projection) is a policy type:
//   * DynShape reads it from the srdl_plan descriptor at run time — the
//     generic kernels compiled into libsrdl.so (wcoj.cu), one per plan class;
//   * a generated shape type (wcoj_jit.cu) returns compile-time constants —
//     the per-rule kernel the paper's compiler emits ("translates high-level
//     rules into a staged pipeline of CUDA kernels rather than interpreting
//     queries at runtime"): NVRTC compiles this header once
//     per distinct plan shape, the shape-bounded loops unroll, the atom
//     properties fold into the code, and only the index pointers, row
//     ranges and segment counts stay run-time data.
//
// Work decomposition. The root level is flattened into T = sum_k outer(k) *
// d2(k) units (prefix array C) and cut into p equal slices [s*ceil(T/p), ...)
// (Alg. 2 "block b's slice"); p is many times the number of resident warps
// and warps fetch slice indexes from a ticket counter (one global atomic per
// slice), so cost variance between slices evens out. A slice finds its first
// key by binary search on C (kappa) and is walked as at most three
// (outer rows x inner rows) rectangles per key, exactly the Fig. 2 scheme.
// Output offsets are per slice, so results do not depend on which warp ran
// which slice.
//
// Inside a rectangle the warp runs leapfrog-style generic join over the
// remaining levels with all 32 lanes cooperating:
//   * candidates of a level come 32 at a time from the source with the
//     smallest narrowed range (run starts = distinct values), every lane
//     narrows the other sources for its own candidate by binary search, and
//     a ballot keeps the survivors;
//   * levels 1..m-4 descend survivor by survivor (DFS state in shared memory,
//     sized per plan); for m >= 4 the survivors of level m-3 are expanded
//     over their level m-2 candidates in flattened chunks (mid batch);
//   * the last two levels are flattened: the survivors of level m-2 become a
//     batch of up to 32 parents, their leaf candidate ranges are prefix-summed
//     across the warp and all lanes walk the concatenated ranges, so a leaf
//     with short fan-out still keeps the warp full and output writes stay
//     coalesced (the paper's "adjacent threads emit adjacent positions").
// Count and materialize run the same code (template flag MODE), so per-slice
// counts are exact and writes land in [offset_s, offset_s + count_s). The
// speculative mode (kSpec) also writes every tuple into arena chunks
// reserved with one global atomic per 128-tuple chunk.
#pragma once

#ifdef __CUDACC_RTC__
#include "srdl.h"
#else
#include "common.cuh"
#endif

// Loop policies. SRDL_LOOP: loops whose trip count is data (rows, chunks)
// stay rolled (the kernel is latency-bound and its hot loops must stay in
// the instruction cache). SRDL_SHAPE_LOOP: loops over the plan's shape
// (atoms of a level, head columns): rolled in the generic kernels, fully
// unrolled in the per-plan kernels, where their bounds are constants.
#ifndef SRDL_UNROLL_LOOPS
#define SRDL_LOOP _Pragma("unroll 1")
#else
#define SRDL_LOOP
#endif
#ifdef SRDL_JIT
#define SRDL_SHAPE_LOOP _Pragma("unroll")
#else
#define SRDL_SHAPE_LOOP SRDL_LOOP
#endif
#ifdef SRDL_NOINLINE_SEARCH
#define SRDL_SEARCH __device__ __noinline__
#else
#define SRDL_SEARCH __device__ __forceinline__
#endif

namespace srdl {

#ifdef __CUDACC_RTC__
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
#endif

#ifndef SRDL_JOIN_WARPS
#define SRDL_JOIN_WARPS 4
#endif
constexpr int kJoinWarps = SRDL_JOIN_WARPS;  // warps per CTA (each runs its own slices)
#ifndef SRDL_MIN_BLOCKS
#define SRDL_MIN_BLOCKS 8
#endif
constexpr int kMinBlocks = SRDL_MIN_BLOCKS;  // register budget: 64K / (8 * 128) = 64 registers per thread
constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kSegs = SRDL_MAX_SEGS;
// merge-path leaves: both lists at least kMergeMin long and within a factor
// kMergeRatio of each other (otherwise per-candidate binary search)
#ifndef SRDL_MERGE_MIN
#define SRDL_MERGE_MIN 64
#endif
#ifndef SRDL_MERGE_SKIP  // merge-path tiles: skip a tile that lies wholly below the other (A/B knob)
#define SRDL_MERGE_SKIP 0
#endif
#ifndef SRDL_MERGE_RATIO
#define SRDL_MERGE_RATIO 4
#endif
constexpr uint32_t kMergeMin = SRDL_MERGE_MIN;
constexpr uint32_t kMergeRatio = SRDL_MERGE_RATIO;

// Plan classes (each generic instance carries only the code paths its plans
// can reach). kShallow: depth <= 2; kDepth3: depth 3, level 1 feeds leaf
// batches; kDepth4Mid: depth 4 with a mid batch, level 1 feeds mid batches;
// kGeneral: anything (DFS over the middle levels).
enum Kind : int { kShallow = 0, kDepth3 = 1, kGeneral = 2, kDepth4Mid = 3 };

// kCount: count only; kMaterialize: write at exact offsets (second walk);
// kSpec: count and write speculatively into arena chunks (srdl_spec).
enum Mode : int { kCount = 0, kMaterialize = 1, kSpec = 2 };
constexpr uint32_t kNoChunk = 0xffffffffu;

__host__ __device__ inline int plan_class(uint32_t depth, uint32_t nmid) {
    if (depth <= 2) return kShallow;
    if (depth == 3 && nmid == 0) return kDepth3;
    if (depth == 4 && nmid) return kDepth4Mid;
    return kGeneral;
}

// The plan shape read from the descriptor (generic kernels).
struct DynShape {
    static __device__ __forceinline__ uint32_t depth(const srdl_plan &P) { return P.depth; }
    static __device__ __forceinline__ uint32_t natoms(const srdl_plan &P) { return P.natoms; }
    static __device__ __forceinline__ uint32_t outer(const srdl_plan &P) { return P.outer; }
    static __device__ __forceinline__ uint32_t inner(const srdl_plan &P) { return P.inner; }
    static __device__ __forceinline__ uint32_t head_arity(const srdl_plan &P) { return P.head_arity; }
    static __device__ __forceinline__ int head_level(const srdl_plan &P, uint32_t h) { return P.head_level[h]; }
    static __device__ __forceinline__ uint32_t nspec(const srdl_plan &P, int L) { return P.nspec[L]; }
    static __device__ __forceinline__ uint32_t spec(const srdl_plan &P, int L, uint32_t j) { return P.spec[L][j]; }
    static __device__ __forceinline__ uint32_t leaf_slot(const srdl_plan &P, uint32_t a) { return P.leaf_slot[a]; }
    static __device__ __forceinline__ uint32_t mid_slot(const srdl_plan &P, uint32_t a) { return P.mid_slot[a]; }
    static __device__ __forceinline__ uint32_t nmid(const srdl_plan &P) { return P.nmid; }
    static __device__ __forceinline__ bool negated(const srdl_plan &P, uint32_t a) { return P.atom[a].negated != 0; }
    static __device__ __forceinline__ int check_level(const srdl_plan &P, uint32_t a) { return P.atom[a].check_level; }
    static __device__ __forceinline__ uint32_t lvl_col(const srdl_plan &P, uint32_t a, int L) {
        return P.atom[a].lvl_col[L];
    }
    static __device__ __forceinline__ uint32_t lvl_ncol(const srdl_plan &P, uint32_t a, int L) {
        return P.atom[a].lvl_ncol[L];
    }
};

struct Rng {
    uint32_t lo, hi;
};

// Per-warp DFS state in dynamic shared memory, sized for the plan at hand
// (depth D, atoms A, leaf sources NL, mid-batch sources NM) so small plans
// do not pay for the worst-case footprint.
struct View {
    uint64_t *leaf_pref;  // [33] exclusive prefix of parent leaf lengths
    uint64_t *mid_pref;   // [33] exclusive prefix of grandparent candidate lengths
    uint64_t *wpre;       // [33] staged root keys: wpre[0] = prefix before the window, then 32 prefixes
    uint32_t *wroot;      // [5 * 32] staged d2, key, outer row, outer degree, inner row
    Rng *rng;             // [(D+1) * A * 2] ranges on entry of level L
    Rng *leaf;            // [32 * NL * 2] per-parent leaf ranges
    Rng *mid;             // [32 * NM * 2] per-grandparent ranges of deep atoms
    uint32_t *vals;       // [D * 32] candidates of the current chunk per level
    uint32_t *bind;       // [D] bound values (serial DFS levels)
    uint32_t *cur;        // [D] next driver row per level
    uint32_t *mask;       // [D] survivors not yet descended
    uint8_t *drv, *dseg;  // [D] driver atom and segment per level
    uint8_t *leaf_drv;    // [32]
    uint8_t *mid_drv;     // [32]
    uint8_t *gp;          // [32] grandparent lane of each mid-batch parent
    uint32_t *gp_active;  // [1] parents come from a mid batch
    uint32_t A, NL, NM;

    __device__ __forceinline__ Rng &R(int L, uint32_t a, uint32_t s) const {
        return rng[((L * A + a) << 1) + s];
    }
    __device__ __forceinline__ Rng &LF(uint32_t p, uint32_t j, uint32_t s) const {
        return leaf[((p * NL + j) << 1) + s];
    }
    __device__ __forceinline__ Rng &MD(uint32_t g, uint32_t j, uint32_t s) const {
        return mid[((g * NM + j) << 1) + s];
    }
    __device__ __forceinline__ uint32_t &V(int L, uint32_t lane) const { return vals[L * 32 + lane]; }
};

__host__ __device__ inline size_t warp_bytes(uint32_t D, uint32_t A, uint32_t NL, uint32_t NM) {
    size_t b = 2 * 33 * 8;                          // prefixes
    b += 33 * 8 + 5 * 32 * 4;                       // root-key window
    b += (size_t)(D + 1) * A * 2 * sizeof(Rng);     // rng
    b += (size_t)32 * NL * 2 * sizeof(Rng);         // leaf
    b += (size_t)32 * NM * 2 * sizeof(Rng);         // mid
    b += (size_t)D * 32 * 4 + (size_t)3 * D * 4;    // vals, bind, cur, mask
    b += (size_t)2 * D + 3 * 32 + 4;                // drv, dseg, leaf_drv, mid_drv, gp, flag
    return (b + 15) & ~(size_t)15;
}

__device__ __forceinline__ View make_view(unsigned char *base, uint32_t D, uint32_t A, uint32_t NL,
                                          uint32_t NM) {
    View v;
    v.A = A;
    v.NL = NL;
    v.NM = NM;
    unsigned char *p = base;
    v.leaf_pref = (uint64_t *)p;
    p += 33 * 8;
    v.mid_pref = (uint64_t *)p;
    p += 33 * 8;
    v.wpre = (uint64_t *)p;
    p += 33 * 8;
    v.wroot = (uint32_t *)p;
    p += 5 * 32 * 4;
    v.rng = (Rng *)p;
    p += (size_t)(D + 1) * A * 2 * sizeof(Rng);
    v.leaf = (Rng *)p;
    p += (size_t)32 * NL * 2 * sizeof(Rng);
    v.mid = (Rng *)p;
    p += (size_t)32 * NM * 2 * sizeof(Rng);
    v.vals = (uint32_t *)p;
    p += (size_t)D * 32 * 4;
    v.bind = (uint32_t *)p;
    p += D * 4;
    v.cur = (uint32_t *)p;
    p += D * 4;
    v.mask = (uint32_t *)p;
    p += D * 4;
    v.gp_active = (uint32_t *)p;
    p += 4;
    v.drv = p;
    p += D;
    v.dseg = p;
    p += D;
    v.leaf_drv = p;
    p += 32;
    v.mid_drv = p;
    p += 32;
    v.gp = p;
    return v;
}

SRDL_SEARCH uint32_t lbound(const uint32_t *__restrict__ col, uint32_t lo, uint32_t hi, uint32_t v) {
    while (lo < hi) {
        uint32_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(col + mid) < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

SRDL_SEARCH uint32_t ubound(const uint32_t *__restrict__ col, uint32_t lo, uint32_t hi, uint32_t v) {
    while (lo < hi) {
        uint32_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(col + mid) <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Column-0 lookup through the index histogram: binary search over the K
// distinct keys (a few MB, L2-resident) instead of the n rows, through the
// fence keys first (every SRDL_FENCE-th key, L1-resident), then one block.
__device__ __forceinline__ void hist_range(const srdl_atom &A, uint32_t v, Rng &r) {
    uint32_t lo = 0, hi = A.hk;
    if (A.hfence) {
        uint32_t flo = 0, fhi = A.hfn;
        while (flo < fhi) {
            const uint32_t mid = (flo + fhi) >> 1;
            if (__ldg(A.hfence + mid) <= v)
                flo = mid + 1;
            else
                fhi = mid;
        }
        // keys[(flo-1) * F] <= v < keys[flo * F]: one block of hkeys left
        if (flo == 0) {
            r.hi = r.lo;
            return;
        }
        lo = (flo - 1) * SRDL_FENCE;
        hi = min(A.hk, flo * SRDL_FENCE);
    }
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(A.hkeys + mid) < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    if (lo < A.hk && __ldg(A.hkeys + lo) == v) {
        r.lo = lo ? (uint32_t)__ldg(A.hprefix + lo - 1) : 0u;
        r.hi = (uint32_t)__ldg(A.hprefix + lo);
    } else {
        r.hi = r.lo;
    }
}

// Column-0 range of value v: dense CSR offsets (two loads) or the histogram.
SRDL_SEARCH void col0_range(const srdl_atom &A, uint32_t v, Rng &r) {
    if (A.doff) {
        if (v < A.dn) {
            r.lo = __ldg(A.doff + v);
            r.hi = __ldg(A.doff + v + 1);
        } else {
            r.hi = r.lo;
        }
    } else {
        hist_range(A, v, r);
    }
}

// Narrow r (rows of segment s of atom a) to rows whose level-L columns all
// equal v. Returns the new length (0 = no match).
template <class SH>
SRDL_SEARCH uint32_t narrow(const srdl_plan &P, uint32_t a, int s, int L, uint32_t v, Rng &r) {
    const srdl_atom &A = P.atom[a];
    const uint32_t first = SH::lvl_col(P, a, L), nc = SH::lvl_ncol(P, a, L);
    uint32_t c0 = first;
    if (c0 == 0 && s == 0 && (A.hkeys || A.doff)) {  // full segment, first column
        col0_range(A, v, r);
        if (nc == 1 || r.lo >= r.hi) return r.hi - r.lo;
        c0 = 1;
    }
    uint32_t lo = r.lo, hi = r.hi;
    SRDL_LOOP
    for (uint32_t c = c0; c < first + nc && lo < hi; ++c) {
        const uint32_t *col = A.seg[s].cols[c];
        uint32_t x = lbound(col, lo, hi, v);
        hi = ubound(col, x, hi, v);
        lo = x;
    }
    if (lo >= hi) hi = lo;
    r.lo = lo;
    r.hi = hi;
    return hi - lo;
}

template <class SH>
SRDL_SEARCH uint32_t narrow_first(const srdl_plan &P, uint32_t a, int s, int L, uint32_t v, Rng &r) {
    const srdl_atom &A = P.atom[a];
    const uint32_t c = SH::lvl_col(P, a, L);
    if (c == 0 && s == 0 && (A.hkeys || A.doff)) {
        col0_range(A, v, r);
        return r.hi - r.lo;
    }
    const uint32_t *col = A.seg[s].cols[c];
    uint32_t x = lbound(col, r.lo, r.hi, v);
    uint32_t y = ubound(col, x, r.hi, v);
    r.lo = x;
    r.hi = y;
    return y - x;
}

// Leaf-level membership: does segment s of atom a (rows r) hold a row whose
// leaf columns equal v? The leaf's narrowed range is never used again, so a
// single-column leaf needs one lower-bound search and an equality test
// instead of narrow()'s lower- and upper-bound searches.
template <class SH>
SRDL_SEARCH bool leaf_member(const srdl_plan &P, uint32_t a, int s, int L, uint32_t v, Rng r) {
    if (SH::lvl_ncol(P, a, L) != 1) return narrow<SH>(P, a, s, L, v, r) != 0;
    const srdl_atom &A = P.atom[a];
    const uint32_t c = SH::lvl_col(P, a, L);
    if (c == 0 && s == 0 && (A.hkeys || A.doff)) {
        col0_range(A, v, r);
        return r.lo < r.hi;
    }
    const uint32_t *col = A.seg[s].cols[c];
    const uint32_t x = lbound(col, r.lo, r.hi, v);
    return x < r.hi && __ldg(col + x) == v;
}

// Head column h of the tuple whose leaf value is v (parent: its lane in the
// parent batch).
template <class SH>
__device__ __forceinline__ uint32_t head_value(const srdl_plan &P, const View &S, uint32_t h, uint32_t parent,
                                               uint32_t v, int leaf) {
    const int lvl = SH::head_level(P, h);
    if (lvl < 0) return P.head_const[h];
    if (lvl == leaf) return v;
    if (lvl == leaf - 1) return S.V(leaf - 1, parent);
    if (lvl == leaf - 2 && SH::nmid(P) && *S.gp_active) return S.V(leaf - 2, S.gp[parent]);
    return S.bind[lvl];
}

// One head tuple at output row `pos` (materialize). Streaming stores
// (evict-first): the output is written once and must not push the
// L2-resident input indexes out of L2.
template <class SH>
__device__ __forceinline__ void store_tuple(const srdl_plan &P, const srdl_exec &X, const View &S, uint64_t pos,
                                            uint32_t parent, uint32_t v, int leaf) {
    SRDL_SHAPE_LOOP
    for (uint32_t h = 0; h < SH::head_arity(P); ++h) __stcs(X.out[h] + pos, head_value<SH>(P, S, h, parent, v, leaf));
    if (X.bitmap) atomicAdd(X.bitmap + pos, 1u);
}

// One head tuple into the speculative arena at `pos`.
template <class SH>
__device__ __forceinline__ void spec_put(const srdl_plan &P, const View &S, const srdl_spec *Q, uint64_t pos,
                                         uint32_t parent, uint32_t v, int leaf) {
    SRDL_SHAPE_LOOP
    for (uint32_t h = 0; h < SH::head_arity(P); ++h) __stcs(Q->cols[h] + pos, head_value<SH>(P, S, h, parent, v, leaf));
}

// Lane 0 reserves the next arena chunk (one global atomic per chunk) and
// links it after `prev`; the chunk id (>= nchunks: arena full) is broadcast.
// Out of line: once per chunk of tuples, and one copy keeps the emit sites
// small.
static __device__ __noinline__ uint32_t reserve_chunk(const srdl_spec *Q, uint32_t prev) {
    uint32_t c = 0;
    if (lane_id() == 0) {
        c = atomicAdd(Q->cursor, 1u);
        if (c < Q->nchunks && prev != kNoChunk) Q->chunk_next[prev] = c;
    }
    return __shfl_sync(kFull, c, 0);
}

template <int MODE, class SH>
struct Sink {
    uint64_t n;          // tuples emitted so far in this slice (uniform)
    uint64_t base;       // write offset of this slice (materialize)
    const srdl_spec *Q;  // speculative arena (kSpec)
    uint32_t cur;        // current chunk of the slice (kSpec), kNoChunk = none yet
    uint32_t fill;       // tuples in the current chunk
    uint32_t first;      // first chunk of the slice
    bool spill;          // arena exhausted: the slice is re-walked later

    __device__ __forceinline__ bool next_chunk() {
        const uint32_t c = reserve_chunk(Q, cur);
        if (c >= Q->nchunks) {
            spill = true;
            return false;
        }
        if (cur == kNoChunk) first = c;
        cur = c;
        fill = 0;
        return true;
    }

    __device__ __forceinline__ void emit(const srdl_plan &P, const srdl_exec &X, const View &S, bool alive,
                                         uint32_t parent, uint32_t v, int leaf) {
        const uint32_t m = __ballot_sync(kFull, alive);
        if (MODE == kMaterialize && alive)
            store_tuple<SH>(P, X, S, base + n + __popc(m & ((1u << lane_id()) - 1u)), parent, v, leaf);
        if (MODE == kSpec && m && !spill) {
            const uint32_t cnt = __popc(m), rank = __popc(m & ((1u << lane_id()) - 1u));
            const uint32_t B = Q->chunk;
            if (cur == kNoChunk || fill == B) next_chunk();
            // the batch fits the current chunk or spills into the next one:
            // reserve first, then every lane stores once (one store site)
            const uint32_t c1 = cur, f1 = fill, room = B - fill;
            const bool two = cnt > room;
            if (!spill && (!two || next_chunk())) {
                if (alive)
                    spec_put<SH>(P, S, Q,
                                 rank < room ? (uint64_t)c1 * B + f1 + rank : (uint64_t)cur * B + (rank - room),
                                 parent, v, leaf);
                fill = two ? cnt - room : f1 + cnt;
            }
        }
        n += __popc(m);
    }
};

// Atom of source j at level L where j is a small run-time selector: the
// candidates are enumerated so that a constant shape folds each arm.
template <class SH>
__device__ __forceinline__ uint32_t spec_of(const srdl_plan &P, int L, uint32_t j) {
    return SH::spec(P, L, j);
}

__device__ __forceinline__ void prefetch_l1(const uint32_t *p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Warp-cooperative merge-path intersection of two single-segment sorted
// leaf lists (both positive, one column each): tiles of 32 values from both
// lists are loaded coalesced, each lane locates its A value in the B tile
// with a 5-step shuffle search, and the tiles advance past
// min(last A, last B). Used for "heavy" parents whose lists are long and of
// comparable length, where per-element binary search would cost
// min(a,b)*log(max(a,b)) dependent loads against (a+b)/32 coalesced steps.
template <int MODE, class SH>
__device__ void merge_pair(const srdl_plan &P, const srdl_exec &X, const View &S, uint32_t p,
                           Sink<MODE, SH> &sink) {
    const int leaf = (int)SH::depth(P) - 1;
    const uint32_t ja = S.leaf_drv[p], jb = 1u - ja;
    const uint32_t a0 = SH::spec(P, leaf, 0), a1 = SH::spec(P, leaf, 1);
    const uint32_t aa = ja ? a1 : a0, ab = ja ? a0 : a1;
    const uint32_t *ca = P.atom[aa].seg[0].cols[ja ? SH::lvl_col(P, a1, leaf) : SH::lvl_col(P, a0, leaf)];
    const uint32_t *cb = P.atom[ab].seg[0].cols[ja ? SH::lvl_col(P, a0, leaf) : SH::lvl_col(P, a1, leaf)];
    uint32_t ia = S.LF(p, ja, 0).lo, ea = S.LF(p, ja, 0).hi;
    uint32_t ib = S.LF(p, jb, 0).lo, eb = S.LF(p, jb, 0).hi;
    const uint32_t l = lane_id();
    SRDL_LOOP
    while (ia < ea && ib < eb) {
        const bool va = ia + l < ea, vb = ib + l < eb;
        const uint32_t av = va ? __ldg(ca + ia + l) : 0xffffffffu;
        const uint32_t bv = vb ? __ldg(cb + ib + l) : 0xffffffffu;
        // the next tiles of both lists into L1 while this one is matched:
        // every step consumes a full tile of at least one list, so the
        // step after waits on an L1 hit instead of an L2 round trip
        // (a 32-value tile spans at most two 128-byte lines: lanes 0-3 touch
        // the first and last word of both next tiles)
        if (l < 4) {
            const uint32_t *base = (l & 1) ? cb + ib : ca + ia;
            const uint32_t end = (l & 1) ? eb - ib : ea - ia;
            const uint32_t off = 32 + (l >> 1) * 31;
            if (off < end) prefetch_l1(base + off);
        }
        const uint32_t na_tile = min(32u, ea - ia), nb_tile = min(32u, eb - ib);
        const uint32_t alast = __shfl_sync(kFull, av, na_tile - 1);
        const uint32_t blast = __shfl_sync(kFull, bv, nb_tile - 1);
#if SRDL_MERGE_SKIP
        // disjoint tiles (warp-uniform test): the lower one has no match
        if (alast < __shfl_sync(kFull, bv, 0)) {
            ia += na_tile;
            continue;
        }
        if (blast < __shfl_sync(kFull, av, 0)) {
            ib += nb_tile;
            continue;
        }
#endif
        const uint32_t m = min(alast, blast);
        uint32_t cnt = 0;  // B tile values < av
#pragma unroll
        for (uint32_t st = 16; st; st >>= 1) {
            const uint32_t probe = __shfl_sync(kFull, bv, cnt + st - 1);
            if (probe < av) cnt += st;
        }
        const uint32_t hit = __shfl_sync(kFull, bv, cnt);
        const bool take_a = va && av <= m;
        sink.emit(P, X, S, take_a && hit == av, p, av, leaf);
        ia += __popc(__ballot_sync(kFull, take_a));
        ib += __popc(__ballot_sync(kFull, vb && bv <= m));
    }
}

// Owner of flat index f: last lane p with pref[p] <= f (pref nondecreasing).
__device__ __forceinline__ uint32_t owner_of(const uint64_t *pref, uint64_t f) {
    uint32_t lo = 0, hi = 32;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (pref[mid] <= f)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo - 1;
}

// Warp exclusive prefix of per-lane lengths into pref[0..32]; returns total.
__device__ __forceinline__ uint64_t warp_prefix(uint64_t len, uint64_t *pref) {
    const uint32_t l = lane_id();
    uint64_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(kFull, incl, o);
        if (l >= (uint32_t)o) incl += y;
    }
    __syncwarp();
    pref[l] = incl - len;
    const uint64_t total = __shfl_sync(kFull, incl, 31);
    if (l == 31) pref[32] = total;
    __syncwarp();
    return total;
}

// Flattened leaf walk over the parents with len > 0 (per-lane driver range
// lengths): prefix sum across the warp, every lane takes one (parent, row).
template <int MODE, class SH>
__device__ void flat_leaves(const srdl_plan &P, const srdl_exec &X, const View &S, uint64_t len,
                            Sink<MODE, SH> &sink) {
    const int leaf = (int)SH::depth(P) - 1;
    const uint32_t nls = SH::nspec(P, leaf);
    const uint32_t l = lane_id();
    const uint64_t total = warp_prefix(len, S.leaf_pref);
    SRDL_LOOP
    for (uint64_t base = 0; base < total; base += 32) {
        const uint64_t f = base + l;
        bool alive = f < total;
        uint32_t p = 0, v = 0;
        if (alive) {
            p = owner_of(S.leaf_pref, f);
            const uint32_t j = S.leaf_drv[p];
            const uint32_t da = spec_of<SH>(P, leaf, j);
            const uint64_t local = f - S.leaf_pref[p];
            const Rng r0 = S.LF(p, j, 0);
            const uint32_t n0 = r0.hi - r0.lo;
            int s = 0;
            uint32_t row, seg_lo;
            if (local < n0) {
                row = r0.lo + (uint32_t)local;
                seg_lo = r0.lo;
            } else {
                s = 1;
                seg_lo = S.LF(p, j, 1).lo;
                row = seg_lo + (uint32_t)(local - n0);
            }
            const uint32_t *col = P.atom[da].seg[s].cols[SH::lvl_col(P, da, leaf)];
            v = __ldg(col + row);
            alive = row == seg_lo || __ldg(col + row - 1) != v;
            if (alive && s == 1 && n0) {
                Rng t = r0;
                alive = narrow_first<SH>(P, da, 0, leaf, v, t) == 0;  // already produced by segment 0
            }
            SRDL_SHAPE_LOOP
            for (uint32_t jj = 0; jj < nls; ++jj) {
                if (!alive) break;
                const uint32_t a = SH::spec(P, leaf, jj);
                if (jj == j && SH::lvl_ncol(P, a, leaf) == 1) continue;
                bool found = false;
#pragma unroll
                for (uint32_t q = 0; q < kSegs; ++q) {
                    if (found || q >= P.atom[a].nseg) break;
                    const Rng t = S.LF(p, jj, q);
                    if (t.lo < t.hi) found = leaf_member<SH>(P, a, q, leaf, v, t);
                }
                if (SH::negated(P, a) == found) alive = false;
            }
        }
        sink.emit(P, X, S, alive, p, v, leaf);
    }
    __syncwarp();
}

// Leaf level m-1 for a batch of parents (bit p of `parents` = lane p of the
// level m-2 chunk; for m == 2 the single parent is the root rectangle).
template <int MODE, class SH>
__device__ void leaf_batch(const srdl_plan &P, const srdl_exec &X, const View &S, uint32_t parents,
                           Sink<MODE, SH> &sink) {
    const int leaf = (int)SH::depth(P) - 1;
    const uint32_t nls = SH::nspec(P, leaf);
    const uint32_t l = lane_id();
    // two plain positive sources on the leaf variable: merge-path candidates
    bool pairable = nls == 2;
    if (pairable) {
        const uint32_t a0 = SH::spec(P, leaf, 0), a1 = SH::spec(P, leaf, 1);
        pairable = !SH::negated(P, a0) && !SH::negated(P, a1) && SH::lvl_ncol(P, a0, leaf) == 1 &&
                   SH::lvl_ncol(P, a1, leaf) == 1;
    }
    uint64_t len = 0;
    bool heavy = false;
    if ((parents >> l) & 1u) {
        uint32_t best = 0xffffffffu, bj = 0, worst = 0;
        SRDL_SHAPE_LOOP
        for (uint32_t j = 0; j < nls; ++j) {
            const uint32_t a = SH::spec(P, leaf, j);
            if (SH::negated(P, a)) continue;
            uint32_t t = 0;
#pragma unroll
            for (uint32_t s = 0; s < kSegs; ++s)
                if (s < P.atom[a].nseg) t += S.LF(l, j, s).hi - S.LF(l, j, s).lo;
            if (t < best) {
                best = t;
                bj = j;
            }
            worst = t > worst ? t : worst;
        }
        len = best;
        S.leaf_drv[l] = (uint8_t)bj;
        if (pairable && best >= kMergeMin && (uint64_t)worst <= (uint64_t)best * kMergeRatio) {
            const Rng a1 = S.LF(l, 0, 1), b1 = S.LF(l, 1, 1);
            const bool single = (P.atom[SH::spec(P, leaf, 0)].nseg < 2 || a1.lo >= a1.hi) &&
                                (P.atom[SH::spec(P, leaf, 1)].nseg < 2 || b1.lo >= b1.hi);
            if (single) {
                heavy = true;
                len = 0;  // handled by merge_pair below
            }
        }
    }
    const uint32_t heavy_mask = __ballot_sync(kFull, heavy);
    // Parents are emitted in lane order (runs of flattened light parents,
    // then one merge-path heavy parent), so a head that projects the
    // variables in order receives lexicographically sorted tuples.
    uint32_t remaining = parents;
    SRDL_LOOP
    while (remaining) {
        const uint32_t hv = heavy_mask & remaining;
        const uint32_t first_heavy = hv ? (uint32_t)(__ffs(hv) - 1) : 32u;
        const uint32_t run = first_heavy == 32u ? remaining : remaining & ((1u << first_heavy) - 1u);
        if (run) flat_leaves<MODE, SH>(P, X, S, ((run >> l) & 1u) ? len : 0, sink);
        remaining &= ~run;
        if (first_heavy < 32u) {
            merge_pair<MODE, SH>(P, X, S, first_heavy, sink);
            remaining &= ~(1u << first_heavy);
        }
    }
}

// Mid batch (plans of depth >= 4): the survivors of level m-3 (bit g of
// `gps`, their deep-atom ranges in S.mid) are expanded over their level
// m-2 candidates in flattened chunks of 32; each chunk's survivors become a
// parent batch for the leaf. Replaces one serial descent per survivor.
template <int MODE, class SH>
__device__ void mid_batch(const srdl_plan &P, const srdl_exec &X, const View &S, uint32_t gps,
                          Sink<MODE, SH> &sink) {
    const int leaf = (int)SH::depth(P) - 1, Lm = leaf - 1;
    const uint32_t l = lane_id();
    uint64_t len = 0;
    if ((gps >> l) & 1u) {
        uint32_t best = 0xffffffffu, bj = 0;
        SRDL_SHAPE_LOOP
        for (uint32_t j = 0; j < SH::nspec(P, Lm); ++j) {
            const uint32_t a = SH::spec(P, Lm, j);
            if (SH::negated(P, a)) continue;
            const uint32_t slot = SH::mid_slot(P, a);
            uint32_t t = 0;
#pragma unroll
            for (uint32_t s = 0; s < kSegs; ++s)
                if (s < P.atom[a].nseg) t += S.MD(l, slot, s).hi - S.MD(l, slot, s).lo;
            if (t < best) {
                best = t;
                bj = j;
            }
        }
        len = best;
        S.mid_drv[l] = (uint8_t)bj;
    }
    const uint64_t total = warp_prefix(len, S.mid_pref);
    if (l == 0) *S.gp_active = 1u;
    __syncwarp();
    SRDL_LOOP
    for (uint64_t base = 0; base < total; base += 32) {
        const uint64_t f = base + l;
        bool alive = f < total;
        uint32_t v = 0;
        if (alive) {
            const uint32_t g = owner_of(S.mid_pref, f);
            const uint32_t da = spec_of<SH>(P, Lm, S.mid_drv[g]);
            const uint32_t dslot = SH::mid_slot(P, da);
            const uint64_t local = f - S.mid_pref[g];
            const Rng r0 = S.MD(g, dslot, 0);
            const uint32_t n0 = r0.hi - r0.lo;
            int s = 0;
            uint32_t row, seg_lo;
            if (local < n0) {
                row = r0.lo + (uint32_t)local;
                seg_lo = r0.lo;
            } else {
                s = 1;
                seg_lo = S.MD(g, dslot, 1).lo;
                row = seg_lo + (uint32_t)(local - n0);
            }
            const uint32_t *col = P.atom[da].seg[s].cols[SH::lvl_col(P, da, Lm)];
            v = __ldg(col + row);
            alive = row == seg_lo || __ldg(col + row - 1) != v;
            if (alive && s == 1 && n0) {
                Rng t = r0;
                alive = narrow_first<SH>(P, da, 0, Lm, v, t) == 0;
            }
            SRDL_SHAPE_LOOP
            for (uint32_t j = 0; j < SH::nspec(P, Lm); ++j) {
                if (!alive) break;
                const uint32_t b = SH::spec(P, Lm, j);
                const uint32_t slot = SH::mid_slot(P, b), ls = SH::leaf_slot(P, b);
                uint32_t tot = 0;
#pragma unroll
                for (uint32_t q = 0; q < kSegs; ++q) {
                    if (q >= P.atom[b].nseg) break;
                    Rng t = S.MD(g, slot, q);
                    if (t.lo < t.hi)
                        tot += narrow<SH>(P, b, q, Lm, v, t);
                    else
                        t.hi = t.lo;
                    if (ls != SRDL_NO_ATOM) S.LF(l, ls, q) = t;
                }
                if (SH::negated(P, b) ? (SH::check_level(P, b) == Lm && tot != 0) : tot == 0) alive = false;
            }
            if (alive) {
                SRDL_SHAPE_LOOP
                for (uint32_t j = 0; j < SH::nspec(P, leaf); ++j) {
                    const uint32_t b = SH::spec(P, leaf, j);
                    if (SH::lvl_ncol(P, b, Lm)) continue;
#pragma unroll
                    for (uint32_t q = 0; q < kSegs; ++q)
                        if (q < P.atom[b].nseg) S.LF(l, j, q) = S.MD(g, SH::mid_slot(P, b), q);
                }
                S.gp[l] = (uint8_t)g;
            }
            S.V(Lm, l) = v;
        }
        const uint32_t m = __ballot_sync(kFull, alive);
        __syncwarp();
        if (m) leaf_batch<MODE, SH>(P, X, S, m, sink);
    }
    __syncwarp();
    if (l == 0) *S.gp_active = 0u;
    __syncwarp();
}

// Pick the smallest candidate source of level L and reset the chunk cursor.
template <class SH>
__device__ __forceinline__ void open_level(const srdl_plan &P, const View &S, int L) {
    if (lane_id() == 0) {
        uint32_t best = 0xffffffffu, ba = 0;
        SRDL_SHAPE_LOOP
        for (uint32_t j = 0; j < SH::nspec(P, L); ++j) {
            const uint32_t a = SH::spec(P, L, j);
            if (SH::negated(P, a)) continue;
            uint32_t t = 0;
#pragma unroll
            for (uint32_t s = 0; s < kSegs; ++s)
                if (s < P.atom[a].nseg) t += S.R(L, a, s).hi - S.R(L, a, s).lo;
            if (t < best) {
                best = t;
                ba = a;
            }
        }
        S.drv[L] = (uint8_t)ba;
        S.dseg[L] = 0;
        S.cur[L] = S.R(L, ba, 0).lo;
        S.mask[L] = 0;
    }
    __syncwarp();
}

// Next 32 driver rows of level L -> filtered candidates. False when exhausted.
template <int MODE, int KIND, class SH>
__device__ bool load_chunk(const srdl_plan &P, const srdl_exec &X, const View &S, int L, Sink<MODE, SH> &sink) {
    const uint32_t l = lane_id();
    const uint32_t a = S.drv[L];
    const srdl_atom &D = P.atom[a];
    uint32_t s = S.dseg[L];
    uint32_t r = S.cur[L];
    SRDL_LOOP
    while (true) {
        if (s >= D.nseg) return false;
        if (r < S.R(L, a, s).hi) break;
        ++s;
        if (s < D.nseg) r = S.R(L, a, s).lo;
    }
    const Rng seg = S.R(L, a, s);
    const uint32_t row = r + l;
    const uint32_t *col = D.seg[s].cols[SH::lvl_col(P, a, L)];
    bool alive = row < seg.hi;
    uint32_t v = 0;
    if (alive) {
        v = __ldg(col + row);
        alive = row == seg.lo || __ldg(col + row - 1) != v;
    }
    if (alive && s == 1) {
        Rng t = S.R(L, a, 0);
        if (t.lo < t.hi) alive = narrow_first<SH>(P, a, 0, L, v, t) == 0;
    }
    const int leaf = (int)SH::depth(P) - 1;
    const bool parents_level = KIND != kDepth4Mid && L == leaf - 1;
    const bool gp_level = (KIND == kGeneral || KIND == kDepth4Mid) && SH::nmid(P) && L == leaf - 2;
    SRDL_SHAPE_LOOP
    for (uint32_t j = 0; j < SH::nspec(P, L); ++j) {
        if (!alive) break;
        const uint32_t b = SH::spec(P, L, j);
        const uint32_t slot = parents_level ? SH::leaf_slot(P, b) : (gp_level ? SH::mid_slot(P, b) : SRDL_NO_ATOM);
        const bool keep = slot != SRDL_NO_ATOM;
        if (b == a && SH::lvl_ncol(P, b, L) == 1 && !keep) continue;
        uint32_t tot = 0;
#pragma unroll
        for (uint32_t q = 0; q < kSegs; ++q) {
            if (q >= P.atom[b].nseg) break;
            Rng t = S.R(L, b, q);
            if (t.lo < t.hi)
                tot += narrow<SH>(P, b, q, L, v, t);
            else
                t.hi = t.lo;
            if (keep) {
                if (parents_level)
                    S.LF(l, slot, q) = t;
                else
                    S.MD(l, slot, q) = t;
            }
        }
        if (SH::negated(P, b) ? (SH::check_level(P, b) == L && tot != 0) : tot == 0) alive = false;
    }
    if (parents_level && alive) {
        // leaf sources not constrained at this level keep their ranges
        SRDL_SHAPE_LOOP
        for (uint32_t j = 0; j < SH::nspec(P, leaf); ++j) {
            const uint32_t b = SH::spec(P, leaf, j);
            if (SH::lvl_ncol(P, b, L)) continue;
#pragma unroll
            for (uint32_t q = 0; q < kSegs; ++q)
                if (q < P.atom[b].nseg) S.LF(l, j, q) = S.R(L, b, q);
        }
    }
    if (gp_level && alive) {
        // deep sources not constrained at this level keep their ranges
        SRDL_SHAPE_LOOP
        for (uint32_t b = 0; b < SH::natoms(P); ++b) {
            const uint32_t slot = SH::mid_slot(P, b);
            if (slot == SRDL_NO_ATOM || SH::lvl_ncol(P, b, L)) continue;
#pragma unroll
            for (uint32_t q = 0; q < kSegs; ++q)
                if (q < P.atom[b].nseg) S.MD(l, slot, q) = S.R(L, b, q);
        }
    }
    S.V(L, l) = v;
    const uint32_t m = __ballot_sync(kFull, alive);
    if (l == 0) {
        S.cur[L] = seg.hi - r > 32 ? r + 32 : seg.hi;
        S.dseg[L] = (uint8_t)s;
        S.mask[L] = (parents_level || gp_level) ? 0u : m;
    }
    __syncwarp();
    if (parents_level && m) leaf_batch<MODE, SH>(P, X, S, m, sink);
    if constexpr (KIND == kGeneral || KIND == kDepth4Mid) {
        if (gp_level && m) mid_batch<MODE, SH>(P, X, S, m, sink);
    }
    return true;
}

// Bind survivor `ln` of level L and derive the level L+1 ranges.
template <class SH>
__device__ __forceinline__ void descend(const srdl_plan &P, const View &S, int L, uint32_t ln) {
    const uint32_t l = lane_id();
    const uint32_t v = S.V(L, ln);
    if (l == 0) S.bind[L] = v;
    SRDL_LOOP
    for (uint32_t t = l; t < SH::natoms(P) * SRDL_MAX_SEGS; t += 32) {
        const uint32_t a = t / SRDL_MAX_SEGS, s = t % SRDL_MAX_SEGS;
        Rng r = S.R(L, a, s);
        if (SH::lvl_ncol(P, a, L) && s < P.atom[a].nseg && r.lo < r.hi) narrow<SH>(P, a, s, L, v, r);
        S.R(L + 1, a, s) = r;
    }
    __syncwarp();
}

// Staged root-key window fields (S.wroot[field * 32 + j]).
enum : uint32_t { kWD2 = 0, kWKey = 1, kWOlo = 2, kWOdeg = 3, kWIlo = 4 };

// One (key, outer rows [r0,r1), inner rows [c0,c1)) rectangle.
template <int MODE, int KIND, class SH>
__device__ void run_rect(const srdl_plan &P, const srdl_exec &X, const View &S, uint32_t j, uint32_t key,
                         uint64_t r0, uint64_t r1, uint64_t c0, uint64_t c1, Sink<MODE, SH> &sink) {
    const uint32_t l = lane_id();
    const uint32_t a = l / SRDL_MAX_SEGS, s = l % SRDL_MAX_SEGS;
    const bool mine = a < SH::natoms(P);
    const uint32_t am = mine ? a : 0;
    uint32_t lo = 0, hi = 0;
    bool has0 = false;
    const srdl_atom &A = P.atom[am];
    if (mine && s < A.nseg) {
        lo = A.seg[s].lo;
        hi = A.seg[s].hi;
    }
    if (mine) has0 = SH::lvl_ncol(P, am, 0) != 0;
    if (has0 && lo < hi) {
        if (a == SH::outer(P) && X.outer_lo) {  // single segment: rows straight from the histogram
            lo += S.wroot[kWOlo * 32 + j];
            hi = lo + S.wroot[kWOdeg * 32 + j];
        } else if (a == SH::inner(P) && X.inner_lo) {
            lo += S.wroot[kWIlo * 32 + j];
            hi = lo + S.wroot[kWD2 * 32 + j];
        } else {
            Rng t{lo, hi};
            narrow_first<SH>(P, am, s, 0, key, t);
            lo = t.lo;
            hi = t.hi;
        }
    }
    const uint32_t n_here = hi - lo;
    const uint32_t n0 = __shfl_sync(kFull, n_here, l & ~1u);
    if (mine && (a == SH::outer(P) || a == SH::inner(P))) {
        const uint64_t q0 = a == SH::outer(P) ? r0 : c0;
        const uint64_t q1 = a == SH::outer(P) ? r1 : c1;
        uint64_t f, e;
        if (s == 0) {
            f = q0 < n0 ? q0 : n0;
            e = q1 < n0 ? q1 : n0;
        } else {
            f = q0 > n0 ? q0 - n0 : 0;
            e = q1 > n0 ? q1 - n0 : 0;
            if (f > n_here) f = n_here;
            if (e > n_here) e = n_here;
        }
        hi = lo + (uint32_t)e;
        lo = lo + (uint32_t)f;
    }
    const uint32_t nc0 = mine ? SH::lvl_ncol(P, am, 0) : 0;
    if (has0 && nc0 > 1 && lo < hi) {
        const uint32_t first = SH::lvl_col(P, am, 0);
        SRDL_LOOP
        for (uint32_t c = first + 1; c < first + nc0 && lo < hi; ++c) {
            const uint32_t *col = A.seg[s].cols[c];
            uint32_t x = lbound(col, lo, hi, key);
            hi = ubound(col, x, hi, key);
            lo = x;
        }
        if (lo > hi) hi = lo;
    }
    const uint32_t len = hi - lo;
    const uint32_t tot = len + __shfl_xor_sync(kFull, len, 1);
    bool dead = false;
    if (mine && s == 0 && has0)
        dead = SH::negated(P, am) ? (SH::check_level(P, am) == 0 && tot != 0) : tot == 0;
    if (mine) S.R(1, a, s) = Rng{lo, hi};
    if (__any_sync(kFull, dead)) return;
    __syncwarp();
    if (l == 0) {
        S.bind[0] = key;
        S.V(0, 0) = key;
    }
    if (KIND == kShallow || (KIND == kGeneral && SH::depth(P) <= 2)) {
        if (SH::depth(P) == 1) {
            sink.emit(P, X, S, l == 0, 0, key, 0);
            return;
        }
        SRDL_LOOP
        for (uint32_t t = l; t < SH::nspec(P, 1) * SRDL_MAX_SEGS; t += 32) {
            const uint32_t jj = t / SRDL_MAX_SEGS, q = t % SRDL_MAX_SEGS;
            S.LF(0, jj, q) = S.R(1, SH::spec(P, 1, jj), q);
        }
        __syncwarp();
        leaf_batch<MODE, SH>(P, X, S, 1u, sink);
        return;
    }
    if constexpr (KIND == kDepth3 || KIND == kDepth4Mid) {
        // level 1 is the parents level (depth 3) or the grandparents level
        // of a mid batch (depth 4): its chunks feed the flattened levels
        __syncwarp();
        open_level<SH>(P, S, 1);
        SRDL_LOOP
        while (load_chunk<MODE, KIND, SH>(P, X, S, 1, sink)) {
        }
    } else if constexpr (KIND == kGeneral) {
        __syncwarp();
        // DFS over levels 1..m-2; level m-2 hands its survivors to leaf_batch
        // (and, with a mid batch, level m-3 hands its survivors to mid_batch)
        int L = 1;
        open_level<SH>(P, S, L);
        SRDL_LOOP
        while (true) {
            const uint32_t m = S.mask[L];
            if (m == 0) {
                if (load_chunk<MODE, KIND, SH>(P, X, S, L, sink)) continue;
                if (L == 1) break;
                --L;
                continue;
            }
            const uint32_t ln = __ffs(m) - 1;
            __syncwarp();
            if (l == 0) S.mask[L] = m & (m - 1);
            descend<SH>(P, S, L, ln);
            ++L;
            open_level<SH>(P, S, L);
        }
    }
}

// Slices the root work [0, T) is cut into: enough to occupy every launched
// warp several times, coarser ones (>= min_units units) only when T is large.
// The gather kernel uses the same count (slices beyond it are empty).
__device__ __forceinline__ uint64_t slices_used(const srdl_exec &X, uint64_t T) {
    uint64_t used = (T + X.min_units - 1) / X.min_units;
    const uint64_t floor_slices = (uint64_t)X.nwarps * 4 < T ? (uint64_t)X.nwarps * 4 : T;
    if (used < floor_slices) used = floor_slices;
    return used < 1 ? 1 : (used > X.nslices ? X.nslices : used);
}

// The kernel body: slice loop of one warp (every warp of the grid runs it).
template <int MODE, int KIND, class SH>
__device__ __forceinline__ void wcoj_body(const srdl_plan &P, const srdl_exec &X, const srdl_spec &Q) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t NL = SH::nspec(P, SH::depth(P) - 1) ? SH::nspec(P, SH::depth(P) - 1) : 1;
    const size_t wb = warp_bytes(SH::depth(P), SH::natoms(P), NL, SH::nmid(P));
    const View S = make_view(smem + wib * wb, SH::depth(P), SH::natoms(P), NL, SH::nmid(P));
    if (lane_id() == 0) *S.gp_active = 0u;
    __syncwarp();
    const uint64_t K = X.nkeys;
    const uint64_t T = K ? X.prefix[K - 1] : 0;
    const uint64_t used = slices_used(X, T);
    const uint64_t step = (T + used - 1) / used;
    SRDL_LOOP
    while (true) {
        // dynamic slice fetch: any warp may run any slice, offsets are per slice
        uint32_t sl = 0;
        if (lane_id() == 0) sl = atomicAdd(X.ticket, 1u);
        sl = __shfl_sync(kFull, sl, 0);
        if (sl >= used) break;
        uint64_t bs = (uint64_t)sl * step, be = bs + step;
        if (bs > T) bs = T;
        if (be > T) be = T;
        // materialize after a speculative count: only the spilled slices
        if (MODE == kMaterialize && Q.slice_spill && !Q.slice_spill[sl]) continue;
        Sink<MODE, SH> sink{0, MODE == kMaterialize ? X.slice_offsets[sl] : 0, &Q, kNoChunk, 0, kNoChunk, false};
        if (bs < be) {
            // kappa: first key whose inclusive prefix exceeds bs
            uint64_t lo = 0, hi = K;
            while (lo < hi) {
                uint64_t mid = (lo + hi) >> 1;
                if (X.prefix[mid] <= bs)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            // root keys are staged 32 at a time in shared memory (lane i
            // loads entry kb + i of every work array: one coalesced load per
            // array per window) instead of a chain of uniform global loads
            // per key
            const uint32_t l = lane_id();
            uint64_t kb = lo;
            uint32_t j = 32;  // forces the first window load
            SRDL_LOOP
            for (uint64_t k = lo; k < K; ++k, ++j) {
                if (j == 32) {
                    const uint64_t before = k == lo ? (lo ? X.prefix[lo - 1] : 0) : S.wpre[32];
                    __syncwarp();
                    kb = k;
                    j = 0;
                    const uint64_t e = kb + l;
                    if (l == 0) S.wpre[0] = before;
                    if (e < K) {
                        S.wpre[1 + l] = X.prefix[e];
                        S.wroot[kWD2 * 32 + l] = X.d2[e];
                        S.wroot[kWKey * 32 + l] = X.keys[e];
                        if (X.outer_lo) {
                            S.wroot[kWOlo * 32 + l] = X.outer_lo[e];
                            S.wroot[kWOdeg * 32 + l] = X.outer_deg[e];
                        }
                        if (X.inner_lo) S.wroot[kWIlo * 32 + l] = X.inner_lo[e];
                    }
                    __syncwarp();
                }
                const uint64_t start = S.wpre[j];
                if (start >= be) break;
                const uint64_t end = S.wpre[j + 1];
                const uint64_t u0 = (bs > start ? bs : start) - start;
                const uint64_t u1 = (be < end ? be : end) - start;
                if (u0 >= u1) continue;
                const uint32_t d2 = S.wroot[kWD2 * 32 + j];
                const uint32_t key = S.wroot[kWKey * 32 + j];
                uint64_t ra, ca, rb, cb;
                if (u1 < (1ull << 32)) {  // 32-bit division (the common case)
                    const uint32_t x0 = (uint32_t)u0, x1 = (uint32_t)u1;
                    ra = x0 / d2;
                    ca = x0 - (uint32_t)ra * d2;
                    rb = x1 / d2;
                    cb = x1 - (uint32_t)rb * d2;
                } else {
                    ra = u0 / d2, ca = u0 % d2, rb = u1 / d2, cb = u1 % d2;
                }
                if (ra == rb) {
                    run_rect<MODE, KIND, SH>(P, X, S, j, key, ra, ra + 1, ca, cb, sink);
                    continue;
                }
                if (ca) {
                    run_rect<MODE, KIND, SH>(P, X, S, j, key, ra, ra + 1, ca, d2, sink);
                    ++ra;
                }
                if (ra < rb) run_rect<MODE, KIND, SH>(P, X, S, j, key, ra, rb, 0, d2, sink);
                if (cb) run_rect<MODE, KIND, SH>(P, X, S, j, key, rb, rb + 1, 0, cb, sink);
            }
        }
        if (lane_id() == 0) {
            if (MODE == kMaterialize) {
                if (sink.n != X.slice_counts[sl]) atomicExch(X.error, 1u);
            } else {
                X.slice_counts[sl] = sink.n;
            }
            if (MODE == kSpec) {
                Q.slice_first[sl] = sink.first;
                Q.slice_spill[sl] = sink.spill ? 1u : 0u;
                if (sink.spill) atomicAdd((unsigned long long *)Q.spills, 1ull);
            }
        }
        __syncwarp();
    }
}

}  // namespace srdl
