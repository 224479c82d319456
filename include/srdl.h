/*
 * srdl.h — C ABI of the sm_100a semi-naive fixpoint library (libsrdl.so).
 *
 * This is the drop-in boundary under the reference's Python API: every
 * numeric operation the reference evaluates with numpy on the host
 * (pkg/src/flatlog/rowops.py, storage.py, executor.py) has exactly one entry
 * point here, taking plain device pointers, row counts and a CUDA stream.
 * No torch types cross this boundary; a ctypes (or cgo/JNI) binding can call
 * it directly. See INTEGRATION.md for the reference-side binding.
 *
 * Conventions
 *   - Relations are Structure-of-Arrays: `arity` device arrays of uint32 ids,
 *     rows sorted lexicographically over the columns in index order.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Every function returns 0 on success and a negative code on error;
 *     srdl_last_error() gives the message (thread-local).
 *   - Host-side counts written through `uint64_t *n_out` require a stream
 *     synchronisation, which the function performs (two-phase allocation:
 *     the caller sizes the next buffer from that count).
 *   - Scratch memory comes from a stack arena per (device, stream, host
 *     thread) inside libsrdl; every scratch buffer lives within one call.
 */
#ifndef SRDL_H
#define SRDL_H

#ifdef __CUDACC_RTC__
/* NVRTC (the per-plan kernel JIT, csrc/wcoj_jit.cu) has no C library
 * headers; the fixed-width types come from here. */
typedef unsigned char uint8_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned long size_t;
#else
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SRDL_VERSION 1
#define SRDL_MAX_ATOMS 12   /* body atoms per rule instance        */
#define SRDL_MAX_LEVELS 12  /* variables per rule instance         */
#define SRDL_MAX_COLS 8     /* columns per atom                    */
#define SRDL_MAX_HEAD 12    /* head arity                          */
#define SRDL_MAX_SEGS 2     /* body + head buffer of one index     */
#define SRDL_NO_ATOM 255u
#define SRDL_NO_SYMBOL 0xFFFFFFFFu

#define SRDL_OK 0
#define SRDL_ERR_CUDA -1
#define SRDL_ERR_ARG -2
#define SRDL_ERR_INTERNAL -3

/* ------------------------------------------------------------------ misc */

int srdl_version(void);
const char *srdl_last_error(void);
/* Number of SMs of the current device (grid sizing), or a negative code. */
int srdl_sm_count(void);
/* Kernels launched by this library since load (process-wide counter). */
uint64_t srdl_launch_count(void);
/* Work launched on `waiter` after this call starts after all work launched on
 * `signaler` before it (event record + stream wait; the engine's fork/join of
 * side streams — reference runtime.py:225-257 runs phases of independent
 * plans concurrently; this is the device-side ordering that replaces its
 * thread-pool join). */
int srdl_stream_wait(void *waiter, void *signaler);
/* Device-wide prefix sums (exclusive or inclusive; total = sum, exclusive
 * only, device pointer or NULL). in and out may alias. */
int srdl_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, int exclusive, uint32_t *total, void *stream);
int srdl_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, int exclusive, uint64_t *total, void *stream);

/* --------------------------------------------------------------- storage
 * reference: rowops.sort_dedup (rowops.py:60) / storage.sort_dedup
 * (storage.py:304). Sorts n rows of `arity` columns lexicographically and
 * removes duplicates. `bits` = significant bits per id (ceil(log2(#symbols)),
 * at most 32): columns are radix-sorted on packed keys of bits*arity bits.
 * out: `arity` arrays with capacity n. *n_out = distinct rows (host).
 * n_out == NULL: the caller guarantees the rows are distinct (a re-sort of a
 * delta under another column order); no host round trip, n rows written. */
int srdl_sort_dedup(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                    uint32_t *const *out, uint64_t *n_out, void *stream);

/* reference: RelationState.take_delta (storage.py:373-380), the delta of
 * one iteration re-sorted under another index order. The rows are distinct
 * and sorted by an order whose restriction to columns nkey.. of the target
 * order (cols[] is given in TARGET order) is already their relative order,
 * so one STABLE sort on the first nkey target columns finishes the job:
 * nkey * bits key bits instead of arity * bits (e.g. (h, v) -> (v, h) sorts
 * on v alone). out: `arity` arrays of n rows, target order. */
int srdl_sort_reorder(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits, uint32_t nkey,
                      uint32_t *const *out, void *stream);

/* Compute Delta through a device hash set of the full relation (csrc/
 * hashset.cu; reference storage.compute_delta, storage.py:311-324). `slots`
 * is an open-addressing set of 2^log2cap packed row keys (UINT64_MAX =
 * empty; keys are rows packed column 0 first with `bits` bits per column,
 * arity * bits <= 63).
 * srdl_hset_insert: add n rows.
 * srdl_hset_filter: the packed keys of the staged rows NOT in the set,
 *   compacted into keys_out (capacity n, any order), their count into
 *   *count_dev (device) — only they need sorting.
 * srdl_sort_unique_keys: sort m packed keys in place, drop duplicates and
 *   unpack the distinct rows into out (capacity m); count into *count_dev. */
int srdl_hset_insert(uint64_t *slots, uint32_t log2cap, const uint32_t *const *cols, uint32_t arity, uint64_t n,
                     uint32_t bits, void *stream);
int srdl_hset_filter(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits, const uint64_t *slots,
                     uint32_t log2cap, uint64_t *keys_out, uint32_t *count_dev, void *stream);
int srdl_sort_unique_keys(uint64_t *keys, uint64_t m, uint32_t arity, uint32_t bits, uint32_t *const *out,
                          uint32_t *count_dev, void *stream);

/* reference: storage.compute_delta (storage.py:311): distinct staged rows
 * minus the rows of up to eight sorted, duplicate-free segments (the full
 * relation's head and body, plus deltas of earlier chunks when a staging
 * buffer exceeds 2^31 rows). Fuses sort, unique and the anti-join.
 * seg_cols[s] points to `arity` column pointers of segment s. */
int srdl_compute_delta(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                       const uint32_t *const *const *seg_cols, const uint64_t *seg_rows,
                       uint32_t nseg, uint32_t *const *out, uint64_t *n_out, void *stream);

/* reference: rowops.merge_sorted (rowops.py:77) and the single-pass
 * head->body flush of ColumnarRelation.merge_delta (storage.py:272).
 * Merges two sorted, mutually disjoint row sets into out (na+nb rows). */
int srdl_merge(const uint32_t *const *a, uint64_t na, const uint32_t *const *b, uint64_t nb,
               uint32_t arity, uint32_t *const *out, void *stream);

/* reference: rowops.is_sorted_strict (rowops.py:64). *ok = 1 iff rows are
 * strictly increasing (sorted, no duplicates). */
/* srdl_compute_delta without the host round trip: the number of rows
 * written to `out` (capacity n) lands in *count_dev (device memory), so the
 * engine can launch the delta of every head relation of a stratum and read
 * all sizes back at once (reference: storage.compute_delta, storage.py:311). */
int srdl_compute_delta_async(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t bits,
                             const uint32_t *const *const *seg_cols, const uint64_t *seg_rows,
                             uint32_t nseg, uint32_t *const *out, uint32_t *count_dev, void *stream);

int srdl_is_sorted_strict(const uint32_t *const *cols, uint32_t arity, uint64_t n, int *ok,
                          void *stream);

/* Gather rows: out[c][i] = cols[c][idx[i]] (index builds, column permutes). */
int srdl_gather(const uint32_t *const *cols, uint32_t arity, const uint32_t *idx, uint64_t n,
                uint32_t *const *out, void *stream);

/* ------------------------------------------------------------ histograms
 * reference: storage.Histogram.over_column (storage.py:48). Run-length of a
 * sorted column: keys[K], degrees[K], inclusive prefix[K] (uint64).
 * keys/degrees/prefix have capacity n; *k_out = K (host). */
int srdl_histogram(const uint32_t *col, uint64_t n, uint32_t *keys, uint32_t *degrees,
                   uint64_t *prefix, uint64_t *k_out, void *stream);

/* reference: storage.Histogram.updated (storage.py:63): union of two
 * histograms, degrees of equal keys added. Outputs have capacity na+nb. */
int srdl_histogram_merge(const uint32_t *ka, const uint32_t *da, uint64_t na, const uint32_t *kb,
                         const uint32_t *db, uint64_t nb, uint32_t *keys, uint32_t *degrees,
                         uint64_t *prefix, uint64_t *k_out, void *stream);

/* Histogram of a sorted delta column AND its union with an existing
 * histogram (fkeys/fdeg, nf keys; nf may be 0), with one host readback
 * (reference: Histogram.over_column + Histogram.updated, storage.py:48-76;
 * replaces srdl_histogram + srdl_histogram_merge on the per-iteration
 * delta path). Delta outputs hold n entries, union outputs nf + n; the
 * first *kd_out / *ku_out are the histograms (prefix entries past them
 * repeat the total). */
int srdl_histogram_union(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                         uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix, uint64_t *kd_out,
                         uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint64_t *ku_out, void *stream);

/* srdl_histogram_union without the host round trip: (K_delta, K_union) land
 * in k_dev[0..1] (device memory); outputs as srdl_histogram_union. */
int srdl_histogram_union_async(const uint32_t *col, uint64_t n, const uint32_t *fkeys, const uint32_t *fdeg,
                               uint64_t nf, uint32_t *dkeys, uint32_t *ddeg, uint64_t *dprefix,
                               uint32_t *ukeys, uint32_t *udeg, uint64_t *uprefix, uint32_t *k_dev,
                               void *stream);

/* Dense column-0 offsets from a histogram (keys[K], inclusive prefix[K]):
 * off[v] = number of rows whose column 0 is < v, for v in [0, n_ids];
 * off has n_ids + 1 entries. The CSR row index of a sorted relation. */
int srdl_dense_offsets(const uint32_t *keys, const uint64_t *prefix, uint64_t nkeys,
                       uint32_t n_ids, uint32_t *off, void *stream);

/* Largest id over `arity` columns of n rows into *max_dev (device memory;
 * 0 for n == 0): the id space an engine reserves for integer EDB columns
 * (reference: interning of integer constants, interning.py). */
int srdl_max_id(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t *max_dev, void *stream);

/* Fence keys of a sorted key array: fence[i] = keys[i * SRDL_FENCE] for
 * i < ceil(n / SRDL_FENCE) (the first level of the two-level column-0 search
 * in the WCOJ kernels; reference: the bisect in storage.narrow_segments,
 * storage.py:122, over Histogram.keys). */
int srdl_key_fence(const uint32_t *keys, uint64_t n, uint32_t *fence, void *stream);

/* Narrow one sorted segment on its leading columns to constant values
 * (reference: executor.prepare constant narrowing, executor.py:188-206,
 * storage.narrow_segments, storage.py:122). Returns [*lo, *hi) on the host. */
int srdl_narrow_prefix(const uint32_t *const *cols, uint64_t n, const uint32_t *values,
                       uint32_t nvalues, uint64_t *lo, uint64_t *hi, void *stream);

/* ------------------------------------------------------------------ WCOJ */

typedef struct {
    const uint32_t *cols[SRDL_MAX_COLS]; /* index-order columns        */
    uint32_t lo, hi;                     /* rows left after constants  */
} srdl_segment;

typedef struct {
    srdl_segment seg[SRDL_MAX_SEGS];
    uint32_t nseg;
    uint32_t negated;
    uint32_t arity;
    uint32_t nconst;
    int32_t check_level;                 /* negated: level of the probe, else -1 */
    uint8_t lvl_col[SRDL_MAX_LEVELS];    /* first index column bound at level L */
    uint8_t lvl_ncol[SRDL_MAX_LEVELS];   /* columns bound at level L (0 = none) */
    /* optional histogram of index column 0 over the single segment
     * (keys[hk], inclusive row prefix[hk]): column-0 narrowing becomes a
     * binary search over the distinct keys (L2-resident) instead of the rows */
    const uint32_t *hkeys;
    const uint64_t *hprefix;
    uint32_t hk;
    /* optional dense column-0 offsets over the single segment: rows with
     * column 0 == v are [doff[v], doff[v+1]) for v < dn (two loads) */
    uint32_t dn;
    const uint32_t *doff;
    /* optional fence keys of the histogram: hfence[i] = hkeys[i * SRDL_FENCE]
     * for i < hfn. The column-0 search first bisects this short array (it
     * stays in L1), then one SRDL_FENCE-key block of hkeys, instead of
     * log2(hk) dependent L2 round trips. */
    const uint32_t *hfence;
    uint32_t hfn;
    uint32_t reserved;
} srdl_atom;

/* One compiled rule instance (reference: planner.JoinPlan, planner.py:53-73). */
typedef struct {
    uint32_t depth;  /* number of variables m >= 1 */
    uint32_t natoms;
    uint32_t outer;  /* root source whose rows are flattened (Alg. 1)   */
    uint32_t inner;  /* second root source or SRDL_NO_ATOM               */
    uint32_t head_arity;
    int32_t head_level[SRDL_MAX_HEAD];  /* >= 0: variable level; -1: constant */
    uint32_t head_const[SRDL_MAX_HEAD];
    uint32_t nspec[SRDL_MAX_LEVELS];    /* atoms with columns at level L       */
    uint8_t spec[SRDL_MAX_LEVELS][SRDL_MAX_ATOMS];
    uint8_t leaf_slot[SRDL_MAX_ATOMS];  /* position in spec[depth-1] or NO_ATOM */
    /* atoms with columns at the last two levels (depth >= 4): slot in the
     * per-lane "mid batch" range table, or NO_ATOM; nmid = 0 disables the
     * flattening of level depth-2 over the survivors of level depth-3 */
    uint8_t mid_slot[SRDL_MAX_ATOMS];
    uint32_t nmid;
    srdl_atom atom[SRDL_MAX_ATOMS];
} srdl_plan;

/* histogram keys per fence block (srdl_atom.hfence, srdl_key_fence) */
#define SRDL_FENCE 64

/* at most this many atoms may constrain the last variable of a plan */
#define SRDL_MAX_LEAF_SPECS 6
/* mid batching is used when at most this many atoms touch the last two levels */
#define SRDL_MAX_MID_SPECS 8

/* Root work space of one plan execution (Alg. 1 phase 1, Fig. 2).
 * The flattened units [0, T) are cut into `nslices` equal slices; launched
 * warps fetch slice indexes from `ticket` (one atomic per slice), so the
 * output offsets depend only on the slice, never on which warp ran it. */
typedef struct {
    const uint32_t *keys;    /* K root keys (outer histogram keys)            */
    const uint32_t *d2;      /* K inner degrees (1 without inner source)      */
    const uint64_t *prefix;  /* K inclusive prefix of outer_degree * d2       */
    const uint32_t *outer_deg; /* K outer degrees                             */
    const uint32_t *outer_lo;  /* K first outer row of each key, or NULL       */
    const uint32_t *inner_lo;  /* K first inner row of each key, or NULL       */
    uint64_t nkeys;
    uint32_t nwarps;         /* slicing width (>= 4 x nwarps slices); same for count and materialize */
    uint32_t nslices;        /* capacity of the slice arrays                  */
    uint64_t min_units;      /* slices used = clamp(ceil(T / min_units), 1, nslices) */
    uint32_t *ticket;        /* device counter, zero before each launch       */
    uint64_t *slice_counts;  /* nslices: tuples counted per slice             */
    uint64_t *slice_offsets; /* nslices: exclusive prefix of slice_counts     */
    uint64_t *total;         /* device scalar: sum of slice_counts            */
    uint32_t *out[SRDL_MAX_HEAD];
    uint32_t *error;         /* device flag, non-zero on count/write mismatch */
    uint32_t *bitmap;        /* optional (audit): per-output-slot write counter */
} srdl_exec;

/* Speculative output of the count pass (srdl_wcoj_count_spec). The count
 * walk also writes every tuple into chunks of `chunk` tuples reserved from a
 * bounded arena with one atomic per chunk; a slice's chunks are linked
 * (slice_first, chunk_next). srdl_wcoj_gather then copies each slice's
 * tuples to its exact offset — the same bytes, in the same order, as a
 * second walk (srdl_wcoj_materialize) would write, without repeating the
 * join. A slice that finds the arena full is flagged in slice_spill and
 * re-walked by srdl_wcoj_materialize_spilled; the arena bound keeps the
 * two-phase guarantee that allocation never exceeds a known size. */
typedef struct {
    uint32_t *cols[SRDL_MAX_HEAD]; /* head_arity arrays of nchunks * chunk  */
    uint32_t nchunks;              /* arena capacity in chunks              */
    uint32_t chunk;                /* tuples per chunk (power of two >= 32) */
    uint32_t *cursor;              /* device: next free chunk (zeroed by count_spec) */
    uint64_t *spills;              /* device: number of spilled slices (zeroed by count_spec) */
    uint32_t *chunk_next;          /* device [nchunks]: next chunk of the same slice */
    uint32_t *slice_first;         /* device [nslices]: first chunk of the slice */
    uint32_t *slice_spill;         /* device [nslices]: 1 = re-walk the slice */
} srdl_spec;

/* reference: executor.build_partition (executor.py:246). From the outer
 * histogram (keys, degrees, inclusive prefix) and the inner histogram (may be
 * empty), write d2[K], the inclusive work prefix[K] (uint64) and, when the
 * row-start arrays are given, the first outer / inner row of every key
 * (outer_lo = oprefix - odeg; inner_lo = iprefix - ideg of the same key). */
int srdl_root_work(const uint32_t *okeys, const uint32_t *odeg, const uint64_t *oprefix,
                   uint64_t nk, const uint32_t *ikeys, const uint32_t *ideg,
                   const uint64_t *iprefix, uint64_t nik, int has_inner, uint32_t *d2,
                   uint64_t *prefix, uint32_t *outer_lo, uint32_t *inner_lo, void *stream);

/* reference: executor.count_pass (executor.py:439). Count kernel over the
 * flattened slices + exclusive scan into slice_offsets/total. No host sync. */
int srdl_wcoj_count(const srdl_plan *plan, const srdl_exec *ex, void *stream);

/* reference: executor.materialize_pass (executor.py:458). Re-walks the
 * slices writing head tuples at slice_offsets; sets *error on divergence. */
int srdl_wcoj_materialize(const srdl_plan *plan, const srdl_exec *ex, void *stream);

/* Count pass that also writes the tuples speculatively (see srdl_spec);
 * the counts, offsets and total are exactly those of srdl_wcoj_count. */
int srdl_wcoj_count_spec(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec, void *stream);

/* Copy every non-spilled slice's tuples from the arena to ex->out at its
 * offset (after srdl_wcoj_count_spec; reference: executor.materialize_pass
 * output layout, executor.py:458). */
int srdl_wcoj_gather(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec, void *stream);

/* srdl_wcoj_materialize restricted to the slices flagged in spec->slice_spill. */
int srdl_wcoj_materialize_spilled(const srdl_plan *plan, const srdl_exec *ex, const srdl_spec *spec,
                                  void *stream);

/* ---------------------------------------------------- per-rule kernels
 * The compiler half of the paper (rules become CUDA kernels, PAPER.md:231;
 * no reference counterpart: the reference interprets plans in numpy,
 * executor.py:342-431). For the static shape of a plan (the srdl_plan
 * fields other than pointers, row ranges and segment counts) the library
 * generates and NVRTC-compiles a kernel with that shape as compile-time
 * constants (csrc/wcoj_jit.cu), cached per shape in process and on disk
 * ($SRDL_JIT_CACHE, default ~/.cache/srdl-jit). srdl_wcoj_count /
 * _count_spec / _materialize* use it when it is built and fall back to the
 * generic kernel of the plan's class otherwise; both give identical
 * results. Mode: SRDL_JIT=0 (off) | async (default) | sync. */

/* Schedule the kernels of n plans (array of descriptors; only the shape
 * fields are read) in `mode` (0 count, 1 materialize, 2 speculative count)
 * on the background compiler; wait != 0 blocks until they are built.
 * Returns how many of them have a kernel ready. */
int srdl_wcoj_jit_prepare(const srdl_plan *plans, uint32_t n, int mode, int wait);
/* Block until the background compiler is idle. */
void srdl_wcoj_jit_wait(void);
/* Drop queued compilations and wait for running ones (process exit). */
void srdl_wcoj_jit_shutdown(void);
/* 0 off, 1 async, 2 sync; returns the previous mode. */
int srdl_wcoj_jit_set_mode(int mode);
/* Generated source of a plan's kernel (truncated to cap bytes); returns its length. */
uint64_t srdl_wcoj_jit_source(const srdl_plan *plan, int mode, char *buf, uint64_t cap);
/* NVRTC-compile without loading (no GPU needed): 0 ok (*cubin_bytes set),
 * 1 compile error (log in srdl_last_error), 2 NVRTC unavailable. */
int srdl_wcoj_jit_compile_check(const srdl_plan *plan, int mode, uint64_t *cubin_bytes);
/* out[4] = kernels compiled, disk-cache hits, failures, mode in effect. */
void srdl_wcoj_jit_stats(uint64_t *out);

/* ------------------------------------------------------------ multi-GPU
 * Owner of a value among `world` ranks (hash partitioning of root keys):
 * owner(v) = ((v * 2654435761) >> 8) % world, identical on host and device. */

/* Stable partition of rows by the owner of column `key_col`: out holds the
 * rows of rank 0, then rank 1, ...; counts[world] (host) the rows per rank. */
int srdl_route_rows(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                    uint32_t world, uint32_t *const *out, uint64_t *counts, void *stream);

/* The send buffer of one all-to-all exchange, without a host round trip:
 * rows grouped by the owner of column `key_col` (stable within a rank),
 * written row-major (send[i * arity + c], n * arity words), and the rows per
 * rank into counts_dev[world] (device memory). Replaces srdl_route_rows
 * (one pass and one host read per rank) on the exchange path. */
int srdl_route_pack(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                    uint32_t world, uint32_t *send, uint64_t *counts_dev, void *stream);

/* Received row-major rows (recv[i * arity + c]) back to `arity` columns. */
int srdl_unpack_rows(const uint32_t *recv, uint32_t arity, uint64_t n, uint32_t *const *out, void *stream);

/* Keep the rows whose column `key_col` is owned by `rank` (stable);
 * *n_out (host) = rows kept. out has capacity n. */
int srdl_filter_owned(const uint32_t *const *cols, uint32_t arity, uint64_t n, uint32_t key_col,
                      uint32_t world, uint32_t rank, uint32_t *const *out, uint64_t *n_out,
                      void *stream);

/* Zero the work of root keys not owned by `rank` (inclusive prefix is
 * recomputed): every rank then enumerates only its own root keys. */
int srdl_root_own(const uint32_t *keys, uint64_t nk, const uint32_t *odeg, const uint32_t *d2,
                  uint32_t world, uint32_t rank, uint64_t *prefix, void *stream);

/* ------------------------------------------------------------- generators
 * Synthetic inputs for the benchmarks (not on the evaluation path).
 * R-MAT edge list (Chakrabarti et al.): n = 2^scale vertices, probabilities
 * a, b, c (d = 1-a-b-c), counter-based RNG keyed by seed. */
int srdl_gen_rmat(uint32_t scale, uint64_t nedges, float a, float b, float c, uint64_t seed,
                  uint32_t *src, uint32_t *dst, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SRDL_H */
