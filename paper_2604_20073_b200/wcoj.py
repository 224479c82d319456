"""Plan execution on the device: histogram -> count -> allocate -> materialize.

Mirrors the reference executor API (reference: pkg/src/flatlog/executor.py:
45-549: WorkPartition, decode_workunit, build_partition, count_pass,
materialize_pass, PlanExecution, execute_plan) with every data-touching
step running in libsrdl:

* prepare    resolve each plan atom to an index version (full / delta, per
             column order) and narrow it on its constant columns;
* histogram  root work space: outer histogram (maintained incrementally by
             the storage layer, or rebuilt over a constant-narrowed range),
             inner degrees d2 and the inclusive prefix of outer * d2;
* count      the per-rule (csrc/wcoj_jit.cu) or generic (csrc/wcoj_kernel.cuh)
             count kernel over the root slices + exclusive scan;
* allocate   one exactly-sized output buffer (the only host sync);
* materialize the same walk writing at the per-warp offsets.

`p` is the reference's worker count. On the device the slices are warps:
the kernel uses max(p, DEVICE_WARPS) slices; results do not depend on it.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import audit
from . import device as dev
from .compiler import DELTA, FULL, JoinPlan
from .faults import InternalError
from .partition import WorkPartition, decode_workunit, encode_workunit, rectangles  # noqa: F401
from .syntax import VAR

WARPS_PER_SM = 32  # slice-array sizing; the launcher picks the resident wave itself
SLICES_PER_WARP = 256  # slice-array capacity per launched warp (fetched dynamically)
MIN_SLICE_UNITS = int(os.environ.get("SRDL_MIN_SLICE_UNITS", 65536))  # root work units per slice, at least (profiles/r02/knobs: triangle 78.4 ms at 4096 and 16384, 67.2 ms at 65536)

def _timed(name, fn, algo_bytes=0):
    """One WCOJ library call under the bench's event hook (dev.PROFILE)."""
    rc, rec = dev.timed(name, algo_bytes, fn)
    return rc, rec


def input_bytes(prep) -> int:
    """Algorithmic input bytes of one WCOJ launch: every column of every
    index segment the plan reads, once (4 B per id)."""
    return sum(4 * pa.arity * (hi - lo) for pa, src in zip(prep.plan.atoms, prep.segs) for _, lo, hi in src)


def device_warps(p: int = 1) -> int:
    return max(int(p), dev.sm_count() * WARPS_PER_SM)


def _resolve(store, pa):
    state = store[pa.relation]
    return state.full(pa.column_order) if pa.version == FULL else state.delta(pa.column_order)


class Prepared:
    """Read-only device view of one plan execution's sources."""

    __slots__ = ("plan", "rels", "segs", "ok", "head_resolved", "n_ids", "_desc", "derived")

    def __init__(self, plan, rels, segs, ok, head_resolved, n_ids=0, derived=None):
        self.plan = plan
        self.rels = rels
        self.segs = segs  # per atom: [(rows tensor, lo, hi), ...] body first
        self.ok = ok
        self.head_resolved = head_resolved
        self.n_ids = n_ids  # ids are < n_ids (symbol table size)
        self._desc = None
        # relations derived by the running stratum (their indexes change every
        # iteration); None = unknown, treat every index as changing
        self.derived = derived

    def descriptor(self) -> dev.PlanDesc:
        if self._desc is None:
            self._desc = encode_plan(self)
        return self._desc


def prepare(plan: JoinPlan, store, interner, derived=None) -> Prepared:
    ok = True
    rels, segs = [], []
    for pa in plan.atoms:
        rel = _resolve(store, pa)
        src = [(t, 0, t.shape[1]) for t in rel.segments()]
        if pa.n_const:
            ids = [interner.lookup(c) for c in pa.const_values]
            if any(i is None for i in ids):
                src = []
            else:
                narrowed = []
                for t, lo, hi in src:
                    a, b = dev.narrow_prefix(t, lo, hi, ids)
                    if a < b:
                        narrowed.append((t, a, b))
                src = narrowed
        rels.append(rel)
        segs.append(src)
        if not pa.negated and not src:
            ok = False
        if pa.negated and pa.check_level == -1 and src:
            ok = False
    head = tuple((True, x) if kind == VAR else (False, interner.intern(x)) for kind, x in plan.head_cols)
    return Prepared(plan, rels, segs, ok, head, len(interner), derived)


def encode_shape(plan: JoinPlan, head_resolved=None) -> dev.PlanDesc:
    """The static part of the srdl_plan descriptor: depth, atoms, which index
    columns every atom binds at every level, negations, the head projection.
    It is all the per-plan kernel compiler (csrc/wcoj_jit.cu) needs; index
    pointers, row ranges and segment counts are filled in by encode_plan."""
    if plan.depth > dev.MAX_LEVELS or len(plan.atoms) > dev.MAX_ATOMS:
        raise InternalError(f"plan {plan.plan_id}: {plan.depth} variables / {len(plan.atoms)} atoms "
                            f"exceed the device limits ({dev.MAX_LEVELS}/{dev.MAX_ATOMS})")
    if plan.head_arity > dev.MAX_HEAD:
        raise InternalError(f"plan {plan.plan_id}: head arity {plan.head_arity} > {dev.MAX_HEAD}")
    d = dev.PlanDesc()
    d.depth = plan.depth
    d.natoms = len(plan.atoms)
    d.outer = plan.outer_atom if plan.outer_atom is not None else dev.NO_ATOM
    d.inner = plan.inner_atom if plan.inner_atom is not None else dev.NO_ATOM
    d.head_arity = plan.head_arity
    heads = head_resolved if head_resolved is not None else [(kind == VAR, x if kind == VAR else 0)
                                                           for kind, x in plan.head_cols]
    for h, (is_var, x) in enumerate(heads):
        d.head_level[h] = x if is_var else -1
        d.head_const[h] = 0 if is_var else x
    for lvl, specs in enumerate(plan.narrow_specs):
        d.nspec[lvl] = len(specs)
        for j, (a, _cols) in enumerate(specs):
            d.spec[lvl][j] = a
    for a in range(dev.MAX_ATOMS):
        d.leaf_slot[a] = dev.NO_ATOM
    if plan.depth:
        leaf_specs = plan.narrow_specs[plan.depth - 1]
        if len(leaf_specs) > dev.MAX_LEAF_SPECS:
            raise InternalError(f"plan {plan.plan_id}: {len(leaf_specs)} sources on the last variable "
                                f"(device limit {dev.MAX_LEAF_SPECS})")
        for j, (a, _cols) in enumerate(leaf_specs):
            d.leaf_slot[a] = j
    for a in range(dev.MAX_ATOMS):
        d.mid_slot[a] = dev.NO_ATOM
    if plan.depth >= 4:
        deep = [a for a, pa in enumerate(plan.atoms)
                if any(lvl >= plan.depth - 2 for lvl in pa.col_levels)]
        if len(deep) <= dev.MAX_MID_SPECS:
            for slot, a in enumerate(deep):
                d.mid_slot[a] = slot
            d.nmid = len(deep)
    for a, pa in enumerate(plan.atoms):
        if pa.arity > dev.MAX_COLS:
            raise InternalError(f"relation {pa.relation}: arity {pa.arity} > {dev.MAX_COLS}")
        ad = d.atom[a]
        ad.negated = int(pa.negated)
        ad.arity = pa.arity
        ad.nconst = pa.n_const
        ad.check_level = pa.check_level
        for lvl, cols in pa.levels_with_columns().items():
            ad.lvl_col[lvl] = cols[0]
            ad.lvl_ncol[lvl] = len(cols)
    return d


_SHAPES: dict = {}  # id(plan) -> (plan, head_resolved, shape descriptor)


def _shape_template(plan: JoinPlan, head_resolved) -> dev.PlanDesc:
    """encode_shape, memoised per plan object and head constants: the shape
    is fixed for the life of a compiled program, while the descriptor is
    rebuilt for every plan execution (every iteration)."""
    hit = _SHAPES.get(id(plan))
    if hit is None or hit[0] is not plan or hit[1] != head_resolved:
        if len(_SHAPES) > 4096:
            _SHAPES.clear()
        hit = _SHAPES[id(plan)] = (plan, head_resolved, encode_shape(plan, head_resolved))
    return hit[2]


def encode_plan(prep: Prepared) -> dev.PlanDesc:
    """JoinPlan + resolved segments -> the fixed-size srdl_plan descriptor."""
    plan = prep.plan
    d = dev.PlanDesc()
    C.pointer(d)[0] = _shape_template(plan, prep.head_resolved)  # copy of the shape fields
    for a, pa in enumerate(plan.atoms):
        ad = d.atom[a]
        src = prep.segs[a]
        ad.nseg = len(src)
        for s, (rows, lo, hi) in enumerate(src):
            ptrs = dev.col_ptrs(rows)
            for c in range(pa.arity):
                ad.seg[s].cols[c] = ptrs[c]
            ad.seg[s].lo = lo
            ad.seg[s].hi = hi
        if len(src) == 1 and pa.n_const == 0 and src[0][1] == 0 and src[0][2] == src[0][0].shape[1]:
            hist = prep.rels[a].hist
            if hist.nkeys and hist_covers(prep.rels[a], src[0][0]):
                ad.hkeys = hist.keys.data_ptr()
                ad.hprefix = hist.prefix.data_ptr()
                ad.hk = hist.nkeys
                fence = hist.fence()
                if fence is not None:
                    ad.hfence = fence.data_ptr()
                    ad.hfn = fence.numel()
                static = prep.derived is not None and pa.relation not in prep.derived
                dense = prep.rels[a].dense_offsets(prep.n_ids, static) if prep.n_ids else None
                if dense is not None:
                    ad.doff = dense.data_ptr()
                    ad.dn = prep.n_ids
    return d


KERNEL_MODES = {"count": 0, "materialize": 1, "spec": 2}


def jit_prepare(plans, mode="spec", wait=False) -> int:
    """Schedule the per-plan kernels of `plans` (csrc/wcoj_jit.cu: NVRTC on
    the background compiler threads, disk-cached) so they are ready before
    the first iterations need them; wait=True blocks until they are built.
    Returns how many of the plans have one ready (0 with the JIT off)."""
    plans = [p for p in plans if p.depth]
    if not plans:
        return 0
    arr = (dev.PlanDesc * len(plans))(*[encode_shape(p) for p in plans])
    return dev.lib().srdl_wcoj_jit_prepare(arr, len(plans), KERNEL_MODES[mode], int(wait))


def emits_sorted_distinct(plan: JoinPlan) -> bool:
    """The plan's output, in emission order, is strictly increasing: its head
    is every variable in level order (one row per binding, so distinct) and
    the walk enumerates bindings lexicographically — slices are contiguous
    in root-key order, rectangles row-major, candidates and leaf batches in
    row order, merge-path parents in lane order (csrc/wcoj_kernel.cuh)."""
    return bool(plan.depth) and plan.head_arity == plan.depth and all(
        kind == VAR and x == h for h, (kind, x) in enumerate(plan.head_cols))


def execution_sorted(prep: "Prepared") -> bool:
    """This execution of the plan emits strictly increasing rows: the plan
    does (emits_sorted_distinct) and every source is ONE sorted segment — an
    index with a head buffer is walked body first, then head, so a level's
    candidates are then two sorted runs, not one."""
    return emits_sorted_distinct(prep.plan) and all(len(src) <= 1 for src in prep.segs)


def hist_covers(rel, rows) -> bool:
    """The index histogram describes exactly `rows` (its only segment)."""
    return rel.size == rows.shape[1]


class DevicePartition:
    """Root work space on the device (keys, outer degrees, d2, prefix, and
    the first outer/inner row of every key when the sources are single
    segments)."""

    __slots__ = ("keys", "outer_degrees", "d2", "prefix", "outer_lo", "inner_lo", "p", "nwarps",
                 "nslices", "_total")

    def __init__(self, keys, outer_degrees, d2, prefix, p, outer_lo=None, inner_lo=None):
        self.keys = keys
        self.outer_degrees = outer_degrees
        self.d2 = d2
        self.prefix = prefix
        self.outer_lo = outer_lo
        self.inner_lo = inner_lo
        self.p = p
        self.nwarps = device_warps(p)
        self.nslices = self.nwarps * SLICES_PER_WARP
        self._total = None

    @classmethod
    def empty(cls, p: int) -> "DevicePartition":
        z32 = torch.empty(0, dtype=dev.U32, device=dev.device())
        return cls(z32, z32, z32, torch.empty(0, dtype=dev.U64, device=dev.device()), p)

    @property
    def nkeys(self) -> int:
        return self.keys.numel()

    @property
    def total(self) -> int:
        if self._total is None:
            self._total = int(self.prefix[-1].item()) if self.nkeys else 0
        return self._total

    def to_host(self, p: int | None = None) -> WorkPartition:
        """The same partition in the reference's numpy form."""
        return WorkPartition(
            self.keys.cpu().numpy(),
            self.outer_degrees.cpu().numpy().astype(np.int64),
            self.d2.cpu().numpy().astype(np.int64),
            p or self.p,
        )

    def slices_used(self) -> int:
        """Slices the kernels cut [0, T) into (csrc/wcoj_kernel.cuh `slices_used`)."""
        used = max(-(-self.total // MIN_SLICE_UNITS), min(self.nwarps * 4, self.total))
        return min(max(used, 1), self.nslices)

    def max_slice(self) -> int:
        t = self.total
        return -(-t // self.slices_used()) if t else 0


def build_partition(plan: JoinPlan, store, p: int, prep: Prepared | None = None, interner=None,
                    dist=None):
    if p < 1:
        raise InternalError("worker count must be >= 1")
    if prep is None:
        prep = prepare(plan, store, interner)
    if plan.depth == 0 or not prep.ok:
        return DevicePartition.empty(p)
    outer = plan.atoms[plan.outer_atom]
    if outer.n_const == 0:
        hist = prep.rels[plan.outer_atom].hist
    else:
        from .columns import Histogram

        hist = Histogram.empty()
        for rows, lo, hi in prep.segs[plan.outer_atom]:
            hist = hist.updated(rows[outer.n_const, lo:hi].contiguous())
    okeys, odeg = hist.keys, hist.degrees
    if okeys.numel() == 0:
        return DevicePartition.empty(p)
    single_outer = len(prep.segs[plan.outer_atom]) == 1
    if plan.inner_atom is not None:
        ih = prep.rels[plan.inner_atom].hist
        single_inner = len(prep.segs[plan.inner_atom]) == 1
        d2, prefix, olo, ilo = dev.root_work(okeys, odeg, hist.prefix, ih.keys, ih.degrees, ih.prefix,
                                             outer_rows=single_outer, inner_rows=single_inner)
    else:
        d2, prefix, olo, ilo = dev.root_work(okeys, odeg, hist.prefix, outer_rows=single_outer)
    if dist is not None and dist.world > 1:
        dev.root_own(okeys, odeg, d2, prefix, dist.world, dist.rank)  # this rank's root keys only
    return DevicePartition(okeys, odeg, d2, prefix, p, olo, ilo)


@dataclass
class CountResult:
    """Per-slice counts (device), their exclusive prefix and the total."""

    slice_counts: torch.Tensor
    slice_offsets: torch.Tensor
    total_dev: torch.Tensor
    ticket: torch.Tensor | None = None
    _total: int | None = None
    spec: "SpecArena | None" = None  # speculative output of the count walk
    spills: int | None = None  # slices the arena could not hold (host, after readback)
    event: list | None = None  # the count launch's dev.PROFILE record (bench)

    @classmethod
    def none(cls) -> "CountResult":
        """A plan with no root work: nothing on the device, total 0."""
        return cls(None, None, None, None, 0)

    @classmethod
    def constant(cls, n_slices: int, first: int) -> "CountResult":
        d = dev.device()
        counts = torch.zeros(n_slices, dtype=dev.U64, device=d)
        counts[0] = first
        offs = torch.zeros(n_slices, dtype=dev.U64, device=d)
        offs[1:] = first
        return cls(counts, offs, torch.full((1,), first, dtype=dev.U64, device=d), None, first)

    @property
    def total(self) -> int:
        if self._total is None:
            self._total = int(self.total_dev.item())
        return self._total

    @property
    def tc(self) -> np.ndarray:
        return self.slice_counts.cpu().numpy()

    @property
    def offsets(self) -> np.ndarray:
        return self.slice_offsets.cpu().numpy()


def _exec_desc(partition: DevicePartition, counts: CountResult, out=None, error=None,
               bitmap=None) -> dev.ExecDesc:
    x = dev.ExecDesc()
    x.keys = partition.keys.data_ptr()
    x.d2 = partition.d2.data_ptr()
    x.prefix = partition.prefix.data_ptr()
    x.outer_deg = partition.outer_degrees.data_ptr()
    x.outer_lo = partition.outer_lo.data_ptr() if partition.outer_lo is not None else None
    x.inner_lo = partition.inner_lo.data_ptr() if partition.inner_lo is not None else None
    x.nkeys = partition.nkeys
    x.nwarps = partition.nwarps
    x.nslices = partition.nslices
    x.min_units = MIN_SLICE_UNITS
    x.ticket = counts.ticket.data_ptr()
    x.slice_counts = counts.slice_counts.data_ptr()
    x.slice_offsets = counts.slice_offsets.data_ptr()
    x.total = counts.total_dev.data_ptr()
    if out is not None:
        for h in range(out.shape[0]):
            x.out[h] = out[h].data_ptr()
    if error is not None:
        x.error = error.data_ptr()
    if bitmap is not None:
        x.bitmap = bitmap.data_ptr()
    return x


SPEC_CHUNK = int(os.environ.get("SRDL_SPEC_CHUNK", 128))  # tuples per speculative arena chunk (srdl_spec.chunk)


class SpecArena:
    """Device arena the speculative count walk writes into (srdl_spec)."""

    __slots__ = ("cols", "chunk_next", "slice_first", "slice_spill", "meta", "nchunks", "_desc")

    def __init__(self, arity: int, capacity: int, nslices: int, storage: torch.Tensor | None = None,
                 pool=None, key=None):
        """storage: a uint32 device region to carve the tuple columns and
        chunk links from (the engine's persistent arena), else allocated;
        pool/key: a dev.BufferPool slot for the per-slice bookkeeping."""
        d = dev.device()
        per_chunk = SPEC_CHUNK * arity + 1  # tuple columns + one link word
        if storage is not None:
            capacity = min(capacity, (storage.numel() // per_chunk) * SPEC_CHUNK)
        self.nchunks = max(0, capacity // SPEC_CHUNK)
        words = self.nchunks * SPEC_CHUNK
        if storage is None:
            storage = torch.empty(max(self.nchunks * per_chunk, 1), dtype=dev.U32, device=d)
        self.cols = storage[:arity * words].view(arity, words)
        self.chunk_next = storage[arity * words:arity * words + max(self.nchunks, 1)]
        # [spills, cursor], per-slice first chunk and spill flag: one allocation
        parts = ((2, torch.int64), (nslices, dev.U32), (nslices, dev.U32))
        self.meta, self.slice_first, self.slice_spill = (pool.get(key, *parts) if pool is not None
                                                         else dev.carve(*parts))
        self._desc = None

    @property
    def spills_dev(self) -> torch.Tensor:
        return self.meta[0:1]

    def descriptor(self) -> dev.SpecDesc:
        if self._desc is None:
            q = dev.SpecDesc()
            for h in range(self.cols.shape[0]):
                q.cols[h] = self.cols[h].data_ptr()
            q.nchunks = self.nchunks
            q.chunk = SPEC_CHUNK
            q.spills = self.meta.data_ptr()
            q.cursor = self.meta.data_ptr() + 8
            q.chunk_next = self.chunk_next.data_ptr()
            q.slice_first = self.slice_first.data_ptr()
            q.slice_spill = self.slice_spill.data_ptr()
            self._desc = q
        return self._desc


def count_pass(plan, store, partition, prep=None, interner=None, pool=None, spec_capacity=0,
               spec_storage=None, buffers=None, key=None) -> CountResult:
    """Read-only pass: exact per-slice output counts, nothing written.
    spec_capacity > 0: the walk also writes its tuples speculatively into an
    arena of that many tuples (srdl_wcoj_count_spec); materialize_pass then
    gathers them instead of walking again."""
    if prep is None:
        prep = prepare(plan, store, interner)
    n = partition.nslices
    if plan.depth == 0:
        return CountResult.constant(n, 1 if prep.ok else 0)
    if not prep.ok or partition.nkeys == 0:
        return CountResult.constant(n, 0)
    # per-slice counts and offsets, the total, the slice ticket (zeroed by
    # srdl_wcoj_count): one allocation
    parts = ((n, dev.U64), (n, dev.U64), (1, dev.U64), (1, torch.int32))
    counts = CountResult(*(buffers.get(("count", key), *parts) if buffers is not None else dev.carve(*parts)))
    desc = prep.descriptor()
    x = _exec_desc(partition, counts)
    algo = input_bytes(prep) if dev.PROFILE is not None else 0
    if spec_capacity >= SPEC_CHUNK:
        counts.spec = SpecArena(plan.head_arity, spec_capacity, n, spec_storage, buffers,
                                ("spec", key) if buffers is not None else None)
        q = counts.spec.descriptor()
        rc, counts.event = _timed("wcoj_count", lambda: dev.lib().srdl_wcoj_count_spec(
            C.byref(desc), C.byref(x), C.byref(q), dev.stream_handle()), algo)
        dev.check(rc, "wcoj_count_spec")
    else:
        rc, counts.event = _timed("wcoj_count", lambda: dev.lib().srdl_wcoj_count(
            C.byref(desc), C.byref(x), dev.stream_handle()), algo)
        dev.check(rc, "wcoj_count")
    return counts


def materialize_pass(plan, store, partition, counts: CountResult, out_cols, prep=None, interner=None,
                     pool=None, error=None, bitmap=None):
    """Second pass: the same walk, writing every slice's tuples at its offset."""
    if prep is None:
        prep = prepare(plan, store, interner)
    total = counts.total
    if total == 0:
        return out_cols
    if plan.depth == 0:
        vals = [x for _, x in prep.head_resolved]
        out_cols[:, 0] = torch.tensor(vals, dtype=torch.int64).to(torch.uint32).to(out_cols.device)
        if bitmap is not None:
            bitmap += 1
        return out_cols
    own_flag = error is None
    if own_flag:
        error = torch.zeros(1, dtype=torch.int32, device=dev.device())
    desc = prep.descriptor()
    x = _exec_desc(partition, counts, out_cols, error, bitmap)
    out_bytes = 4 * plan.head_arity * total  # every derived tuple written once
    if counts.spec is not None and bitmap is None:
        # the count walk already wrote the tuples: copy them to their offsets,
        # and walk again only the slices the arena could not hold
        q = counts.spec.descriptor()
        spills = counts.spills if counts.spills is not None else int(counts.spec.spills_dev.item())
        if counts.event is not None:  # the count walk wrote the tuples (into the arena)
            counts.event[3] += out_bytes
        prof = dev.PROFILE is not None
        rc, _ = _timed("wcoj_gather", lambda: dev.lib().srdl_wcoj_gather(
            C.byref(desc), C.byref(x), C.byref(q), dev.stream_handle()), 2 * out_bytes if prof else 0)
        dev.check(rc, "wcoj_gather")
        if spills:
            rc, _ = _timed("wcoj_materialize", lambda: dev.lib().srdl_wcoj_materialize_spilled(
                C.byref(desc), C.byref(x), C.byref(q), dev.stream_handle()),
                input_bytes(prep) + out_bytes if prof else 0)
            dev.check(rc, "wcoj_materialize_spilled")
        counts.spec = None  # release the arena
    else:
        rc, _ = _timed("wcoj_materialize", lambda: dev.lib().srdl_wcoj_materialize(
            C.byref(desc), C.byref(x), dev.stream_handle()),
            input_bytes(prep) + out_bytes if dev.PROFILE is not None else 0)
        dev.check(rc, "wcoj_materialize")
    if own_flag and int(error.item()):
        raise InternalError(f"plan {plan.plan_id}: materialized tuple count diverged from the count pass")
    return out_cols


class PlanExecution:
    """One plan's pipeline split into phases so schedulers can interleave
    the same phase of independent plans (reference executor.PlanExecution)."""

    def __init__(self, plan, store, p, interner, pool=None, dist=None, derived=None):
        self.plan = plan
        self.store = store
        self.p = p
        self.interner = interner
        self.dist = dist
        self.derived = derived
        self.prep = None
        self.partition = None
        self.counts = None
        self.out = None
        self.error = None
        self.bitmap = None
        self.aux_peak = 0

    def histogram(self):
        self.prep = prepare(self.plan, self.store, self.interner, self.derived)
        self.partition = build_partition(self.plan, self.store, self.p, self.prep, dist=self.dist)
        if self.plan.depth and self.prep.ok:
            # encode now, on the calling (main) stream: the descriptor builds
            # and caches per-index device data (dense column-0 offsets) that
            # the count kernels of other plans, on other streams, read too
            self.prep.descriptor()
        return self.partition

    # The stream schedule splits histogram() in two: sources + descriptor on
    # the main stream, the root work space on the plan's side stream.

    def prepare_sources(self):
        self.prep = prepare(self.plan, self.store, self.interner, self.derived)
        if self.plan.depth and self.prep.ok:
            self.prep.descriptor()  # may build dense offsets other plans read: main stream
        return self.prep

    def needs_main_stream_partition(self) -> bool:
        """The root work space launches nothing (no work) or needs torch ops
        (a constant-led outer atom: its histogram is rebuilt over the
        narrowed range), so it is built on the main stream."""
        plan = self.plan
        return plan.depth == 0 or not self.prep.ok or plan.atoms[plan.outer_atom].n_const > 0

    def build_root_space(self):
        self.partition = build_partition(self.plan, self.store, self.p, self.prep, dist=self.dist)
        return self.partition

    def has_work(self) -> bool:
        """False when the count pass would launch nothing useful (an empty
        source or no root keys): the stream schedule then skips the plan
        without touching the device."""
        if self.plan.depth == 0:
            return True
        return bool(self.prep.ok) and self.partition.nkeys > 0

    def count(self, spec_capacity: int = 0, spec_storage=None, buffers=None, key=None) -> CountResult:
        """buffers/key: a dev.BufferPool slot for the per-slice arrays (the
        stream schedule reuses one per stream slot across iterations)."""
        self.counts = count_pass(self.plan, self.store, self.partition, self.prep, spec_capacity=spec_capacity,
                                 spec_storage=spec_storage, buffers=buffers, key=key)
        return self.counts

    def allocate(self, out=None):
        total = self.counts.total
        self.out = out if out is not None else dev.empty_rows(self.plan.head_arity, total)
        self.aux_peak = max(self.aux_peak, total)
        if audit.enabled:
            self.bitmap = torch.zeros(total, dtype=torch.int32, device=dev.device())
        return self.out

    def materialize(self, error=None):
        materialize_pass(self.plan, self.store, self.partition, self.counts, self.out, self.prep,
                         error=error, bitmap=self.bitmap)
        if audit.enabled:
            audit.record_execution(self)
        return self.out


def execute_plan(plan, store, p, interner, pool=None) -> torch.Tensor:
    """Histogram, count, allocate once, materialize; returns the staged head
    tuples as a (head_arity, total) device tensor (attribute order)."""
    run = PlanExecution(plan, store, p, interner, pool)
    run.histogram()
    run.count()
    run.allocate()
    return run.materialize()
