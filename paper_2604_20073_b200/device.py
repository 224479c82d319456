"""ctypes binding to libsrdl.so (the C ABI in include/srdl.h) + buffer helpers.

This is the only module that talks to the native library. Device buffers
are torch tensors (PyTorch is used purely as the device allocator and stream
provider); every call passes raw pointers, row counts and the current CUDA
stream. There is no CPU fallback: if the library or a CUDA device is
missing, `lib()` raises DeviceUnavailable.

Layout conventions
  * a row set is a 2-D uint32 tensor of shape (arity, n): row-major over
    columns, so column c is the contiguous vector t[c] (SoA);
  * 64-bit unsigned device arrays (prefix sums, counts) are int64 tensors.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .faults import DeviceUnavailable, InternalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsrdl.so")

MAX_ATOMS = 12
MAX_LEVELS = 12
MAX_COLS = 8
MAX_HEAD = 12
MAX_SEGS = 2
MAX_LEAF_SPECS = 6
MAX_MID_SPECS = 8
MAX_DIFF_SEGS = 8
NO_ATOM = 255
NO_SYMBOL = 0xFFFFFFFF

U32 = torch.uint32
U64 = torch.int64  # bit pattern of uint64 device arrays


class Segment(C.Structure):
    _fields_ = [("cols", C.c_void_p * MAX_COLS), ("lo", C.c_uint32), ("hi", C.c_uint32)]


class AtomDesc(C.Structure):
    _fields_ = [
        ("seg", Segment * MAX_SEGS),
        ("nseg", C.c_uint32),
        ("negated", C.c_uint32),
        ("arity", C.c_uint32),
        ("nconst", C.c_uint32),
        ("check_level", C.c_int32),
        ("lvl_col", C.c_uint8 * MAX_LEVELS),
        ("lvl_ncol", C.c_uint8 * MAX_LEVELS),
        ("hkeys", C.c_void_p),
        ("hprefix", C.c_void_p),
        ("hk", C.c_uint32),
        ("dn", C.c_uint32),
        ("doff", C.c_void_p),
        ("hfence", C.c_void_p),
        ("hfn", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class SpecDesc(C.Structure):
    _fields_ = [
        ("cols", C.c_void_p * MAX_HEAD),
        ("nchunks", C.c_uint32),
        ("chunk", C.c_uint32),
        ("cursor", C.c_void_p),
        ("spills", C.c_void_p),
        ("chunk_next", C.c_void_p),
        ("slice_first", C.c_void_p),
        ("slice_spill", C.c_void_p),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("depth", C.c_uint32),
        ("natoms", C.c_uint32),
        ("outer", C.c_uint32),
        ("inner", C.c_uint32),
        ("head_arity", C.c_uint32),
        ("head_level", C.c_int32 * MAX_HEAD),
        ("head_const", C.c_uint32 * MAX_HEAD),
        ("nspec", C.c_uint32 * MAX_LEVELS),
        ("spec", (C.c_uint8 * MAX_ATOMS) * MAX_LEVELS),
        ("leaf_slot", C.c_uint8 * MAX_ATOMS),
        ("mid_slot", C.c_uint8 * MAX_ATOMS),
        ("nmid", C.c_uint32),
        ("atom", AtomDesc * MAX_ATOMS),
    ]


class ExecDesc(C.Structure):
    _fields_ = [
        ("keys", C.c_void_p),
        ("d2", C.c_void_p),
        ("prefix", C.c_void_p),
        ("outer_deg", C.c_void_p),
        ("outer_lo", C.c_void_p),
        ("inner_lo", C.c_void_p),
        ("nkeys", C.c_uint64),
        ("nwarps", C.c_uint32),
        ("nslices", C.c_uint32),
        ("min_units", C.c_uint64),
        ("ticket", C.c_void_p),
        ("slice_counts", C.c_void_p),
        ("slice_offsets", C.c_void_p),
        ("total", C.c_void_p),
        ("out", C.c_void_p * MAX_HEAD),
        ("error", C.c_void_p),
        ("bitmap", C.c_void_p),
    ]


_LIB = None
_SIGNATURES = {
    "srdl_version": (C.c_int, []),
    "srdl_last_error": (C.c_char_p, []),
    "srdl_sm_count": (C.c_int, []),
    "srdl_launch_count": (C.c_uint64, []),
    "srdl_stream_wait": (C.c_int, [C.c_void_p, C.c_void_p]),
    "srdl_scan_u32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]),
    "srdl_scan_u64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p]),
    "srdl_sort_dedup": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_sort_reorder": (
        C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]
    ),
    "srdl_hset_insert": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32,
                                   C.c_void_p]),
    "srdl_hset_filter": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_uint32,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "srdl_sort_unique_keys": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "srdl_compute_delta": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
         C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_merge": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p],
    ),
    "srdl_is_sorted_strict": (
        C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.POINTER(C.c_int), C.c_void_p]
    ),
    "srdl_gather": (
        C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
    ),
    "srdl_histogram": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_histogram_merge": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
         C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_histogram_union": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
         C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_compute_delta_async": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
         C.c_void_p, C.c_void_p],
    ),
    "srdl_histogram_union_async": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "srdl_wcoj_count_spec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srdl_wcoj_gather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srdl_wcoj_materialize_spilled": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "srdl_max_id": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "srdl_key_fence": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]),
    "srdl_dense_offsets": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]
    ),
    "srdl_narrow_prefix": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64),
         C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_root_work": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "srdl_wcoj_count": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(ExecDesc), C.c_void_p]),
    "srdl_wcoj_jit_prepare": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int, C.c_int]),
    "srdl_wcoj_jit_wait": (None, []),
    "srdl_wcoj_jit_shutdown": (None, []),
    "srdl_wcoj_jit_set_mode": (C.c_int, [C.c_int]),
    "srdl_wcoj_jit_source": (C.c_uint64, [C.c_void_p, C.c_int, C.c_char_p, C.c_uint64]),
    "srdl_wcoj_jit_compile_check": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]),
    "srdl_wcoj_jit_stats": (None, [C.POINTER(C.c_uint64)]),
    "srdl_wcoj_materialize": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(ExecDesc), C.c_void_p]),
    "srdl_route_rows": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "srdl_route_pack": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "srdl_unpack_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "srdl_filter_owned": (
        C.c_int,
        [C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
         C.POINTER(C.c_uint64), C.c_void_p],
    ),
    "srdl_root_own": (
        C.c_int,
        [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p],
    ),
    "srdl_gen_rmat": (
        C.c_int,
        [C.c_uint32, C.c_uint64, C.c_float, C.c_float, C.c_float, C.c_uint64, C.c_void_p,
         C.c_void_p, C.c_void_p],
    ),
}


def load_library(path: str | None = None):
    """Open libsrdl.so and declare its C signatures (no CUDA needed).
    SRDL_LIBRARY names an alternative in-tree build (A/B experiments)."""
    path = path or os.environ.get("SRDL_LIBRARY") or LIB_PATH
    if not os.path.exists(path):
        raise DeviceUnavailable(
            f"{path} is missing: build it with `python -m paper_2604_20073_b200.build` "
            "(the engine has no CPU fallback)"
        )
    lib = C.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded library, after checking that a CUDA device is usable."""
    global _LIB
    if _LIB is None:
        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device: the sm_100a engine has no CPU fallback")
        _LIB = load_library()
        if _LIB.srdl_version() != 1:
            raise DeviceUnavailable("libsrdl.so version mismatch; rebuild it")
        import atexit

        # background kernel compiles must not outlive the interpreter
        atexit.register(_LIB.srdl_wcoj_jit_shutdown)
    return _LIB


JIT_MODES = {"off": 0, "async": 1, "sync": 2}


def jit_stats() -> dict:
    """Per-plan kernel compiler counters (csrc/wcoj_jit.cu)."""
    out = (C.c_uint64 * 4)()
    lib().srdl_wcoj_jit_stats(out)
    mode = {v: k for k, v in JIT_MODES.items()}.get(int(out[3]), "?")
    return {"compiled": int(out[0]), "disk_hits": int(out[1]), "failures": int(out[2]), "mode": mode}


def jit_mode(mode: str) -> str:
    """Set the per-plan kernel mode ("off", "async", "sync"); returns the
    previous one."""
    prev = lib().srdl_wcoj_jit_set_mode(JIT_MODES[mode])
    return {v: k for k, v in JIT_MODES.items()}[prev]


def jit_wait():
    """Block until the background kernel compiler is idle."""
    lib().srdl_wcoj_jit_wait()


_DEVICES: dict = {}
_get_device = getattr(torch._C, "_cuda_getDevice", None)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def device() -> torch.device:
    """The current CUDA device (cached torch.device per index: the engine
    asks for it on every buffer allocation)."""
    i = _get_device() if _get_device is not None else torch.cuda.current_device()
    d = _DEVICES.get(i)
    if d is None:
        d = _DEVICES[i] = torch.device("cuda", i)
    return d


_LAUNCH = None  # (torch Stream, handle) while launch_on() is active


class launch_on:
    """Launch library calls on `stream` while buffers keep being allocated on
    torch's current stream. The engine uses it for fork-join phases: the
    main stream launches nothing between the fork (stream.wait_stream(main))
    and the join (main.wait_stream(stream)), so memory freed by the host in
    between is only reused by main-stream work ordered after the join."""

    def __init__(self, stream):
        self.stream = stream

    def __enter__(self):
        global _LAUNCH
        self.prev = _LAUNCH
        _LAUNCH = (self.stream, self.stream.cuda_stream)
        return self

    def __exit__(self, *exc):
        global _LAUNCH
        _LAUNCH = self.prev


def _uses(*tensors):
    """Inside launch_on(): the side stream reads these tensors, so the
    caching allocator must not reuse their memory before that stream gets
    past this point (a temporary the host drops right after the launch)."""
    if _LAUNCH is not None:
        s = _LAUNCH[0]
        for t in tensors:
            if t is not None and t.numel():
                t.record_stream(s)


def stream_wait(waiter, signaler):
    """Order `waiter` after the work launched so far on `signaler` (torch
    Streams; libsrdl's event ring instead of Stream.wait_stream)."""
    check(_LIB.srdl_stream_wait(waiter.cuda_stream, signaler.cuda_stream), "stream_wait")


def stream_handle() -> int:
    """cudaStream_t library calls launch on: the launch_on() stream, else
    torch's current stream on the current device (the raw accessor:
    torch.cuda.current_stream() builds a Stream object per call, a
    measurable cost at thousands of library calls per fixpoint)."""
    if _LAUNCH is not None:
        return _LAUNCH[1]
    if _raw_stream is not None and _get_device is not None:
        return _raw_stream(_get_device())
    return torch.cuda.current_stream().cuda_stream


# Benchmark hook: when a list, every library call made through `timed`
# appends [family, start_event, end_event, algorithmic_bytes] recorded on
# the launching (current) stream; bench.py reads them after the timed steps.
PROFILE = None


def timed(family: str, algo_bytes: int, fn):
    """Run fn (one C-ABI call); under PROFILE bracket it with CUDA events on
    the current stream. Returns (fn's result, the record or None) — callers
    that learn the output size only later may add to record[3]."""
    if PROFILE is None:
        return fn(), None
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    on = _LAUNCH[0] if _LAUNCH is not None else None
    a.record(on)
    rc = fn()
    b.record(on)
    rec = [family, a, b, int(algo_bytes)]
    PROFILE.append(rec)
    return rc, rec


def check(rc: int, what: str):
    if rc != 0:
        msg = _LIB.srdl_last_error().decode(errors="replace") if _LIB else "?"
        raise InternalError(f"{what} failed ({rc}): {msg}")


_SM = None


def sm_count() -> int:
    global _SM
    if _SM is None:
        n = lib().srdl_sm_count()
        _SM = n if n > 0 else 148
    return _SM


# ---------------------------------------------------------------- buffers


def carve(*parts):
    """Several device buffers from ONE allocation: parts are (n, dtype)
    pairs; returns one tensor view per part (each 256-byte aligned). The
    engine allocates a few buffers per library call thousands of times per
    fixpoint; one allocation per call instead of several is a measurable
    share of the host time per iteration (tools/host_profile.py)."""
    offs, total = [], 0
    for n, dt in parts:
        offs.append(total)
        total += -(-max(int(n), 0) * _ITEMSIZE[dt] // 256) * 256
    buf = torch.empty(max(total, 256), dtype=torch.uint8, device=device())
    return [buf[o:o + int(n) * _ITEMSIZE[dt]].view(dt) for o, (n, dt) in zip(offs, parts)]


_ITEMSIZE = {torch.uint32: 4, torch.int32: 4, torch.int64: 8, torch.uint8: 1}


def empty_rows(arity: int, n: int = 0) -> torch.Tensor:
    return torch.empty((arity, n), dtype=U32, device=device())


def to_device_rows(cols) -> torch.Tensor:
    """Host columns (sequence of 1-D arrays) -> (arity, n) uint32 device tensor."""
    import numpy as np

    arr = np.ascontiguousarray(np.stack([np.asarray(c, dtype=np.uint32) for c in cols]))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def nrows(rows: torch.Tensor) -> int:
    return rows.shape[1]


def col_ptrs(rows: torch.Tensor, order=None):
    """ctypes array of column pointers (optionally permuted to `order`)."""
    arity = rows.shape[0]
    order = range(arity) if order is None else order
    base = rows.data_ptr()
    stride = rows.stride(0) * 4
    # a single-row set may carry any stride on the row axis (e.g. a transposed
    # (1, arity) tensor); column c still starts at base + c * stride(0)
    if rows.shape[1] > 1 and rows.stride(1) != 1:
        raise InternalError("row set columns must be contiguous")
    ptrs = (C.c_void_p * MAX_COLS)()
    for k, c in enumerate(order):
        ptrs[k] = base + c * stride
    return ptrs


def sym_bits(nsym: int) -> int:
    return max(1, int(nsym - 1).bit_length()) if nsym > 1 else 1


# ------------------------------------------------------------- operations


def sort_dedup(rows: torch.Tensor, bits: int = 32, order=None, distinct: bool = False) -> torch.Tensor:
    """Distinct rows sorted lexicographically (columns taken in `order`).
    distinct=True: the rows are known to be distinct (no host round trip)."""
    arity, n = rows.shape
    order = list(range(arity)) if order is None else list(order)
    out = empty_rows(len(order), n)
    if n == 0:
        return out
    got = C.c_uint64(0)
    _uses(rows, out)
    rc, rec = timed("sort_dedup", 4 * arity * n, lambda: lib().srdl_sort_dedup(
        col_ptrs(rows, order), len(order), n, bits, col_ptrs(out), None if distinct else C.byref(got),
        stream_handle()))
    check(rc, "sort_dedup")
    if rec is not None:
        rec[3] += 4 * len(order) * (n if distinct else got.value)
    return out if distinct else _trim(out, got.value)


def reorder_key_columns(order) -> int:
    """For rows sorted in attribute order, the number of leading columns of
    `order` a stable sort must key on so that the rows end up sorted in
    `order`: the smallest P whose remaining columns order[P:] keep their
    attribute order (0 = already in order)."""
    order = list(order)
    for p in range(len(order) + 1):
        if order[p:] == sorted(order[p:]):
            return p
    return len(order)


def sort_reorder(rows: torch.Tensor, bits: int, order) -> torch.Tensor:
    """Distinct rows sorted in attribute order, re-sorted under `order` with
    one stable sort on its leading columns (srdl_sort_reorder); falls back
    to the full sort when those columns do not fit a 64-bit key."""
    arity, n = rows.shape
    order = list(order)
    nkey = reorder_key_columns(order)
    if nkey == 0:
        return rows
    if nkey * bits > 64:
        return sort_dedup(rows, bits, order=order, distinct=True)
    out = empty_rows(arity, n)
    if n == 0:
        return out
    _uses(rows, out)
    rc, _ = timed("sort_dedup", 8 * arity * n, lambda: lib().srdl_sort_reorder(
        col_ptrs(rows, order), arity, n, bits, nkey, col_ptrs(out), stream_handle()))
    check(rc, "sort_reorder")
    return out


class HashSet:
    """Device hash set of a relation's packed rows (csrc/hashset.cu): the
    full relation's membership test for Compute Delta, kept up to date by
    inserting each delta. Capacity a power of two, at most half full."""

    def __init__(self, arity: int, bits: int, expect: int):
        self.arity, self.bits = arity, bits
        self.log2cap = max(10, int(2 * max(expect, 1) - 1).bit_length())
        self.slots = torch.full((1 << self.log2cap,), -1, dtype=torch.int64, device=device())
        self.size = 0

    def fits(self, extra: int) -> bool:
        return 2 * (self.size + extra) <= (1 << self.log2cap)

    def insert(self, rows: torch.Tensor):
        n = rows.shape[1]
        if n:
            _uses(rows, self.slots)
            rc, _ = timed("compute_delta", 4 * self.arity * n + 8 * n, lambda: lib().srdl_hset_insert(
                self.slots.data_ptr(), self.log2cap, col_ptrs(rows), self.arity, n, self.bits, stream_handle()))
            check(rc, "hset_insert")
            self.size += n

    def filter(self, rows: torch.Tensor, count_slot: torch.Tensor):
        """(u64 keys of the rows not in the set, compacted, capacity n; their
        count lands in count_slot) — no host round trip."""
        n = rows.shape[1]
        keys = torch.empty(max(n, 1), dtype=torch.int64, device=device())
        _uses(rows, self.slots, keys)
        rc, _ = timed("compute_delta", 4 * self.arity * n + 8 * n, lambda: lib().srdl_hset_filter(
            col_ptrs(rows) if n else None, self.arity, n, self.bits, self.slots.data_ptr(), self.log2cap,
            keys.data_ptr(), count_slot.data_ptr(), stream_handle()))
        check(rc, "hset_filter")
        return keys


def sort_unique_keys(keys: torch.Tensor, m: int, arity: int, bits: int, count_slot: torch.Tensor):
    """Distinct rows (arity, capacity m) of m packed keys, sorted; the row
    count lands in count_slot."""
    out = empty_rows(arity, m)
    _uses(keys, out)
    rc, rec = timed("compute_delta", 16 * m, lambda: lib().srdl_sort_unique_keys(
        keys.data_ptr(), m, arity, bits, col_ptrs(out) if m else None, count_slot.data_ptr(), stream_handle()))
    check(rc, "sort_unique_keys")
    return out, rec


def compute_delta(rows: torch.Tensor, segments, bits: int = 32) -> torch.Tensor:
    """sort_dedup(rows) minus the rows of the given sorted segments."""
    arity, n = rows.shape
    out = empty_rows(arity, n)
    if n == 0:
        return out
    segs = [s for s in segments if nrows(s)]
    if len(segs) > MAX_DIFF_SEGS:
        raise InternalError(f"compute_delta: at most {MAX_DIFF_SEGS} segments")
    seg_ptr_arrays = [col_ptrs(s) for s in segs]
    seg_cols = (C.c_void_p * MAX_DIFF_SEGS)(*[C.addressof(a) for a in seg_ptr_arrays])
    seg_rows = (C.c_uint64 * MAX_DIFF_SEGS)(*[nrows(s) for s in segs])
    got = C.c_uint64(0)
    rc, rec = timed("compute_delta", 4 * arity * n, lambda: lib().srdl_compute_delta(
        col_ptrs(rows), arity, n, bits, seg_cols, seg_rows, len(segs), col_ptrs(out), C.byref(got),
        stream_handle()))
    check(rc, "compute_delta")
    if rec is not None:
        rec[3] += 4 * arity * got.value
    return _trim(out, got.value)


def compute_delta_async(rows: torch.Tensor, segments, bits: int, count_slot: torch.Tensor):
    """compute_delta into a capacity-n buffer; the row count is written to
    count_slot (a 1-element uint32 device tensor) without a host round trip.
    Returns the buffer and the PROFILE record (None when not profiling): the
    caller adds the written bytes (4 * arity * count) once it reads the count."""
    arity, n = rows.shape
    out = empty_rows(arity, n)
    segs = [s for s in segments if nrows(s)]
    if len(segs) > MAX_DIFF_SEGS:
        raise InternalError(f"compute_delta: at most {MAX_DIFF_SEGS} segments")
    seg_ptr_arrays = [col_ptrs(s) for s in segs]
    seg_cols = (C.c_void_p * MAX_DIFF_SEGS)(*[C.addressof(a) for a in seg_ptr_arrays])
    seg_rows = (C.c_uint64 * MAX_DIFF_SEGS)(*[nrows(s) for s in segs])
    _uses(rows, out, *segs)
    rc, rec = timed("compute_delta", 4 * arity * n, lambda: lib().srdl_compute_delta_async(
        col_ptrs(rows) if n else None, arity, n, bits, seg_cols, seg_rows, len(segs),
        col_ptrs(out) if n else None, count_slot.data_ptr(), stream_handle()))
    check(rc, "compute_delta_async")
    return out, rec


class BufferPool:
    """Reusable device buffers for per-iteration outputs whose capacity is
    known before their size: `get(key, parts)` returns views (as `carve`)
    into a buffer kept under `key` and grown by 1.5x when too small. The
    caller guarantees that the previous contents of a key are dead when it
    asks again (ping-pong keys for outputs that must survive one iteration).
    Per-iteration capacity allocations of 10-100 MB each were the largest
    host cost of an iteration (tools/host_profile.py: torch.empty)."""

    def __init__(self):
        self.bufs = {}

    def get(self, key, *parts):
        offs, total = [], 0
        for n, dt in parts:
            offs.append(total)
            total += -(-max(int(n), 0) * _ITEMSIZE[dt] // 256) * 256
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < total:
            buf = self.bufs[key] = torch.empty(max(int(total * 1.5), 256), dtype=torch.uint8, device=device())
        return [buf[o:o + int(n) * _ITEMSIZE[dt]].view(dt) for o, (n, dt) in zip(offs, parts)]


def histogram_union_async(col: torch.Tensor, fkeys: torch.Tensor, fdeg: torch.Tensor, k_slots: torch.Tensor,
                          pool: BufferPool | None = None, key=None):
    """histogram_union with capacity-sized outputs; (K_delta, K_union) are
    written to k_slots[0:2] (uint32 device tensor) without a round trip.
    pool/key: take the outputs from a BufferPool instead of allocating."""
    n, nf = col.numel(), fkeys.numel()
    parts = ((n, U32), (n, U32), (n, U64), (n + nf, U32), (n + nf, U32), (n + nf, U64))
    dk, dd, dp, uk, ud, up = pool.get(key, *parts) if pool is not None else carve(*parts)
    _uses(col, fkeys, fdeg, dk, uk)
    # algorithmic: the delta column, the full histogram (keys + degrees) read
    # once, both histograms written (key, degree, prefix: 16 B per key; sized
    # here by their upper bounds n and n + nf)
    rc, _ = timed("histogram", 4 * n + 8 * nf, lambda: lib().srdl_histogram_union_async(
        col.data_ptr() if n else None, n, fkeys.data_ptr() if nf else None, fdeg.data_ptr() if nf else None, nf,
        dk.data_ptr(), dd.data_ptr(), dp.data_ptr(), uk.data_ptr(), ud.data_ptr(), up.data_ptr(),
        k_slots.data_ptr(), stream_handle()))
    check(rc, "histogram_union_async")
    return (dk, dd, dp), (uk, ud, up)


def merge(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Sorted union of two sorted, disjoint row sets."""
    arity = a.shape[0]
    na, nb = nrows(a), nrows(b)
    if nb == 0:
        return a
    if na == 0:
        return b
    out = empty_rows(arity, na + nb)
    _uses(a, b, out)
    rc, _ = timed("merge", 8 * arity * (na + nb), lambda: lib().srdl_merge(
        col_ptrs(a), na, col_ptrs(b), nb, arity, col_ptrs(out), stream_handle()))
    check(rc, "merge")
    return out


def is_sorted_strict(rows: torch.Tensor) -> bool:
    ok = C.c_int(1)
    arity, n = rows.shape
    if n <= 1:
        return True
    rc, _ = timed("is_sorted", 4 * arity * n, lambda: lib().srdl_is_sorted_strict(
        col_ptrs(rows), arity, n, C.byref(ok), stream_handle()))
    check(rc, "is_sorted_strict")
    return bool(ok.value)


def gather(rows: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    arity = rows.shape[0]
    n = idx.numel()
    out = empty_rows(arity, n)
    if n:
        check(lib().srdl_gather(col_ptrs(rows), arity, idx.data_ptr(), n, col_ptrs(out),
                                stream_handle()), "gather")
    return out


def histogram(col: torch.Tensor):
    """(keys u32, degrees u32, inclusive prefix i64) of a sorted column."""
    n = col.numel()
    keys = torch.empty(n, dtype=U32, device=device())
    deg = torch.empty(n, dtype=U32, device=device())
    prefix = torch.empty(n, dtype=U64, device=device())
    if n == 0:
        return keys, deg, prefix
    k = C.c_uint64(0)
    rc, rec = timed("histogram", 4 * n, lambda: lib().srdl_histogram(
        col.data_ptr(), n, keys.data_ptr(), deg.data_ptr(), prefix.data_ptr(), C.byref(k), stream_handle()))
    check(rc, "histogram")
    K = k.value
    if rec is not None:
        rec[3] += 16 * K
    return keys[:K], deg[:K], prefix[:K]


def histogram_merge(ka, da, kb, db):
    na, nb = ka.numel(), kb.numel()
    n = na + nb
    keys = torch.empty(n, dtype=U32, device=device())
    deg = torch.empty(n, dtype=U32, device=device())
    prefix = torch.empty(n, dtype=U64, device=device())
    k = C.c_uint64(0)
    rc, rec = timed("histogram", 8 * (na + nb), lambda: lib().srdl_histogram_merge(
        ka.data_ptr(), da.data_ptr(), na, kb.data_ptr(), db.data_ptr(), nb, keys.data_ptr(), deg.data_ptr(),
        prefix.data_ptr(), C.byref(k), stream_handle()))
    check(rc, "histogram_merge")
    K = k.value
    if rec is not None:
        rec[3] += 16 * K
    return keys[:K], deg[:K], prefix[:K]


def histogram_union(col: torch.Tensor, fkeys: torch.Tensor, fdeg: torch.Tensor):
    """(delta histogram of the sorted column, union with (fkeys, fdeg)) as two
    (keys, degrees, prefix) triples, one host round trip."""
    n, nf = col.numel(), fkeys.numel()
    d = device()
    dk = torch.empty(n, dtype=U32, device=d)
    dd = torch.empty(n, dtype=U32, device=d)
    dp = torch.empty(n, dtype=U64, device=d)
    uk = torch.empty(n + nf, dtype=U32, device=d)
    ud = torch.empty(n + nf, dtype=U32, device=d)
    up = torch.empty(n + nf, dtype=U64, device=d)
    if n == 0:
        return (dk, dd, dp), (fkeys, fdeg, None)
    kd, ku = C.c_uint64(0), C.c_uint64(0)
    rc, rec = timed("histogram", 4 * n + 8 * nf, lambda: lib().srdl_histogram_union(
        col.data_ptr(), n, fkeys.data_ptr() if nf else None, fdeg.data_ptr() if nf else None, nf, dk.data_ptr(),
        dd.data_ptr(), dp.data_ptr(), C.byref(kd), uk.data_ptr(), ud.data_ptr(), up.data_ptr(), C.byref(ku),
        stream_handle()))
    check(rc, "histogram_union")
    a, b = kd.value, ku.value
    if rec is not None:
        rec[3] += 16 * (a + b)
    return (dk[:a], dd[:a], dp[:a]), (uk[:b], ud[:b], up[:b])


FENCE = 64  # SRDL_FENCE


def max_ids(row_sets) -> list:
    """Largest id of each uint32 row set, one kernel per set and ONE host
    read for all of them."""
    out = torch.zeros(max(len(row_sets), 1), dtype=torch.int32, device=device())
    for i, rows in enumerate(row_sets):
        check(lib().srdl_max_id(col_ptrs(rows) if rows.numel() else None, rows.shape[0], rows.shape[1],
                                out[i:i + 1].data_ptr(), stream_handle()), "max_id")
    return [int(v) & 0xFFFFFFFF for v in out.tolist()][:len(row_sets)]


def scan(x: torch.Tensor, exclusive: bool = True):
    """(prefix sums of a 1-D uint32 / int64 device tensor, total or None)."""
    n = x.numel()
    out = torch.empty_like(x)
    total = torch.zeros(1, dtype=x.dtype, device=x.device) if exclusive else None
    fn = lib().srdl_scan_u64 if x.element_size() == 8 else lib().srdl_scan_u32
    check(fn(x.data_ptr() if n else None, out.data_ptr() if n else None, n, int(exclusive),
             total.data_ptr() if total is not None else None, stream_handle()), "scan")
    return out, total


def key_fence(keys: torch.Tensor) -> torch.Tensor:
    """Every FENCE-th key (first level of the kernels' column-0 search)."""
    n = keys.numel()
    out = torch.empty(-(-n // FENCE), dtype=U32, device=device())
    if n:
        check(lib().srdl_key_fence(keys.data_ptr(), n, out.data_ptr(), stream_handle()), "key_fence")
    return out


def dense_offsets(keys, prefix, n_ids: int) -> torch.Tensor:
    """CSR offsets of a sorted column from its histogram (n_ids + 1 entries)."""
    off = torch.empty(n_ids + 1, dtype=U32, device=device())
    check(lib().srdl_dense_offsets(keys.data_ptr() if keys.numel() else None,
                                   prefix.data_ptr() if prefix.numel() else None, keys.numel(),
                                   n_ids, off.data_ptr(), stream_handle()), "dense_offsets")
    return off


def narrow_prefix(rows: torch.Tensor, lo: int, hi: int, values) -> tuple:
    """Rows within [lo, hi) whose leading columns equal `values`."""
    if lo >= hi or not values:
        return lo, hi
    vals = (C.c_uint32 * MAX_COLS)(*values)
    a, b = C.c_uint64(0), C.c_uint64(0)
    sub = rows[:, lo:hi]
    ptrs = (C.c_void_p * MAX_COLS)()
    for c in range(len(values)):
        ptrs[c] = sub[c].data_ptr()
    check(lib().srdl_narrow_prefix(ptrs, hi - lo, vals, len(values), C.byref(a), C.byref(b),
                                   stream_handle()), "narrow_prefix")
    return lo + a.value, lo + b.value


def root_work(okeys, odeg, oprefix=None, ikeys=None, ideg=None, iprefix=None, outer_rows=False,
              inner_rows=False):
    """Root work space: (d2 u32, inclusive work prefix i64, outer_lo, inner_lo).

    outer_lo / inner_lo (u32 first row of every key) are produced only when
    requested (single-segment sources); else None."""
    nk = okeys.numel()
    d2, prefix, olo, ilo = carve((nk, U32), (nk, U64), (nk if outer_rows else 0, U32), (nk if inner_rows else 0, U32))
    olo = olo if outer_rows else None
    ilo = ilo if inner_rows else None
    if nk == 0:
        return d2, prefix, olo, ilo
    has_inner = ikeys is not None
    nik = ikeys.numel() if has_inner else 0

    def p(t):
        return t.data_ptr() if t is not None and t.numel() else None

    rc, _ = timed("root_work", 24 * nk, lambda: lib().srdl_root_work(
        okeys.data_ptr(), odeg.data_ptr(), p(oprefix), nk, p(ikeys) if has_inner else None,
        p(ideg) if has_inner else None, p(iprefix) if has_inner else None, nik, int(has_inner), d2.data_ptr(),
        prefix.data_ptr(), p(olo), p(ilo), stream_handle()))
    check(rc, "root_work")
    return d2, prefix, olo, ilo


def owner(values, world: int):
    """Host mirror of the device owner hash (numpy array or int)."""
    import numpy as np

    v = np.asarray(values, dtype=np.uint64)
    return (((v * np.uint64(2654435761)) & np.uint64(0xFFFFFFFF)) >> np.uint64(8)) % np.uint64(world)


def route_rows(rows: torch.Tensor, key_col: int, world: int):
    """Rows grouped by owner rank of column key_col -> (routed rows, counts)."""
    arity, n = rows.shape
    out = empty_rows(arity, n)
    counts = (C.c_uint64 * max(world, 1))()
    check(lib().srdl_route_rows(col_ptrs(rows), arity, n, key_col, world, col_ptrs(out), counts,
                                stream_handle()), "route_rows")
    return out, [int(counts[r]) for r in range(world)]


def route_pack(rows: torch.Tensor, key_col: int, world: int):
    """(row-major int32 send buffer grouped by owner of column key_col,
    per-rank row counts as an int64 device tensor) — no host round trip."""
    arity, n = rows.shape
    send = torch.empty(n * arity, dtype=torch.int32, device=device())
    counts = torch.empty(world, dtype=torch.int64, device=device())
    check(lib().srdl_route_pack(col_ptrs(rows) if n else None, arity, n, key_col, world,
                                send.data_ptr() if n else None, counts.data_ptr(), stream_handle()), "route_pack")
    return send, counts


def unpack_rows(recv: torch.Tensor, arity: int, n: int) -> torch.Tensor:
    """Row-major received rows -> (arity, n) columns."""
    out = empty_rows(arity, n)
    if n:
        check(lib().srdl_unpack_rows(recv.data_ptr(), arity, n, col_ptrs(out), stream_handle()), "unpack_rows")
    return out


def filter_owned(rows: torch.Tensor, key_col: int, world: int, rank: int) -> torch.Tensor:
    arity, n = rows.shape
    out = empty_rows(arity, n)
    got = C.c_uint64(0)
    check(lib().srdl_filter_owned(col_ptrs(rows), arity, n, key_col, world, rank, col_ptrs(out),
                                  C.byref(got), stream_handle()), "filter_owned")
    return _trim(out, got.value)


def root_own(keys, odeg, d2, prefix, world: int, rank: int):
    """Restrict a root work prefix to the keys this rank owns (in place)."""
    if keys.numel():
        check(lib().srdl_root_own(keys.data_ptr(), keys.numel(), odeg.data_ptr(), d2.data_ptr(), world,
                                  rank, prefix.data_ptr(), stream_handle()), "root_own")


def gen_rmat(scale: int, nedges: int, a=0.57, b=0.19, c=0.19, seed=1) -> torch.Tensor:
    out = empty_rows(2, nedges)
    check(lib().srdl_gen_rmat(scale, nedges, a, b, c, seed, out[0].data_ptr(), out[1].data_ptr(),
                              stream_handle()), "gen_rmat")
    return out


def _trim(rows: torch.Tensor, n: int) -> torch.Tensor:
    """Exact-size result: a view when little is wasted, else a compact copy."""
    cap = rows.shape[1]
    if n == cap:
        return rows
    if n >= cap // 2:
        return rows[:, :n]
    return rows[:, :n].clone()
