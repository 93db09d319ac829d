"""ctypes binding of libtrajseek.so (the C-ABI declared in include/trajseek.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is visible, device calls raise ``RuntimeError`` loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRAJSEEK_LIB") or os.path.join(_HERE, "_lib", "libtrajseek.so")

TSK_OK, TSK_EINVAL, TSK_ECUDA, TSK_ENOMEM, TSK_ENODEV, TSK_EFORMAT, TSK_ETOOMANY = 0, 1, 2, 3, 4, 5, 6


class TooManyHits(RuntimeError):
    """One call's result exceeds what a call returns (2^32 rows); the engine
    splits the plan and calls again (the reference grows its accumulator on
    demand)."""
TSK_NOOP = 1 << 0
TSK_ORDER_REFERENCE = 1 << 1
TSK_ORDER_QUERY_MAJOR = 1 << 2
TSK_SPANS_GIVEN = 1 << 3
TSK_WANT_ORDINALS = 1 << 4
TSK_QUERIES_RESIDENT = 1 << 5
TSK_RESULTS_ON_DEVICE = 1 << 6
TSK_ORDER_CANONICAL = 1 << 7
TSK_COUNT_ONLY = 1 << 8
TSK_OVERLAPS_ONLY = 1 << 9
TSK_EXTENT_MEMBER, TSK_EXTENT_GRID = 0, 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)


class Columns(ctypes.Structure):
    """tsk_columns: one sorted store in SoA form."""

    _fields_ = [("n", _I64), ("traj", _P), ("seg", _P)] + [
        (k, _P) for k in ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")
    ]


# Exported symbols and their signatures; tests check the .so exports each one.
SIGNATURES = {
    "tsk_abi_version": ([], ctypes.c_int),
    "tsk_device_count": ([], ctypes.c_int),
    "tsk_last_error": ([], ctypes.c_char_p),
    "tsk_db_create": ([ctypes.c_int, ctypes.POINTER(Columns), ctypes.POINTER(_P)], ctypes.c_int),
    "tsk_db_free": ([_P], None),
    "tsk_db_size": ([_P], _I64),
    "tsk_db_set_host_ids": ([_P, _PI64, _PI64], ctypes.c_int),
    "tsk_sort_by_start": ([ctypes.c_int, _I64, _PD, _PI64], ctypes.c_int),
    "tsk_index_build": ([_P, _I64, ctypes.c_int, _PI64, _PD], ctypes.c_int),
    "tsk_index_copy": ([_P, _PD, _PD, _PI64, _PI64, _PI64], ctypes.c_int),
    "tsk_candidate_ranges": ([_P, _I64, _PD, _PD, _PI64, _PI64], ctypes.c_int),
    "tsk_search": ([_P, ctypes.POINTER(Columns), _I64, _PI64, _PI64, _PI64, _PI64,
                    ctypes.c_double, ctypes.c_uint32, ctypes.POINTER(_P)], ctypes.c_int),
    "tsk_pair_intervals": ([ctypes.c_int, ctypes.POINTER(Columns), ctypes.POINTER(Columns),
                            ctypes.c_double, ctypes.POINTER(_P)], ctypes.c_int),
    "tsk_result_info": ([_P, _PI64, _PI64, _PD], ctypes.c_int),
    "tsk_result_timing": ([_P, _PD, _PD, _PI64], ctypes.c_int),
    "tsk_result_per_batch": ([_P, _PI64], ctypes.c_int),
    "tsk_result_columns": ([_P] + [ctypes.POINTER(_P)] * 8, ctypes.c_int),
    "tsk_result_free": ([_P], None),
    "tsk_probe_fp64": ([ctypes.c_int, _PD, _PD, _PD], ctypes.c_int),
    "tsk_probe_fp32": ([ctypes.c_int, _PD], ctypes.c_int),
    "tsk_k1_stats": ([ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "tsk_db_replicate": ([_P, ctypes.c_int, ctypes.POINTER(_P)], ctypes.c_int),
    "tsk_result_k1_evals": ([_P, _PI64], ctypes.c_int),
    "tsk_plan_setsplit": ([_I64, _PD, _PD, _I64, _PD, _PD, _PI64, _PI64, ctypes.c_int, _I64, _I64,
                           _I64, _PI64, _PI64, _PI64, _PI64, _PI64, _PD], ctypes.c_int),
    "tsk_plan_greedy": ([_I64, _PD, _PD, _I64, _PD, _PD, _PI64, _PI64, ctypes.c_int, _I64, _PI64,
                         _PI64, _PI64, _PI64, _PI64, _PD], ctypes.c_int),
    "tsk_plan_units": ([_I64, _PI64, _PI64, _PI64, _PI64, ctypes.c_int, _I64, _PI64, _I64], _I64),
    "tsk_canonical_order": ([ctypes.c_int, _I64] + [_PI64] * 4 + [_PD] * 2 + [_PI64] * 4 + [_PD] * 2,
                            ctypes.c_int),
    "tsk_format_double": ([ctypes.c_double, ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
    "tsk_save_store_csv": ([ctypes.c_char_p, _I64, _PI64, _PI64] + [_PD] * 8 + [ctypes.c_int], ctypes.c_int),
    "tsk_write_results_csv": ([ctypes.c_char_p, _I64] + [_PI64] * 4 + [_PD] * 2 + [ctypes.c_int],
                              ctypes.c_int),
    "tsk_load_store_csv": ([ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_P), _PI64, _PI64], ctypes.c_int),
    "tsk_csv_columns": ([_P, _PI64, _PI64] + [_PD] * 8, ctypes.c_int),
    "tsk_csv_free": ([_P], None),
    "tsk_pinned_alloc": ([_I64], _P),
    "tsk_pinned_free": ([_P], None),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libtrajseek.so (raises RuntimeError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libtrajseek.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == TSK_OK:
        return
    msg = load().tsk_last_error().decode(errors="replace")
    if rc == TSK_EINVAL:
        from .core import DomainError

        raise DomainError(msg)
    if rc == TSK_EFORMAT:
        from .core import FormatError

        raise FormatError(msg)
    if rc == TSK_ENOMEM:
        raise MemoryError(msg)
    if rc == TSK_ETOOMANY:
        raise TooManyHits(msg)
    raise RuntimeError(f"libtrajseek error {rc}: {msg}")


def device_count() -> int:
    return int(load().tsk_device_count())


_device = int(os.environ.get("TRAJSEEK_DEVICE", "0"))


def set_device(ordinal: int) -> None:
    """Select the CUDA device new device-resident stores are placed on."""
    global _device
    _device = int(ordinal)


def current_device() -> int:
    return _device


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def columns_of(store) -> tuple[Columns, list]:
    """tsk_columns view of a SegmentStore (keeps contiguous copies alive)."""
    keep = []

    def c(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return _ptr(a)

    col = Columns()
    col.n = len(store)
    col.traj = c(store.traj, np.int64)
    col.seg = c(store.seg, np.int64)
    for k in ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te"):
        setattr(col, k, c(getattr(store, k), np.float64))
    return col, keep


class DeviceStore:
    """Owns a tsk_db handle: a store resident in one GPU's HBM.

    A tsk_db is thread-compatible, not thread-safe (its search workspace,
    query records and index are shared by every call on it), so every call
    on the handle holds ``lock``; the engine also holds it across "ensure
    this index, then search" so two threads cannot swap the device index
    under each other."""

    def __init__(self, store, device: int | None = None, source: "DeviceStore | None" = None):
        self.lock = threading.RLock()
        self.device = current_device() if device is None else int(device)
        lib = load()
        h = ctypes.c_void_p()
        if source is not None:  # device-to-device replica (NVLink between peers)
            check(lib.tsk_db_replicate(source.handle, self.device, ctypes.byref(h)))
        else:
            col, keep = columns_of(store)
            check(lib.tsk_db_create(self.device, ctypes.byref(col), ctypes.byref(h)))
            del keep
        self.handle = h
        self.n = len(store)
        self.index_token = None
        # host id columns for the compact result path (kept alive here)
        self._host_ids = (np.ascontiguousarray(store.traj, np.int64), np.ascontiguousarray(store.seg, np.int64))
        check(lib.tsk_db_set_host_ids(h, self._host_ids[0].ctypes.data_as(_PI64),
                                      self._host_ids[1].ctypes.data_as(_PI64)))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            _lib.tsk_db_free(h)
            self.handle = None


class _Owner:
    """Keeps a tsk_result alive while numpy views of its pinned columns live."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        if self.handle is not None and _lib is not None:
            _lib.tsk_result_free(self.handle)
            self.handle = None


def _view(owner, ptr, n, dtype):
    if n == 0 or not ptr:
        return np.empty(0, dtype=dtype)
    nbytes = n * np.dtype(dtype).itemsize
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    buf._owner = owner  # lifetime: array → buffer → owner → tsk_result
    arr = np.frombuffer(buf, dtype=dtype)
    return arr


class Result:
    """Decoded tsk_result: numpy columns (zero-copy over pinned memory)."""

    def __init__(self, handle):
        lib = load()
        self._owner = _Owner(handle)
        n = _I64()
        nb = _I64()
        ms = ctypes.c_double()
        check(lib.tsk_result_info(handle, ctypes.byref(n), ctypes.byref(nb), ctypes.byref(ms)))
        k1 = ctypes.c_double()
        nl = _I64()
        check(lib.tsk_result_timing(handle, ctypes.byref(ms), ctypes.byref(k1), ctypes.byref(nl)))
        self.n, self.nb = int(n.value), int(nb.value)
        self.device_ms, self.k1_ms = float(ms.value), float(k1.value)
        self.launches = int(nl.value)
        ev = _I64()
        check(lib.tsk_result_k1_evals(handle, ctypes.byref(ev)))
        self.k1_evals = int(ev.value)  # pairs K1's FP32 pre-filter evaluated
        pb = np.empty((self.nb, 4), dtype=np.int64)
        check(lib.tsk_result_per_batch(handle, pb.ctypes.data_as(_PI64)))
        self.per_batch = pb  # first, last, overlaps, hits
        ptrs = [ctypes.c_void_p() for _ in range(8)]
        check(lib.tsk_result_columns(handle, *[ctypes.byref(p) for p in ptrs]))
        names = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end",
                 "query_ord", "entry_ord")
        self.cols = {}
        for name, p in zip(names, ptrs):
            dt = np.float64 if name.startswith("t_") else np.int64
            if not p.value:
                self.cols[name] = None if self.n else np.empty(0, dtype=dt)
            else:
                self.cols[name] = _view(self._owner, p.value, self.n, dt)


def search(dev: DeviceStore, queries, lo, hi, first, last, d: float, flags: int) -> Result:
    lib = load()
    col, keep = columns_of(queries)
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    fp = lp = None
    if first is not None:
        first = np.ascontiguousarray(first, dtype=np.int64)
        last = np.ascontiguousarray(last, dtype=np.int64)
        fp, lp = first.ctypes.data_as(_PI64), last.ctypes.data_as(_PI64)
    h = ctypes.c_void_p()
    with dev.lock:
        check(lib.tsk_search(dev.handle, ctypes.byref(col), lo.shape[0], lo.ctypes.data_as(_PI64),
                             hi.ctypes.data_as(_PI64), fp, lp, float(d), flags, ctypes.byref(h)))
    del keep
    return Result(h)


def pair_intervals(rows, cols, d: float, device: int | None = None) -> Result:
    lib = load()
    rc, rk = columns_of(rows)
    cc, ck = columns_of(cols)
    h = ctypes.c_void_p()
    dev = current_device() if device is None else int(device)
    check(lib.tsk_pair_intervals(dev, ctypes.byref(rc), ctypes.byref(cc), float(d), ctypes.byref(h)))
    del rk, ck
    return Result(h)


def sort_by_start(ts: np.ndarray, device: int | None = None) -> np.ndarray:
    lib = load()
    ts = np.ascontiguousarray(ts, dtype=np.float64)
    perm = np.empty(ts.shape[0], dtype=np.int64)
    dev = current_device() if device is None else int(device)
    check(lib.tsk_sort_by_start(dev, ts.shape[0], ts.ctypes.data_as(_PD), perm.ctypes.data_as(_PI64)))
    return perm


def index_build(dev: DeviceStore, m: int, rule: int):
    lib = load()
    n_ne = _I64()
    hdr = (ctypes.c_double * 3)()
    with dev.lock:
        check(lib.tsk_index_build(dev.handle, int(m), int(rule), ctypes.byref(n_ne), hdr))
        k = int(n_ne.value)
        ne_start = np.empty(k, np.float64)
        ne_end = np.empty(k, np.float64)
        ne_first = np.empty(k, np.int64)
        ne_last = np.empty(k, np.int64)
        ne_bin = np.empty(k, np.int64)
        check(lib.tsk_index_copy(dev.handle, ne_start.ctypes.data_as(_PD), ne_end.ctypes.data_as(_PD),
                                 ne_first.ctypes.data_as(_PI64), ne_last.ctypes.data_as(_PI64),
                                 ne_bin.ctypes.data_as(_PI64)))
    return (hdr[0], hdr[1], hdr[2]), ne_start, ne_end, ne_first, ne_last, ne_bin


def candidate_ranges(dev: DeviceStore, begin: np.ndarray, end: np.ndarray):
    lib = load()
    begin = np.ascontiguousarray(begin, np.float64)
    end = np.ascontiguousarray(end, np.float64)
    k = begin.shape[0]
    first = np.empty(k, np.int64)
    last = np.empty(k, np.int64)
    with dev.lock:
        check(lib.tsk_candidate_ranges(dev.handle, k, begin.ctypes.data_as(_PD), end.ctypes.data_as(_PD),
                                       first.ctypes.data_as(_PI64), last.ctypes.data_as(_PI64)))
    return first, last


def probe_fp64(device: int | None = None) -> dict:
    """Measured FP64 pipe rates (ops/s) of a device (tsk_probe_fp64)."""
    lib = load()
    a, m, f = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    dev = current_device() if device is None else int(device)
    check(lib.tsk_probe_fp64(dev, ctypes.byref(a), ctypes.byref(m), ctypes.byref(f)))
    return {"dadd_per_s": a.value, "dmul_per_s": m.value, "dfma_per_s": f.value}


def probe_fp32(device: int | None = None) -> float:
    """Measured FP32 FFMA rate (ops/s) of a device (tsk_probe_fp32)."""
    lib = load()
    f = ctypes.c_double()
    dev = current_device() if device is None else int(device)
    check(lib.tsk_probe_fp32(dev, ctypes.byref(f)))
    return f.value


K1_STAT_NAMES = ("subtiles", "box_tests", "box_survivors", "subtiles_with_survivors", "prefilter_flags",
                 "sep_survivors", "exact_flushes", "items")


def k1_stats(device: int | None = None, reset: bool = False) -> dict:
    """K1's development counters (all zero unless built with -DTSK_K1_STATS)."""
    lib = load()
    out = (ctypes.c_ulonglong * 8)()
    dev = current_device() if device is None else int(device)
    check(lib.tsk_k1_stats(dev, out, 8, 1 if reset else 0))
    return dict(zip(K1_STAT_NAMES, (int(v) for v in out)))


class _Pinned:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.tsk_pinned_free(self.ptr)
            self.ptr = None


def pinned_empty(n: int, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (freed with the array)."""
    dt = np.dtype(dtype)
    nbytes = max(1, n) * dt.itemsize
    ptr = load().tsk_pinned_alloc(nbytes)
    if not ptr:
        raise MemoryError("tsk_pinned_alloc failed")
    owner = _Pinned(ptr)
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    buf._owner = owner
    return np.frombuffer(buf, dtype=dt)[:n]


def pinned_copy(a: np.ndarray) -> np.ndarray:
    out = pinned_empty(a.shape[0], a.dtype)
    out[...] = a
    return out


def plan_native(kind: str, ts, te, index, *, num_batches=0, min_size=0, max_size=0, bound=0):
    """Run a native planner; returns (lo, hi, first, last, end) arrays."""
    lib = load()
    ts = np.ascontiguousarray(ts, np.float64)
    te = np.ascontiguousarray(te, np.float64)
    nq = ts.shape[0]
    ne = [np.ascontiguousarray(index._ne_start, np.float64), np.ascontiguousarray(index._ne_end, np.float64),
          np.ascontiguousarray(index._ne_first, np.int64), np.ascontiguousarray(index._ne_last, np.int64)]
    out = [np.empty(nq, np.int64) for _ in range(4)] + [np.empty(nq, np.float64)]
    nb = _I64()
    common = [nq, ts.ctypes.data_as(_PD), te.ctypes.data_as(_PD), ne[0].shape[0],
              ne[0].ctypes.data_as(_PD), ne[1].ctypes.data_as(_PD), ne[2].ctypes.data_as(_PI64),
              ne[3].ctypes.data_as(_PI64)]
    tail = [ctypes.byref(nb)] + [o.ctypes.data_as(_PI64) for o in out[:4]] + [out[4].ctypes.data_as(_PD)]
    if kind == "fixed":
        check(lib.tsk_plan_setsplit(*common, 0, num_batches, 0, 0, *tail))
    elif kind == "minmax":
        check(lib.tsk_plan_setsplit(*common, 1, 0, min_size, max_size, *tail))
    elif kind in ("greedy_min", "greedy_max"):
        check(lib.tsk_plan_greedy(*common, 0 if kind == "greedy_min" else 1, bound, *tail))
    else:
        raise ValueError(kind)
    k = int(nb.value)
    return tuple(o[:k] for o in out)


def canonical_order(cols: dict, device: int | None = None) -> dict:
    """Canonically ordered copies of the six result columns, sorted on the GPU."""
    lib = load()
    names = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")
    src = [np.ascontiguousarray(cols[k], np.float64 if k.startswith("t_") else np.int64) for k in names]
    n = src[0].shape[0]
    out = [np.empty(n, dtype=a.dtype) for a in src]
    ptr = lambda a: a.ctypes.data_as(_PD if a.dtype == np.float64 else _PI64)  # noqa: E731
    dev = current_device() if device is None else int(device)
    check(lib.tsk_canonical_order(dev, n, *[ptr(a) for a in src], *[ptr(a) for a in out]))
    return dict(zip(names, out))


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def py_repr(x: float) -> str:
    """repr(float) computed by the native formatter (tests)."""
    b = ctypes.create_string_buffer(48)
    n = load().tsk_format_double(float(x), b, 48)
    return b.value[:n].decode()


def save_store_csv(store, path: str) -> None:
    cols = [np.ascontiguousarray(getattr(store, k), np.int64) for k in ("traj", "seg")]
    cols += [np.ascontiguousarray(getattr(store, k), np.float64)
             for k in ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")]
    check(load().tsk_save_store_csv(os.fsencode(path), len(store), cols[0].ctypes.data_as(_PI64),
                                    cols[1].ctypes.data_as(_PI64),
                                    *[c.ctypes.data_as(_PD) for c in cols[2:]], _threads()))


def write_results_csv(cols: dict, path: str) -> None:
    names = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")
    arr = [np.ascontiguousarray(cols[k], np.float64 if k.startswith("t_") else np.int64) for k in names]
    check(load().tsk_write_results_csv(os.fsencode(path), arr[0].shape[0],
                                       *[a.ctypes.data_as(_PI64) for a in arr[:4]],
                                       *[a.ctypes.data_as(_PD) for a in arr[4:]], _threads()))


def load_store_csv(path: str, strict: bool = False) -> dict:
    """Columns of a segment CSV in file order (raises FormatError)."""
    lib = load()
    h = ctypes.c_void_p()
    n = _I64()
    bad = _I64()
    check(lib.tsk_load_store_csv(os.fsencode(path), 1 if strict else 0, ctypes.byref(h), ctypes.byref(n),
                                 ctypes.byref(bad)))
    try:
        k = int(n.value)
        out = {"traj": np.empty(k, np.int64), "seg": np.empty(k, np.int64)}
        for c in ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te"):
            out[c] = np.empty(k, np.float64)
        check(lib.tsk_csv_columns(h, out["traj"].ctypes.data_as(_PI64), out["seg"].ctypes.data_as(_PI64),
                                  *[out[c].ctypes.data_as(_PD) for c in ("xs", "ys", "zs", "ts", "xe",
                                                                         "ye", "ze", "te")]))
        return out
    finally:
        lib.tsk_csv_free(h)
