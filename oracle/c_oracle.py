"""ctypes loader for the C oracle (oracle/pair_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's baseline arm use this.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_D = ctypes.c_double
_I64 = ctypes.c_int64
_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "pair_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_pair.argtypes = [_PD, _PD, _D, _PD, _PD, ctypes.POINTER(ctypes.c_int)]
        L.orc_pair.restype = ctypes.c_int
        L.orc_floor_divide.argtypes = [_D, _D]
        L.orc_floor_divide.restype = _D
        L.orc_floor_divide_many.argtypes = [_I64, _PD, _D, _PD]
        L.orc_brute_force.argtypes = [
            _I64, ctypes.POINTER(_PD), _I64, ctypes.POINTER(_PD), _D, ctypes.c_int,
            ctypes.POINTER(_PI64), ctypes.POINTER(_PI64), ctypes.POINTER(_PD), ctypes.POINTER(_PD),
            _PI64, _PI64,
        ]
        L.orc_brute_force.restype = _I64
        L.orc_search_spans.argtypes = [
            ctypes.POINTER(_PD), ctypes.POINTER(_PD), _I64, _PI64, _PI64, _PI64, _PI64, _D,
            ctypes.c_int, _I64, _PI64, ctypes.POINTER(_PI64), ctypes.POINTER(_PI64),
            ctypes.POINTER(_PD), ctypes.POINTER(_PD),
        ]
        L.orc_search_spans.restype = _I64
        L.orc_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


_FLOATS = ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")


def pair(a, b, d):
    """a, b: 8-tuples (xs ys zs ts xe ye ze te) → (begin, end) or None."""
    A = (ctypes.c_double * 8)(*a)
    B = (ctypes.c_double * 8)(*b)
    bg, en = ctypes.c_double(), ctypes.c_double()
    tm = ctypes.c_int()
    if lib().orc_pair(A, B, d, ctypes.byref(bg), ctypes.byref(en), ctypes.byref(tm)):
        return bg.value, en.value
    return None


def floor_divide(a: np.ndarray, b: float) -> np.ndarray:
    a = np.ascontiguousarray(a, np.float64)
    out = np.empty_like(a)
    lib().orc_floor_divide_many(a.shape[0], a.ctypes.data_as(_PD), b, out.ctypes.data_as(_PD))
    return out


def _colptrs(store):
    cols = [np.ascontiguousarray(store[k], np.float64) for k in _FLOATS]
    arr = (_PD * 8)(*[c.ctypes.data_as(_PD) for c in cols])
    return arr, cols


def brute_force(store, queries, d, threads=None):
    """Query-major brute force over dict stores → result dict like oracle.brute_force."""
    threads = threads or max(1, os.cpu_count() or 1)
    ep, keep_e = _colptrs(store)
    qp, keep_q = _colptrs(queries)
    qo, eo = _PI64(), _PI64()
    tb, te = _PD(), _PD()
    tm, sm = _I64(), _I64()
    ne = store["ts"].shape[0]
    nq = queries["ts"].shape[0]
    n = lib().orc_brute_force(ne, ep, nq, qp, d, threads, ctypes.byref(qo), ctypes.byref(eo),
                              ctypes.byref(tb), ctypes.byref(te), ctypes.byref(tm), ctypes.byref(sm))
    q_ord = np.ctypeslib.as_array(qo, (n,)).copy() if n else np.empty(0, np.int64)
    e_ord = np.ctypeslib.as_array(eo, (n,)).copy() if n else np.empty(0, np.int64)
    t_b = np.ctypeslib.as_array(tb, (n,)).copy() if n else np.empty(0)
    t_e = np.ctypeslib.as_array(te, (n,)).copy() if n else np.empty(0)
    for p in (qo, eo, tb, te):
        lib().orc_free(ctypes.cast(p, ctypes.c_void_p))
    del keep_e, keep_q
    return {
        "query_traj": queries["traj"][q_ord], "query_seg": queries["seg"][q_ord],
        "entry_traj": store["traj"][e_ord], "entry_seg": store["seg"][e_ord],
        "t_begin": t_b, "t_end": t_e,
    }, int(tm.value), int(sm.value)


def search_spans(store, queries, lo, hi, first, last, d, threads=None, chunk_pairs=1 << 20):
    """Engine over explicit spans (orc_search_spans): batch b = queries
    lo[b]..hi[b] against entries first[b]..last[b] (first < 0: none).

    Returns (result dict in the reference engine's order, per-batch int64
    array (nb, 3) = hits, temporal misses, spatial misses)."""
    threads = threads or max(1, os.cpu_count() or 1)
    ep, keep_e = _colptrs(store)
    qp, keep_q = _colptrs(queries)
    a = [np.ascontiguousarray(x, np.int64) for x in (lo, hi, first, last)]
    nb = a[0].shape[0]
    pb = np.zeros((nb, 3), np.int64)
    qo, eo = _PI64(), _PI64()
    tb, te = _PD(), _PD()
    n = lib().orc_search_spans(ep, qp, nb, *[x.ctypes.data_as(_PI64) for x in a], float(d), threads,
                               int(chunk_pairs), pb.ctypes.data_as(_PI64), ctypes.byref(qo),
                               ctypes.byref(eo), ctypes.byref(tb), ctypes.byref(te))
    q_ord = np.ctypeslib.as_array(qo, (n,)).copy() if n else np.empty(0, np.int64)
    e_ord = np.ctypeslib.as_array(eo, (n,)).copy() if n else np.empty(0, np.int64)
    t_b = np.ctypeslib.as_array(tb, (n,)).copy() if n else np.empty(0)
    t_e = np.ctypeslib.as_array(te, (n,)).copy() if n else np.empty(0)
    for p in (qo, eo, tb, te):
        lib().orc_free(ctypes.cast(p, ctypes.c_void_p))
    del keep_e, keep_q
    return {
        "query_traj": queries["traj"][q_ord], "query_seg": queries["seg"][q_ord],
        "entry_traj": store["traj"][e_ord], "entry_seg": store["seg"][e_ord],
        "t_begin": t_b, "t_end": t_e,
    }, pb


def plan_spans(store, ix, queries, lo, hi):
    """Candidate spans of batches lo..hi the way run_search derives them
    (engine.py:177-182): extent [ts[lo], max te[lo..hi]] → candidate_range
    on the numpy oracle's index (pinned to the reference's goldens)."""
    from . import oracle as orc

    first = np.full(len(lo), -1, np.int64)
    last = np.full(len(lo), -1, np.int64)
    for k, (a, b) in enumerate(zip(lo, hi)):
        fl = orc.cand_range(ix, float(queries["ts"][a]), float(queries["te"][a:b + 1].max()))
        if fl is not None:
            first[k], last[k] = fl
    return first, last
