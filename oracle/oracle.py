"""ctypes wrapper of the CPU oracle (oracle/exactz_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2604_01397_b200/) never imports this module.

Argument marshalling only; every computation happens in the C file, whose
functions cite the paper passages they follow.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "exactz_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

OK, EINVAL, EBOUND, ESTUCK, ENOMEM = 0, 2, 3, 4, 8
NO_C2, NO_C3, REFORM = 1, 2, 16
CLS_REGULAR, CLS_MIN, CLS_MAX, CLS_SADDLE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, IEEE binary32, no contraction/fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        i64, i32, u32, f32 = C.c_int64, C.c_int, C.c_uint32, C.c_float
        L.oracle_ru_sub.argtypes = [f32, f32]; L.oracle_ru_sub.restype = f32
        L.oracle_rd_add.argtypes = [f32, f32]; L.oracle_rd_add.restype = f32
        L.oracle_offsets.argtypes = [P]; L.oracle_offsets.restype = i32
        L.oracle_link_adjacent.argtypes = [i32, i32]; L.oracle_link_adjacent.restype = i32
        L.oracle_mask_components.argtypes = [u32]; L.oracle_mask_components.restype = i32
        L.oracle_neighbors.argtypes = [i64, i64, i64, i64, P]; L.oracle_neighbors.restype = i32
        L.oracle_sos_less.argtypes = [P, i64, i64]; L.oracle_sos_less.restype = i32
        L.oracle_classify.argtypes = [P, i64, i64, i64, P, P, P]; L.oracle_classify.restype = i32
        L.oracle_steepest.argtypes = [P, i64, i64, i64, P, P]; L.oracle_steepest.restype = i32
        L.oracle_labels.argtypes = [P, i64, i64, i64, P, P]; L.oracle_labels.restype = i32
        L.oracle_reference.argtypes = [P, i64, i64, i64, P, P, P, P, P, P]
        L.oracle_reference.restype = i32
        L.oracle_check.argtypes = [P, P, i64, i64, i64, u32, P, P]; L.oracle_check.restype = i32
        L.oracle_validate.argtypes = [P, P, i64, f32, i32]; L.oracle_validate.restype = i32
        L.oracle_correct.argtypes = [P, P, i64, i64, i64, f32, i32, u32, u32, P, P, P, P, P, P,
                                     i64, P]
        L.oracle_correct.restype = i32
        L.oracle_extremum_graph.argtypes = [P, i64, i64, i64, i32, P, i64]
        L.oracle_extremum_graph.restype = i64
        L.oracle_merge_tree.argtypes = [P, i64, i64, i64, i32, P, P, P]
        L.oracle_merge_tree.restype = i32
        L.oracle_vulnerability.argtypes = [P, P, i64, i64, i64, f32, P]
        L.oracle_vulnerability.restype = i32
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims(h: np.ndarray, dims):
    if dims is None:
        shp = h.shape
        # array shape (nz, ny, nx) / (ny, nx) / (nx,), x fastest
        d = list(reversed(shp)) + [1] * (3 - len(shp))
        return int(d[0]), int(d[1]), int(d[2])
    return tuple(int(x) for x in dims)


def ru_sub(a: float, b: float) -> np.float32:
    return np.float32(lib().oracle_ru_sub(float(np.float32(a)), float(np.float32(b))))


def rd_add(a: float, b: float) -> np.float32:
    return np.float32(lib().oracle_rd_add(float(np.float32(a)), float(np.float32(b))))


def offsets() -> np.ndarray:
    out = np.zeros(42, np.int32)
    lib().oracle_offsets(_p(out))
    return out.reshape(14, 3)


def link_adjacent(a: int, b: int) -> bool:
    return bool(lib().oracle_link_adjacent(a, b))


def mask_components(mask: int) -> int:
    return int(lib().oracle_mask_components(mask))


def neighbors(dims, v: int) -> list[int]:
    out = np.zeros(14, np.int64)
    n = lib().oracle_neighbors(*dims, v, _p(out))
    if n < 0:
        raise IndexError(v)
    return [int(x) for x in out[:n]]


def sos_less(h, u: int, v: int) -> bool:
    h = _f32(h).ravel()
    return bool(lib().oracle_sos_less(_p(h), u, v))


def classify(h, dims=None):
    h = _f32(h)
    nx, ny, nz = _dims(h, dims)
    V = nx * ny * nz
    nlc, nuc, cls = (np.zeros(V, np.uint8) for _ in range(3))
    assert lib().oracle_classify(_p(h), nx, ny, nz, _p(nlc), _p(nuc), _p(cls)) == OK
    return nlc, nuc, cls


def steepest(h, dims=None):
    h = _f32(h)
    nx, ny, nz = _dims(h, dims)
    V = nx * ny * nz
    up, dn = np.zeros(V, np.int32), np.zeros(V, np.int32)
    assert lib().oracle_steepest(_p(h), nx, ny, nz, _p(up), _p(dn)) == OK
    return up, dn


def labels(h, dims=None):
    h = _f32(h)
    nx, ny, nz = _dims(h, dims)
    V = nx * ny * nz
    ld, lu = np.zeros(V, np.int32), np.zeros(V, np.int32)
    assert lib().oracle_labels(_p(h), nx, ny, nz, _p(ld), _p(lu)) == OK
    return ld, lu


def reference(f, dims=None):
    f = _f32(f)
    nx, ny, nz = _dims(f, dims)
    V = nx * ny * nz
    bufs = [np.zeros(max(V, 1), np.int32) for _ in range(5)]
    n = np.zeros(3, np.int64)
    assert lib().oracle_reference(_p(f), nx, ny, nz, *[_p(b) for b in bufs], _p(n)) == OK
    S, J, P, m1, M1 = bufs
    nS, nJ, nP = (int(x) for x in n)
    return dict(S=S[:nS].copy(), J=J[:nJ].copy(), P=P[:nP].copy(), m1=m1[:nJ].copy(),
                M1=M1[:nP].copy())


def check(f, g, dims=None, flags: int = 0):
    """One CheckConstraints pass: (marks uint8[V], counts {V_t,n1..n6})."""
    f, g = _f32(f), _f32(g)
    nx, ny, nz = _dims(f, dims)
    V = nx * ny * nz
    mark = np.zeros(V, np.uint8)
    cnt = np.zeros(7, np.int64)
    assert lib().oracle_check(_p(f), _p(g), nx, ny, nz, flags, _p(mark), _p(cnt)) == OK
    return mark, cnt


def validate(f, ghat, xi: float, N: int = 5) -> int:
    f, ghat = _f32(f), _f32(ghat)
    return int(lib().oracle_validate(_p(f), _p(ghat), f.size, float(np.float32(xi)), N))


@dataclass
class Result:
    status: int
    out: np.ndarray
    counts: np.ndarray
    label_min: np.ndarray
    label_max: np.ndarray
    iters: int
    stats: np.ndarray = field(repr=False)  # rows {V_t, applied, n1..n6}


def correct(f, ghat, xi: float, N: int = 5, dims=None, flags: int = 0, max_iters: int = 0,
            stats_cap: int = 100000) -> Result:
    f, ghat = _f32(f), _f32(ghat)
    nx, ny, nz = _dims(f, dims)
    V = nx * ny * nz
    out = np.empty(V, np.float32)
    cnt = np.zeros(V, np.uint8)
    lmin, lmax = np.zeros(V, np.int32), np.zeros(V, np.int32)
    iters = C.c_uint32(0)
    stats = np.zeros((stats_cap, 8), np.int64)
    rows = C.c_int64(0)
    st = lib().oracle_correct(_p(f), _p(ghat), nx, ny, nz, float(np.float32(xi)), N, flags,
                              max_iters, _p(out), _p(cnt), _p(lmin), _p(lmax), C.byref(iters),
                              _p(stats), stats_cap, C.byref(rows))
    r = min(rows.value, stats_cap)
    return Result(st, out, cnt, lmin, lmax, iters.value, stats[:r].copy())


def extremum_graph(h, dims=None, split: bool = False) -> set:
    h = _f32(h)
    nx, ny, nz = _dims(h, dims)
    V = nx * ny * nz
    cap = 14 * V + 1
    e = np.zeros(2 * cap, np.int32)
    n = lib().oracle_extremum_graph(_p(h), nx, ny, nz, int(split), _p(e), cap)
    assert 0 <= n <= cap
    return {(int(a), int(b)) for a, b in e[:2 * n].reshape(-1, 2)}


def merge_tree(h, dims=None, split: bool = False):
    """(tree arcs, elder pairs) of the join (split=False) or split tree."""
    h = _f32(h)
    nx, ny, nz = _dims(h, dims)
    V = nx * ny * nz
    arcs = np.zeros(2 * V + 2, np.int32)
    pairs = np.zeros(2 * V + 2, np.int32)
    n = np.zeros(2, np.int64)
    assert lib().oracle_merge_tree(_p(h), nx, ny, nz, int(split), _p(arcs), _p(pairs), _p(n)) == OK
    A = {(int(a), int(b)) for a, b in arcs[:2 * n[0]].reshape(-1, 2)}
    Pp = {(int(a), int(b)) for a, b in pairs[:2 * n[1]].reshape(-1, 2)}
    return A, Pp


def vulnerability(f, ghat, xi: float, dims=None) -> dict:
    f, ghat = _f32(f), _f32(ghat)
    nx, ny, nz = _dims(f, dims)
    out = np.zeros(5, np.int64)
    assert lib().oracle_vulnerability(_p(f), _p(ghat), nx, ny, nz, float(np.float32(xi)),
                                      _p(out)) == OK
    return dict(D_max=int(out[0]), GV=int(out[1]), GS=int(out[2]), GR=int(out[3]),
                seeds=int(out[4]))
