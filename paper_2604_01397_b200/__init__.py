"""paper_2604_01397_b200 — B200 (sm_100a) EXaCTz topology-correction hot path.

Thin Python binding of the C ABI in include/exactz.h (libexactz.so, built
in-tree by _build.py).  Argument marshalling only: every step of the path runs
in the CUDA kernels of csrc/.  PyTorch is used for device memory and streams.
There is no CPU fallback: importing this package without the built library
raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libexactz.so")

OK, EINVAL, EBOUND, ESTUCK, EUNSUPPORTED, ECUDA, ENCCL, ENOMEM = 0, 2, 3, 4, 5, 6, 7, 8
NO_C2, NO_C3, PROFILE, NO_TRACK, REFORMULATED = 0x1, 0x2, 0x4, 0x8, 0x10
KERNEL_CLASSES = ("validate", "reference", "stencil", "saddle_order", "events", "edit", "labels",
                  "stencil_sparse")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g;"
                      " g.build()'` (nvcc, sm_100a). There is no CPU fallback.")


class IterStats(C.Structure):
    _fields_ = [("violations", C.c_uint64), ("applied", C.c_uint64), ("n", C.c_uint64 * 6),
                ("walk_steps", C.c_uint64), ("evaluated", C.c_uint64), ("links", C.c_uint64),
                ("ms", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("rows", C.POINTER(IterStats)), ("cap", C.c_uint32), ("nrows", C.c_uint32),
                ("ms_setup", C.c_double), ("ms_loop", C.c_double),
                ("kernel_ms", C.c_double * 8), ("kernel_launches", C.c_uint64 * 8),
                ("kernel_bytes", C.c_uint64 * 8), ("n_saddles", C.c_uint64),
                ("n_join", C.c_uint64), ("n_split", C.c_uint64)]


class Opts(C.Structure):
    _fields_ = [("N", C.c_uint32), ("max_iters", C.c_uint32), ("flags", C.c_uint32),
                ("edit_counts", C.c_void_p), ("label_min", C.c_void_p),
                ("label_max", C.c_void_p), ("stats", C.POINTER(Stats))]


import torch  # noqa: E402,F401  (first: libtorch_cuda and libexactz share torch's libnccl.so.2)

_lib = C.CDLL(LIB_PATH)
_P, _i64p = C.c_void_p, C.POINTER(C.c_int64)
_lib.exactz_correct.argtypes = [_P, _P, _i64p, C.c_float, _P, C.POINTER(C.c_uint32),
                                C.POINTER(Opts), _P]
_lib.exactz_correct.restype = C.c_int
_lib.exactz_correct_host.argtypes = _lib.exactz_correct.argtypes
_lib.exactz_correct_host.restype = C.c_int
_lib.exactz_check.argtypes = [_P, _P, _i64p, C.c_float, C.POINTER(C.c_uint64),
                              C.POINTER(IterStats), C.c_uint32, _P]
_lib.exactz_check.restype = C.c_int
_lib.exactz_vulnerability.argtypes = [_P, _P, _i64p, C.c_float, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_uint32), _P]
_lib.exactz_vulnerability.restype = C.c_int
_lib.exactz_edit_log.argtypes = [_P, _P, _P, _i64p, C.c_float, C.c_uint32, C.c_int, _P,
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), _P]
_lib.exactz_edit_log.restype = C.c_int
_lib.exactz_edit_log_apply.argtypes = [_P, C.c_uint64, _P, _P, C.c_int64, _P]
_lib.exactz_edit_log_apply.restype = C.c_int
_lib.exactz_eps_from_relative.argtypes = [_P, C.c_int64, C.c_double, C.POINTER(C.c_float), _P]
_lib.exactz_eps_from_relative.restype = C.c_int
_lib.exactz_strerror.argtypes = [C.c_int]
_lib.exactz_strerror.restype = C.c_char_p
_lib.exactz_last_error.restype = C.c_char_p
_lib.exactz_version.restype = C.c_char_p
_lib.exactz_kernel_launches.restype = C.c_uint64
_lib.exactz_nccl_unique_id.argtypes = [_P]
_lib.exactz_nccl_unique_id.restype = C.c_int
_lib.exactz_comm_init.argtypes = [_P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
_lib.exactz_comm_init.restype = C.c_int
_lib.exactz_comm_destroy.argtypes = [_P]
_lib.exactz_comm_destroy.restype = C.c_int
_lib.exactz_correct_sharded.argtypes = [_P, _P, _P, _i64p, C.c_int64, C.c_int64, C.c_float, _P,
                                        C.POINTER(C.c_uint32), C.POINTER(Opts), _P]
_lib.exactz_correct_sharded.restype = C.c_int
_lib.exactz_correct_slabs.argtypes = [_P, _P, _i64p, C.c_float, C.c_int, _P,
                                      C.POINTER(C.c_uint32), C.POINTER(Opts), _P]
_lib.exactz_correct_slabs.restype = C.c_int
_lib.exactz_slab_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]
_lib.exactz_slab_range.restype = C.c_int


def lib() -> C.CDLL:
    return _lib


def version() -> str:
    return _lib.exactz_version().decode()


def kernel_launches() -> int:
    """This library's own kernel launches so far in this process."""
    return int(_lib.exactz_kernel_launches())


def last_error() -> str:
    return _lib.exactz_last_error().decode()


class ExactzError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {_lib.exactz_strerror(status).decode()} ({last_error()})")


@dataclass
class CorrectResult:
    status: int            # OK or ESTUCK
    iters: int             # edit rounds
    stats: list            # per detection pass: (V_t, applied, n1..n6)
    ms_setup: float
    ms_loop: float
    kernels: dict = None   # PROFILE: class -> (ms, launches, algorithmic bytes)


def _dims(t) -> C.Array:
    shp = list(t.shape)
    d = list(reversed(shp)) + [1] * (3 - len(shp))
    return (C.c_int64 * 3)(*[int(x) for x in d])


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _opts(N, max_iters, flags, edit_counts, label_min, label_max, stats_cap):
    o = Opts()
    o.N, o.max_iters, o.flags = N, max_iters, flags
    o.edit_counts = None if edit_counts is None else edit_counts.data_ptr()
    o.label_min = None if label_min is None else label_min.data_ptr()
    o.label_max = None if label_max is None else label_max.data_ptr()
    st = Stats()
    rows = (IterStats * max(stats_cap, 1))()
    st.rows = C.cast(rows, C.POINTER(IterStats)) if stats_cap else None
    st.cap = stats_cap
    o.stats = C.pointer(st)
    return o, st, rows


def _result(status, iters, st, rows):
    n = min(st.nrows, st.cap)
    table = [(r.violations, r.applied, *list(r.n)) for r in rows[:n]] if st.cap else []
    walks = [int(r.walk_steps) for r in rows[:n]] if st.cap else []
    kern = {KERNEL_CLASSES[k]: (st.kernel_ms[k], int(st.kernel_launches[k]),
                                int(st.kernel_bytes[k])) for k in range(8)}
    res = CorrectResult(status, iters.value, table, st.ms_setup, st.ms_loop, kern)
    res.walk_steps = walks
    res.pass_ms = [float(r.ms) for r in rows[:n]] if st.cap else []
    res.pass_evaluated = [int(r.evaluated) for r in rows[:n]] if st.cap else []
    res.pass_links = [int(r.links) for r in rows[:n]] if st.cap else []
    res.n_saddles, res.n_join, res.n_split = int(st.n_saddles), int(st.n_join), int(st.n_split)
    return res


def exactz_correct(f, g_in, eps: float, out=None, *, N: int = 5, max_iters: int = 0,
                   flags: int = 0, edit_counts=None, label_min=None, label_max=None,
                   stats_cap: int = 0, stream=None) -> CorrectResult:
    """Alg. 1 on device tensors (float32, contiguous, shape (nz,ny,nx)/(ny,nx)/(nx,)).

    `out` (default: a new tensor) receives the corrected field; it may alias
    g_in.  edit_counts (uint8), label_min/label_max (int32) are optional
    device outputs.  Raises ExactzError unless the status is OK or ESTUCK."""
    import torch
    for t in (f, g_in):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("f and g_in must be contiguous float32 CUDA tensors")
    if out is None:
        out = torch.empty_like(g_in)
    o, st, rows = _opts(N, max_iters, flags, edit_counts, label_min, label_max, stats_cap)
    iters = C.c_uint32(0)
    s = _lib.exactz_correct(_ptr(f), _ptr(g_in), _dims(f), float(eps), _ptr(out), C.byref(iters),
                            C.byref(o), _stream(stream))
    if s not in (OK, ESTUCK):
        raise ExactzError(s, "exactz_correct")
    res = _result(s, iters, st, rows)
    res.out = out
    return res


def exactz_correct_host(f, g_in, eps: float, out=None, *, N: int = 5, max_iters: int = 0,
                        flags: int = 0, edit_counts=None, label_min=None, label_max=None,
                        stats_cap: int = 0, stream=None) -> CorrectResult:
    """Alg. 1 on HOST tensors (CPU, float32, contiguous; pinned is fastest):
    the host<->device copies happen inside the C call."""
    import torch
    for t in (f, g_in):
        if t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
            raise ValueError("f and g_in must be contiguous float32 CPU tensors")
    if out is None:
        # pinned like g_in: a D2H copy into pageable memory blocks the host and
        # cannot overlap the late passes
        out = torch.empty(g_in.shape, dtype=torch.float32, pin_memory=g_in.is_pinned())
    V = g_in.numel()
    if f.numel() != V:
        raise ValueError("f and g_in differ in size")
    for name, t, dt in (("out", out, torch.float32), ("edit_counts", edit_counts, torch.uint8),
                        ("label_min", label_min, torch.int32),
                        ("label_max", label_max, torch.int32)):
        if t is not None and (t.is_cuda or t.dtype != dt or not t.is_contiguous()
                              or t.numel() != V):
            raise ValueError(f"{name} must be a contiguous {dt} CPU tensor of {V} elements")
    o, st, rows = _opts(N, max_iters, flags, edit_counts, label_min, label_max, stats_cap)
    iters = C.c_uint32(0)
    s = _lib.exactz_correct_host(_ptr(f), _ptr(g_in), _dims(f), float(eps), _ptr(out),
                                 C.byref(iters), C.byref(o), _stream(stream))
    if s not in (OK, ESTUCK):
        raise ExactzError(s, "exactz_correct_host")
    res = _result(s, iters, st, rows)
    res.out = out
    return res


def exactz_check(f, g, eps: float, flags: int = 0, stream=None):
    """One CheckConstraints pass: (V_t, (n1..n6))."""
    v = C.c_uint64(0)
    row = IterStats()
    s = _lib.exactz_check(_ptr(f), _ptr(g), _dims(f), float(eps), C.byref(v), C.byref(row),
                          flags, _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_check")
    return v.value, tuple(row.n)


def exactz_vulnerability(f, ghat, eps: float, stream=None) -> dict:
    """Theorem 1 bound: D_max, the sizes of the vulnerability
    graphs G_V, G_S, G_R, the number of seed edges and the relaxation sweeps."""
    out = (C.c_int64 * 5)()
    sw = C.c_uint32(0)
    s = _lib.exactz_vulnerability(_ptr(f), _ptr(ghat), _dims(f), float(eps), out, C.byref(sw),
                                  _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_vulnerability")
    return dict(D_max=int(out[0]), GV=int(out[1]), GS=int(out[2]), GR=int(out[3]),
                seeds=int(out[4]), sweeps=int(sw.value))


def exactz_edit_log(g_in, out, edit_counts, eps: float, N: int = 5, level: int = 0,
                    stream=None):
    """The EXCE edit log of a correction (bytes, entries); level > 0: zstd."""
    n = C.c_uint64(0)
    ne = C.c_uint64(0)
    d = _dims(g_in)
    s = _lib.exactz_edit_log(_ptr(g_in), _ptr(out), _ptr(edit_counts), d, float(eps), N, level,
                             None, C.byref(n), C.byref(ne), _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_edit_log")
    buf = (C.c_uint8 * max(n.value, 1))()
    s = _lib.exactz_edit_log(_ptr(g_in), _ptr(out), _ptr(edit_counts), d, float(eps), N, level,
                             buf, C.byref(n), C.byref(ne), _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_edit_log")
    return C.string_at(buf, n.value), ne.value


def exactz_edit_log_apply(log: bytes, g_in, out=None, stream=None):
    """g_in with the EXCE log applied (a new device tensor unless out)."""
    import torch
    if out is None:
        out = torch.empty_like(g_in)
    if out.numel() != g_in.numel():
        raise ValueError("out and g_in differ in size")
    b = (C.c_uint8 * len(log)).from_buffer_copy(log)
    s = _lib.exactz_edit_log_apply(b, len(log), _ptr(g_in), _ptr(out), g_in.numel(),
                                   _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_edit_log_apply")
    return out


def exactz_eps_from_relative(f, rel: float, stream=None) -> float:
    e = C.c_float(0)
    s = _lib.exactz_eps_from_relative(_ptr(f), f.numel(), float(rel), C.byref(e), _stream(stream))
    if s != OK:
        raise ExactzError(s, "exactz_eps_from_relative")
    return e.value


def status_of(fn, *a, **kw) -> int:
    """Call fn and return its status code instead of raising (tests)."""
    try:
        r = fn(*a, **kw)
        return r.status if isinstance(r, CorrectResult) else OK
    except ExactzError as e:
        return e.status


# ----------------------------------------------------------------- sharded path
def exactz_slab_range(nz: int, nranks: int, rank: int):
    """(z_begin, z_count) of rank's z-slab (the C ABI's split)."""
    a, b = C.c_int64(0), C.c_int64(0)
    s = _lib.exactz_slab_range(nz, nranks, rank, C.byref(a), C.byref(b))
    if s != OK:
        raise ExactzError(s, "exactz_slab_range")
    return a.value, b.value


def exactz_correct_slabs(f, g_in, eps: float, nslabs: int, out=None, *, N: int = 5,
                         max_iters: int = 0, flags: int = 0, edit_counts=None, label_min=None,
                         label_max=None, stats_cap: int = 0, stream=None) -> CorrectResult:
    """The sharded algorithm with `nslabs` virtual ranks on the current GPU
    (loopback transport): bit-equal to exactz_correct (out, edit_counts and
    the whole-field int32 label outputs)."""
    import torch
    if out is None:
        out = torch.empty_like(g_in)
    o, st, rows = _opts(N, max_iters, flags, edit_counts, label_min, label_max, stats_cap)
    iters = C.c_uint32(0)
    s = _lib.exactz_correct_slabs(_ptr(f), _ptr(g_in), _dims(f), float(eps), nslabs, _ptr(out),
                                  C.byref(iters), C.byref(o), _stream(stream))
    if s not in (OK, ESTUCK):
        raise ExactzError(s, "exactz_correct_slabs")
    res = _result(s, iters, st, rows)
    res.out = out
    return res


def exactz_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    s = _lib.exactz_nccl_unique_id(buf)
    if s != OK:
        raise ExactzError(s, "exactz_nccl_unique_id")
    return bytes(buf)


class Comm:
    """An NCCL communicator of the sharded path (one rank per GPU)."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        self.h = C.c_void_p(0)
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        s = _lib.exactz_comm_init(buf, nranks, rank, device, C.byref(self.h))
        if s != OK:
            raise ExactzError(s, "exactz_comm_init")
        self.nranks, self.rank = nranks, rank

    def close(self):
        if self.h:
            _lib.exactz_comm_destroy(self.h)
            self.h = C.c_void_p(0)


def exactz_correct_sharded(comm: Comm, f_local, g_local, global_dims, eps: float, out=None, *,
                           N: int = 5, max_iters: int = 0, flags: int = 0, edit_counts=None,
                           label_min=None, label_max=None, stats_cap: int = 0,
                           stream=None) -> CorrectResult:
    """One rank of the z-slab decomposition: f_local/g_local are this rank's
    planes (shape (z_count, ny, nx)); collective over comm.  edit_counts and
    the int32 label outputs cover the local planes (labels: global ids)."""
    import torch
    if out is None:
        out = torch.empty_like(g_local)
    z0, zc = exactz_slab_range(int(global_dims[2]), comm.nranks, comm.rank)
    o, st, rows = _opts(N, max_iters, flags, edit_counts, label_min, label_max, stats_cap)
    iters = C.c_uint32(0)
    dims = (C.c_int64 * 3)(*[int(x) for x in global_dims])
    s = _lib.exactz_correct_sharded(comm.h, _ptr(f_local), _ptr(g_local), dims, z0, zc,
                                    float(eps), _ptr(out), C.byref(iters), C.byref(o),
                                    _stream(stream))
    if s not in (OK, ESTUCK):
        raise ExactzError(s, "exactz_correct_sharded")
    res = _result(s, iters, st, rows)
    res.out = out
    return res
