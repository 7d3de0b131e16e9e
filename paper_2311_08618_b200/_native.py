"""ctypes binding of libh2ldl.so (include/h2ldl.h) and the plan exporter.

The library is the only compute path: there is no CPU fallback.  If the
shared object is missing, or no sm_100 device is usable, every entry point
raises `NativeError` (loudly, at call time).

`upload(H, device)` flattens the origin of a RankStructuredMatrix into the
`h2l_plan` struct (static schedule + one float64 arena) and uploads it once;
the engine is cached on the origin per device, the same lifetime the
reference gives its skeleton caches (`compress.py:99-127`).
"""

import ctypes
import os
import threading

import numpy as np

from .errors import NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2L_LIB", os.path.join(HERE, "libh2ldl.so"))

H2L_OK = 0
H2L_SHIFT_OK = 0
H2L_SHIFT_SINGULAR = 1
KIND = {"strong": 0, "weak": 1, "flat": 2}

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class Plan(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("depth", ctypes.c_int32), ("kind", ctypes.c_int32),
        ("n_dense", ctypes.c_int32), ("n_lowrank", ctypes.c_int32),
        ("n_deferred", ctypes.c_int32),
        ("eps", ctypes.c_double), ("scale0", ctypes.c_double),
        ("ranges", _i64p), ("dense", _i32p), ("lowrank", _i32p), ("deferred", _i32p),
        ("basis_rank", _i32p), ("basis_dim", _i32p), ("basis_off", _i64p),
        ("diag_off", _i64p), ("dense_off", _i64p), ("lowrank_off", _i64p),
        ("arena", _f64p), ("arena_len", ctypes.c_int64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("fill_blocks", ctypes.c_int64), ("recompressions", ctypes.c_int64),
        ("rank_added", ctypes.c_int64), ("max_front", ctypes.c_int64),
        ("dropped_fro", ctypes.c_double), ("flops", ctypes.c_double),
        ("bytes", ctypes.c_double), ("ms_total", ctypes.c_double),
        ("ms_schur", ctypes.c_double), ("ms_bk", ctypes.c_double),
        ("launches", ctypes.c_int64), ("schur_flops", ctypes.c_double),
        ("gemm_flops_exec", ctypes.c_double), ("ms_kind", ctypes.c_double * 8),
        ("ms_host", ctypes.c_double), ("mem_peak", ctypes.c_double),
        ("elim_flops", ctypes.c_double), ("groups", ctypes.c_int64),
        ("paths", ctypes.c_int64 * 4),
    ]

    def as_dict(self):
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["ms_kind"] = list(self.ms_kind)
        d["paths"] = list(self.paths)
        return d


SYMBOLS = ("h2l_create", "h2l_destroy", "h2l_last_error", "h2l_upload", "h2l_inertia",
           "h2l_inertia_device", "h2l_set_option", "h2l_bk_factor", "h2l_bk_inertia",
           "h2l_comm_init", "h2l_inertia_multi", "h2l_comm_destroy", "h2l_version")

_lib = None
_lib_lock = threading.Lock()


def load_library(path=LIB_PATH):
    """Load libh2ldl.so and declare its prototypes (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeError(f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        lib = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        lib.h2l_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
        lib.h2l_destroy.argtypes = [vp]
        lib.h2l_last_error.argtypes = [vp]
        lib.h2l_last_error.restype = ctypes.c_char_p
        lib.h2l_upload.argtypes = [vp, ctypes.POINTER(Plan)]
        lib.h2l_inertia.argtypes = [vp, _f64p, ctypes.c_int32, _i64p, _i32p,
                                    ctypes.POINTER(Stats)]
        lib.h2l_inertia_device.argtypes = [vp, _f64p, ctypes.c_int32, ctypes.c_void_p,
                                           ctypes.POINTER(Stats)]
        lib.h2l_comm_init.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(vp)]
        lib.h2l_inertia_multi.argtypes = [vp, _f64p, ctypes.c_int32, _i64p, _i32p,
                                          ctypes.POINTER(Stats)]
        lib.h2l_comm_destroy.argtypes = [vp]
        lib.h2l_set_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        lib.h2l_bk_factor.argtypes = [ctypes.c_int, _f64p, ctypes.c_int64, ctypes.c_int32, _i64p,
                                      _f64p, _i64p]
        lib.h2l_bk_inertia.argtypes = [ctypes.c_int, _f64p, ctypes.c_int64, ctypes.c_int32,
                                       _i64p, _f64p, _i64p]
        lib.h2l_version.restype = ctypes.c_char_p
        for name in SYMBOLS:
            getattr(lib, name).restype = getattr(lib, name).restype or ctypes.c_int
        lib.h2l_last_error.restype = ctypes.c_char_p
        lib.h2l_version.restype = ctypes.c_char_p
        _lib = lib
        return lib


TESTING_LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "libh2ldl_testing.so")
_tlib = None


def load_testing_library(path=TESTING_LIB_PATH):
    """libh2ldl_testing.so: test / benchmark entry points outside the product ABI
    (GEMM tile variants, BK and Gram-ordering kernels on host matrices, the INT8
    Ozaki Schur kernel on dense inputs).  Only tests/ and tools/ load it."""
    global _tlib
    load_library()
    with _lib_lock:
        if _tlib is None:
            if not os.path.exists(path):
                raise NativeError(f"{path} is missing: run __graft_entry__.build()")
            _tlib = ctypes.CDLL(path)
            _tlib.h2l_testing_last_error.restype = ctypes.c_char_p
        return _tlib


def _check(rc, handle=None, what=""):
    if rc != H2L_OK:
        msg = load_library().h2l_last_error(handle)
        raise NativeError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")


def _ptr(a, typ):
    return a.ctypes.data_as(typ)


class DeviceEngine:
    """One h2l_engine bound to a device holding one uploaded H payload."""

    def __init__(self, device=0):
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.h2l_create(ctypes.byref(h), int(device)), None, "h2l_create")
        self.lib, self.handle, self.device = lib, h, device
        self._keep = None
        self.lock = threading.Lock()

    def __del__(self):
        try:
            if self.handle:
                self.lib.h2l_destroy(self.handle)
                self.handle = None
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def set_option(self, key, value):
        _check(self.lib.h2l_set_option(self.handle, key.encode(), int(value)), self.handle,
               "h2l_set_option")

    def upload(self, H):
        plan, keep = build_plan(H)
        arena = getattr(H, "_arena", None)
        with self.lock:
            if arena is not None:
                # device-built H: the engine reads its arena in place (no 2nd copy in HBM)
                self.set_option("borrow_arena", 1)
            _check(self.lib.h2l_upload(self.handle, ctypes.byref(plan)), self.handle, "h2l_upload")
        # host plan arrays must outlive the call only; a borrowed device arena must
        # outlive the engine: keep a reference to it
        self._keep = (keep, arena)

    def inertia(self, mus):
        """(counts[s,3] int64, status[s] int32, stats dict) for absolute shifts mus."""
        mus = np.ascontiguousarray(np.asarray(mus, dtype=np.float64).reshape(-1))
        s = mus.shape[0]
        counts = np.zeros((s, 3), dtype=np.int64)
        status = np.zeros(s, dtype=np.int32)
        st = Stats()
        with self.lock:
            _check(self.lib.h2l_inertia(self.handle, _ptr(mus, _f64p), s, _ptr(counts, _i64p),
                                        _ptr(status, _i32p), ctypes.byref(st)),
                   self.handle, "h2l_inertia")
        return counts, status, st.as_dict()


    def inertia_device(self, mus, out):
        """Counts straight into device memory: `out` is a CUDA int64 tensor (or a raw
        device pointer) on this engine's device with >= 4*len(mus) elements, filled
        with rows (neg, zero, pos, status).  Returns the stats dict."""
        mus = np.ascontiguousarray(np.asarray(mus, dtype=np.float64).reshape(-1))
        s = mus.shape[0]
        ptr = out if isinstance(out, int) else out.data_ptr()
        if not isinstance(out, int):
            if out.numel() < 4 * s or str(out.dtype) != "torch.int64" or not out.is_cuda:
                raise NativeError("inertia_device: out must be a CUDA int64 tensor of 4*s elements")
        st = Stats()
        with self.lock:
            _check(self.lib.h2l_inertia_device(self.handle, _ptr(mus, _f64p), s, ctypes.c_void_p(ptr),
                                               ctypes.byref(st)), self.handle, "h2l_inertia_device")
        return st.as_dict()


class MultiEngine:
    """One process driving several GPUs (h2l_comm_init / h2l_inertia_multi): one
    DeviceEngine per device, each holding the uploaded H, shifts sharded in
    contiguous slices, counts exchanged by an NCCL all-gather between the
    engines' device buffers."""

    def __init__(self, H, devices):
        self.lib = load_library()
        self.engines = [engine_for(H, d) for d in devices]
        arr = (ctypes.c_void_p * len(self.engines))(*[e.handle.value for e in self.engines])
        c = ctypes.c_void_p()
        _check(self.lib.h2l_comm_init(arr, len(self.engines), ctypes.byref(c)), None, "h2l_comm_init")
        self.comm = c

    def __del__(self):
        try:
            if self.comm:
                self.lib.h2l_comm_destroy(self.comm)
                self.comm = None
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def inertia(self, mus):
        mus = np.ascontiguousarray(np.asarray(mus, dtype=np.float64).reshape(-1))
        s = mus.shape[0]
        counts = np.zeros((s, 3), dtype=np.int64)
        status = np.zeros(s, dtype=np.int32)
        st = Stats()
        _check(self.lib.h2l_inertia_multi(self.comm, _ptr(mus, _f64p), s, _ptr(counts, _i64p),
                                          _ptr(status, _i32p), ctypes.byref(st)),
               None, "h2l_inertia_multi")
        return counts, status, st.as_dict()


def _device_plan(org):
    """Plan over the device arena of a gpu_build.construct_device matrix (no copies)."""
    tree, st = org.tree, org.structure
    depth = tree.depth
    nodes = (1 << (depth + 1)) - 1
    off = org._arena_offsets
    ranges = np.array([r for lv in tree.ranges for r in lv], dtype=np.int64).reshape(-1)
    nleaf = 1 << depth
    diag_off = np.array([off[("D", i)] for i in range(nleaf)], dtype=np.int64)
    dense = np.array(st.dense, dtype=np.int32).reshape(-1, 2)
    dense_off = np.array([off[("O", (i, j))] for i, j in st.dense], dtype=np.int64)
    low = [(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]]
    low_off = np.array([off[("C", k)] for k in low], dtype=np.int64)
    lowrank = np.array(low, dtype=np.int32).reshape(-1, 3)
    dfr = [(l, i, j) for l in sorted(st.deferred) for i, j in st.deferred[l]]
    deferred = np.array(dfr, dtype=np.int32).reshape(-1, 3)
    brank = np.full(nodes, -1, dtype=np.int32)
    bdim = np.zeros(nodes, dtype=np.int32)
    boff = np.full(nodes, -1, dtype=np.int64)
    for (l, i), bs in org.bases.items():
        nd = (1 << l) - 1 + i
        brank[nd] = bs.rank
        bdim[nd] = bs.m
        if bs.m:
            boff[nd] = off[("B", (l, i))]
    arena = org._arena
    keep = [ranges, dense, lowrank, deferred, brank, bdim, boff, diag_off, dense_off, low_off,
            arena]
    plan = Plan(
        n=tree.n, depth=depth, kind=KIND[st.kind], n_dense=len(dense), n_lowrank=len(low),
        n_deferred=len(dfr), eps=float(org.eps), scale0=float(org.scale0()),
        ranges=_ptr(ranges, _i64p), dense=_ptr(dense, _i32p), lowrank=_ptr(lowrank, _i32p),
        deferred=_ptr(deferred, _i32p), basis_rank=_ptr(brank, _i32p),
        basis_dim=_ptr(bdim, _i32p), basis_off=_ptr(boff, _i64p),
        diag_off=_ptr(diag_off, _i64p), dense_off=_ptr(dense_off, _i64p),
        lowrank_off=_ptr(low_off, _i64p),
        arena=ctypes.cast(ctypes.c_void_p(arena.data_ptr()), _f64p), arena_len=arena.numel())
    return plan, keep


def build_plan(H):
    """Flatten origin(H) into an h2l_plan (returns the struct and the arrays it points to).

    Host payloads are concatenated into one numpy arena; a device-built H
    (gpu_build.construct_device) passes its device arena as is."""
    org = H.origin()
    if getattr(org, "_arena", None) is not None:
        return _device_plan(org)
    tree, st = org.tree, org.structure
    depth = tree.depth
    nodes = (1 << (depth + 1)) - 1
    ranges = np.array([r for lv in tree.ranges for r in lv], dtype=np.int64).reshape(-1)
    chunks, pos = [], 0

    def put(a):
        nonlocal pos
        a = np.ascontiguousarray(a, dtype=np.float64)
        off = pos
        chunks.append(a.reshape(-1))
        pos += a.size
        return off

    nleaf = 1 << depth
    diag_off = np.array([put(org.leaf_diag[i]) for i in range(nleaf)], dtype=np.int64)
    dense = np.array(st.dense, dtype=np.int32).reshape(-1, 2)
    dense_off = np.array([put(org.leaf_offdiag[(i, j)]) for i, j in st.dense], dtype=np.int64)
    low = [(l, i, j) for l in sorted(st.lowrank) for i, j in st.lowrank[l]]
    low_off = np.array([put(org.couplings[k]) for k in low], dtype=np.int64)
    lowrank = np.array(low, dtype=np.int32).reshape(-1, 3)
    dfr = [(l, i, j) for l in sorted(st.deferred) for i, j in st.deferred[l]]
    deferred = np.array(dfr, dtype=np.int32).reshape(-1, 3)
    brank = np.full(nodes, -1, dtype=np.int32)
    bdim = np.zeros(nodes, dtype=np.int32)
    boff = np.full(nodes, -1, dtype=np.int64)
    for (l, i), bs in org.bases.items():
        nd = (1 << l) - 1 + i
        brank[nd] = bs.rank
        bdim[nd] = bs.m
        if bs.m:
            boff[nd] = put(bs.square())
    arena = np.concatenate(chunks) if chunks else np.zeros(1)
    arena = np.ascontiguousarray(arena, dtype=np.float64)
    keep = [ranges, dense, lowrank, deferred, brank, bdim, boff, diag_off, dense_off, low_off,
            arena]
    plan = Plan(
        n=tree.n, depth=depth, kind=KIND[st.kind], n_dense=len(dense), n_lowrank=len(low),
        n_deferred=len(dfr), eps=float(org.eps), scale0=float(org.scale0()),
        ranges=_ptr(ranges, _i64p), dense=_ptr(dense, _i32p), lowrank=_ptr(lowrank, _i32p),
        deferred=_ptr(deferred, _i32p), basis_rank=_ptr(brank, _i32p),
        basis_dim=_ptr(bdim, _i32p), basis_off=_ptr(boff, _i64p),
        diag_off=_ptr(diag_off, _i64p), dense_off=_ptr(dense_off, _i64p),
        lowrank_off=_ptr(low_off, _i64p), arena=_ptr(arena, _f64p), arena_len=arena.size)
    return plan, keep


_default_device = 0


def set_default_device(device):
    global _default_device
    _default_device = int(device)


def default_device():
    return _default_device


def engine_for(H, device=None):
    """Engine holding origin(H) on `device` (uploaded on first use, then cached)."""
    org = H.origin()
    dev = _default_device if device is None else int(device)
    eng = org._device.get(dev)
    if eng is None:
        eng = DeviceEngine(dev)
        eng.upload(org)
        org._device[dev] = eng
    return eng


def bk_factor_device(A_batch, tol, device=None):
    """Batched BK on the device (KAT boundary of `_core.bk_factor`).

    A_batch: (count, n, n) float64, overwritten copy returned with ipiv, info."""
    lib = load_library()
    A = np.ascontiguousarray(np.array(A_batch, dtype=np.float64, copy=True))
    if A.ndim == 2:
        A = A[None]
    count, n = A.shape[0], A.shape[1]
    tol = np.ascontiguousarray(np.broadcast_to(np.asarray(tol, dtype=np.float64), (count,)))
    ipiv = np.zeros((count, n), dtype=np.int64)
    info = np.zeros(count, dtype=np.int64)
    dev = _default_device if device is None else device
    _check(lib.h2l_bk_factor(dev, _ptr(A, _f64p), n, count, _ptr(ipiv, _i64p), _ptr(tol, _f64p),
                             _ptr(info, _i64p)), None, "h2l_bk_factor")
    return A, ipiv, info


def bk_inertia_device(F_batch, ipiv, zero_tol, device=None):
    lib = load_library()
    F = np.ascontiguousarray(np.asarray(F_batch, dtype=np.float64))
    if F.ndim == 2:
        F = F[None]
    count, n = F.shape[0], F.shape[1]
    ip = np.ascontiguousarray(np.asarray(ipiv, dtype=np.int64).reshape(count, n))
    zt = np.ascontiguousarray(np.broadcast_to(np.asarray(zero_tol, dtype=np.float64), (count,)))
    out = np.zeros((count, 3), dtype=np.int64)
    dev = _default_device if device is None else device
    _check(lib.h2l_bk_inertia(dev, _ptr(F, _f64p), n, count, _ptr(ip, _i64p), _ptr(zt, _f64p),
                              _ptr(out, _i64p)), None, "h2l_bk_inertia")
    return out
