"""Thin ctypes binding of libjacc.so (include/jacc.h): same names, argument
marshalling only.  Every step of the path runs in the library's C++ runtime
and sm_100a kernels; there is no Python or CPU fallback.  Importing this
module raises if the shared library has not been built.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjacc.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
lib = ctypes.CDLL(LIB_PATH)

# ---- constants (mirror include/jacc.h) -----------------------------------
JACC_OK = 0
JACC_ERR_INVALID = -1
JACC_ERR_OVERLAP = -2
JACC_ERR_NOT_PRESENT = -3
JACC_ERR_UNKNOWN_LOOP = -4
JACC_ERR_OOM = -5
JACC_ERR_CUDA = -6
JACC_ERR_NCCL = -7
JACC_ERR_STATE = -8
JACC_MAX_DEVICES = 16
JACC_MERGE_EAGER = 0
JACC_MERGE_HALO = 1
JACC_MODE_MULTI = 0
JACC_MODE_DUP = 1
JACC_LOOP_SQUARE_F32 = 1
JACC_LOOP_JACOBI2D_F64 = 2
JACC_LOOP_DOT_F64 = 3
JACC_LOOP_SUM_F64 = 4
JACC_LOOP_GEMM_F64 = 5
JACC_LOOP_SCATTER_ADD_F64 = 6
JACC_LOOP_SCATTER_ADD_I32 = 7
JACC_LOOP_HIMENO_F32 = 8
JACC_LOOP_HIMENO_COPY_F32 = 9
JACC_LOOP_FIG4_F64 = 10
JACC_ARG_ARRAY_IN = 0
JACC_ARG_ARRAY_OUT = 1
JACC_ARG_ARRAY_INOUT = 2
JACC_ARG_SCALAR_F64 = 3
JACC_ARG_SCALAR_I64 = 4
JACC_ARG_REDUCE_SUM_F64 = 5
EMPTY_RANGE = (2**64 - 1, 0)

EXPORTS = [
    "jacc_init", "jacc_finalize", "jacc_num_devices", "jacc_partition", "jacc_set_merge_policy", "jacc_set_mode",
    "jacc_data_create", "jacc_data_delete", "jacc_update_device", "jacc_update_host",
    "jacc_launch", "jacc_wait", "jacc_get_dirty_range", "jacc_get_dirty_bitmap",
    "jacc_get_replica", "jacc_last_timing", "jacc_set_profiling", "jacc_profile_totals",
    "jacc_profile_reset", "jacc_get_stream", "jacc_error_string",
    "jacc_unique_id", "jacc_init_rank", "jacc_export_runtime", "jacc_import_runtime",
    "jacc_export_region", "jacc_import_region", "jacc_rank",
    "jacc_adaptive_replay", "jacc_adaptive_history",
    "jacc_graph_begin", "jacc_graph_end", "jacc_graph_replay", "jacc_graph_destroy",
    "jacc_select_split_dim", "jacc_exchange_plan", "jacc_set_split_dim",
    "jacc_set_scatter_split", "jacc_set_queues", "jacc_queue_replay", "jacc_get_info", "jacc_set_trace",
]
JACC_MAX_QUEUES = 32
JACC_ASYNC_AUTO = -2
JACC_MODE_ADAPTIVE = 2
JACC_UNIQUE_ID_BYTES = 128
JACC_RUNTIME_HANDLE_BYTES = 256
JACC_REGION_HANDLE_BYTES = 64


class jacc_range(ctypes.Structure):
    _fields_ = [("ndims", ctypes.c_int), ("lo", ctypes.c_int64 * 3), ("hi", ctypes.c_int64 * 3)]


class jacc_copy2d_plan(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("count", "height", "width_bytes", "pitch_bytes",
                                              "first_offset_bytes", "outer_stride_bytes")]


class jacc_info(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int) for k in ("n_devices", "distinct_gpus", "combine", "peer_pairs",
                                            "multiprocess", "rank")]


JACC_COMBINE_PEER = 0
JACC_COMBINE_NCCL = 1


class jacc_arg(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("ptr", ctypes.c_void_p), ("f64", ctypes.c_double),
                ("i64", ctypes.c_int64)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_PU64 = ctypes.POINTER(ctypes.c_uint64)
_PD = ctypes.POINTER(ctypes.c_double)
for _name, _args in {
    "jacc_init": [_I, ctypes.POINTER(_I)],
    "jacc_finalize": [],
    "jacc_set_merge_policy": [_I],
    "jacc_set_mode": [_I],
    "jacc_set_split_dim": [_I],
    "jacc_set_scatter_split": [_I],
    "jacc_set_queues": [_I],
    "jacc_queue_replay": [_I, _I, _P, _P, _P, _P, _P, _P, _P],
    "jacc_data_create": [_P, _SZ, _SZ, _I, ctypes.POINTER(ctypes.c_int64)],
    "jacc_data_delete": [_P],
    "jacc_update_device": [_P, _SZ, _SZ],
    "jacc_update_host": [_P, _SZ, _SZ],
    "jacc_launch": [_I, ctypes.POINTER(jacc_range), ctypes.POINTER(jacc_arg), _I, _I],
    "jacc_wait": [_I],
    "jacc_get_dirty_range": [_P, _I, _PU64, _PU64],
    "jacc_get_dirty_bitmap": [_P, _I, _P, _SZ],
    "jacc_get_replica": [_P, _I, _P, _SZ],
    "jacc_last_timing": [_PD, _PD, _PU64],
    "jacc_set_profiling": [_I],
    "jacc_profile_totals": [_I, _PD, _PD, _PU64, _PU64],
    "jacc_profile_reset": [],
    "jacc_get_stream": [_I, ctypes.POINTER(_P), ctypes.POINTER(_I)],
    "jacc_partition": [ctypes.c_int64, _I, _I, ctypes.POINTER(ctypes.c_int64),
                       ctypes.POINTER(ctypes.c_int64)],
    "jacc_unique_id": [_P, _SZ],
    "jacc_init_rank": [_I, _I, _I, _P, ctypes.c_char_p],
    "jacc_export_runtime": [_P, _SZ],
    "jacc_import_runtime": [_I, _P, _SZ],
    "jacc_export_region": [_P, _P, _SZ],
    "jacc_import_region": [_P, _I, _P, _SZ],
    "jacc_adaptive_replay": [_I, ctypes.c_double, _I, _P, _P, _P, _P],
    "jacc_graph_begin": [],
    "jacc_select_split_dim": [_I, ctypes.POINTER(_I), ctypes.POINTER(_I), _I, ctypes.POINTER(_I)],
    "jacc_exchange_plan": [_I, ctypes.POINTER(ctypes.c_int64), _SZ, _I, _I, _I,
                           ctypes.POINTER(jacc_copy2d_plan)],
    "jacc_graph_end": [ctypes.POINTER(_I)],
    "jacc_graph_replay": [_I, _I],
    "jacc_graph_destroy": [_I],
    "jacc_adaptive_history": [_I, _I, _P, _P, _P, _P, ctypes.POINTER(_I), ctypes.POINTER(_I)],
    "jacc_set_trace": [ctypes.c_char_p],
    "jacc_get_info": [ctypes.POINTER(jacc_info)],
}.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
lib.jacc_rank.argtypes = []
lib.jacc_rank.restype = ctypes.c_int
lib.jacc_num_devices.argtypes = []
lib.jacc_num_devices.restype = ctypes.c_int
lib.jacc_error_string.argtypes = [ctypes.c_int]
lib.jacc_error_string.restype = ctypes.c_char_p


class JaccError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        super().__init__(f"{what}: {lib.jacc_error_string(status).decode()} ({status})")


def _ck(st, what):
    if st != JACC_OK:
        raise JaccError(st, what)
    return st


def _addr(x):
    """Host address of a numpy array (or an int address)."""
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return int(x)


# ---- API (same names as the C-ABI) -----------------------------------------
def jacc_init(n_devices=1, device_ids=None):
    ids = None
    if device_ids is not None:
        ids = (ctypes.c_int * len(device_ids))(*device_ids)
    return _ck(lib.jacc_init(n_devices, ids), "jacc_init")


def jacc_finalize():
    return _ck(lib.jacc_finalize(), "jacc_finalize")


def jacc_num_devices():
    return lib.jacc_num_devices()


def jacc_partition(E, n, d):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _ck(lib.jacc_partition(E, n, d, ctypes.byref(lo), ctypes.byref(hi)), "jacc_partition")
    return lo.value, hi.value


def jacc_set_merge_policy(policy):
    return _ck(lib.jacc_set_merge_policy(policy), "jacc_set_merge_policy")


def jacc_set_scatter_split(iteration_split):
    return _ck(lib.jacc_set_scatter_split(1 if iteration_split else 0), "jacc_set_scatter_split")


def jacc_set_split_dim(dim):
    return _ck(lib.jacc_set_split_dim(dim), "jacc_set_split_dim")


def jacc_set_mode(mode):
    return _ck(lib.jacc_set_mode(mode), "jacc_set_mode")


def jacc_data_create(arr, extents=None, elem_size=None, nbytes=None):
    """Register a numpy array (C-contiguous) as a present region."""
    if isinstance(arr, np.ndarray):
        assert arr.flags.c_contiguous
        extents = arr.shape if extents is None else extents
        elem_size = arr.itemsize if elem_size is None else elem_size
        nbytes = arr.nbytes if nbytes is None else nbytes
    ext = (ctypes.c_int64 * len(extents))(*extents)
    return _ck(lib.jacc_data_create(_addr(arr), nbytes, elem_size, len(extents), ext),
               "jacc_data_create")


def jacc_data_delete(arr):
    return _ck(lib.jacc_data_delete(_addr(arr)), "jacc_data_delete")


def jacc_update_device(arr, offset_bytes=0, nbytes=None):
    if nbytes is None:
        nbytes = arr.nbytes - offset_bytes
    return _ck(lib.jacc_update_device(_addr(arr), offset_bytes, nbytes), "jacc_update_device")


def jacc_update_host(arr, offset_bytes=0, nbytes=None):
    if nbytes is None:
        nbytes = arr.nbytes - offset_bytes
    return _ck(lib.jacc_update_host(_addr(arr), offset_bytes, nbytes), "jacc_update_host")


def arg(kind, x=None, f64=0.0, i64=0):
    """jacc_arg: arrays by host address (numpy array or int), reductions by a
    host double (numpy float64 array of size >= 1)."""
    return jacc_arg(kind, _addr(x) if x is not None else None, f64, i64)


def make_range(lo, hi):
    lo = list(lo) if hasattr(lo, "__len__") else [lo]
    hi = list(hi) if hasattr(hi, "__len__") else [hi]
    r = jacc_range()
    r.ndims = len(lo)
    for k in range(len(lo)):
        r.lo[k], r.hi[k] = lo[k], hi[k]
    return r


def jacc_launch(loop_id, rng, args, async_id=-1):
    arr = (jacc_arg * len(args))(*args)
    rp = ctypes.byref(rng) if rng is not None else None
    return _ck(lib.jacc_launch(loop_id, rp, arr, len(args), async_id), "jacc_launch")


def jacc_launch_status(loop_id, rng, args, async_id=-1):
    """Same as jacc_launch but returns the status instead of raising."""
    arr = (jacc_arg * len(args))(*args) if args else None
    rp = ctypes.byref(rng) if rng is not None else None
    return lib.jacc_launch(loop_id, rp, arr, len(args) if args else 0, async_id)


def jacc_wait(async_id=-1):
    return _ck(lib.jacc_wait(async_id), "jacc_wait")


def jacc_get_dirty_range(arr, dev):
    mn, mx = ctypes.c_uint64(), ctypes.c_uint64()
    _ck(lib.jacc_get_dirty_range(_addr(arr), dev, ctypes.byref(mn), ctypes.byref(mx)),
        "jacc_get_dirty_range")
    return mn.value, mx.value


def jacc_get_dirty_bitmap(arr, dev, nelem):
    out = np.zeros((nelem + 31) // 32, dtype=np.uint32)
    _ck(lib.jacc_get_dirty_bitmap(_addr(arr), dev, out.ctypes.data, out.size),
        "jacc_get_dirty_bitmap")
    return out


def jacc_get_replica(arr, dev):
    out = np.empty_like(arr)
    _ck(lib.jacc_get_replica(_addr(arr), dev, out.ctypes.data, out.nbytes), "jacc_get_replica")
    return out


def jacc_last_timing():
    k, m, b = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint64()
    _ck(lib.jacc_last_timing(ctypes.byref(k), ctypes.byref(m), ctypes.byref(b)), "jacc_last_timing")
    return k.value, m.value, b.value


def jacc_set_profiling(on):
    return _ck(lib.jacc_set_profiling(1 if on else 0), "jacc_set_profiling")


def jacc_profile_totals(dev):
    k, m = ctypes.c_double(), ctypes.c_double()
    nl, b = ctypes.c_uint64(), ctypes.c_uint64()
    _ck(lib.jacc_profile_totals(dev, ctypes.byref(k), ctypes.byref(m), ctypes.byref(nl),
                                ctypes.byref(b)), "jacc_profile_totals")
    return k.value, m.value, nl.value, b.value


def jacc_profile_reset():
    return _ck(lib.jacc_profile_reset(), "jacc_profile_reset")


def jacc_get_stream(dev):
    s, o = ctypes.c_void_p(), ctypes.c_int()
    _ck(lib.jacc_get_stream(dev, ctypes.byref(s), ctypes.byref(o)), "jacc_get_stream")
    return s.value, o.value


def jacc_set_trace(path):
    """JSON-lines trace of every launch (D13); None closes it."""
    p = None if path is None else str(path).encode()
    return _ck(lib.jacc_set_trace(p), "jacc_set_trace")


def jacc_get_info():
    """Runtime facts for measurements: devices, distinct GPUs, reduction
    combine ("nccl" | "peer"), peer-access pairs, process mode."""
    info = jacc_info()
    _ck(lib.jacc_get_info(ctypes.byref(info)), "jacc_get_info")
    d = {k: getattr(info, k) for k, _ in jacc_info._fields_}
    d["combine"] = "nccl" if info.combine == JACC_COMBINE_NCCL else "peer"
    return d


def jacc_error_string(status):
    return lib.jacc_error_string(status).decode()


# ---- one process per GPU ------------------------------------------------------
def _blob(n):
    return ctypes.create_string_buffer(n)


def jacc_unique_id():
    b = _blob(JACC_UNIQUE_ID_BYTES)
    _ck(lib.jacc_unique_id(b, len(b)), "jacc_unique_id")
    return bytes(b.raw)


def jacc_init_rank(rank, world, cuda_ordinal, unique_id, shm_name):
    uid = ctypes.create_string_buffer(unique_id, JACC_UNIQUE_ID_BYTES) if unique_id else None
    return _ck(lib.jacc_init_rank(rank, world, cuda_ordinal, uid, shm_name.encode()),
               "jacc_init_rank")


def jacc_export_runtime():
    b = _blob(JACC_RUNTIME_HANDLE_BYTES)
    _ck(lib.jacc_export_runtime(b, len(b)), "jacc_export_runtime")
    return bytes(b.raw)


def jacc_import_runtime(peer, blob):
    b = ctypes.create_string_buffer(blob, len(blob))
    return _ck(lib.jacc_import_runtime(peer, b, len(blob)), "jacc_import_runtime")


def jacc_export_region(arr):
    b = _blob(JACC_REGION_HANDLE_BYTES)
    _ck(lib.jacc_export_region(_addr(arr), b, len(b)), "jacc_export_region")
    return bytes(b.raw)


def jacc_import_region(arr, peer, blob):
    b = ctypes.create_string_buffer(blob, len(blob))
    return _ck(lib.jacc_import_region(_addr(arr), peer, b, len(blob)), "jacc_import_region")


def jacc_rank():
    return lib.jacc_rank()


# ---- adaptive utilization controller (NEXT-1) --------------------------------
def jacc_adaptive_replay(n, peak_p2p, trace):
    """States before each observation + final state (pure host logic)."""
    m = len(trace)
    tk = np.ascontiguousarray([t[0] for t in trace], dtype=np.float64)
    tc = np.ascontiguousarray([t[1] for t in trace], dtype=np.float64)
    ws = np.ascontiguousarray([t[2] for t in trace], dtype=np.float64)
    out = np.zeros(m + 1, dtype=np.int32)
    _ck(lib.jacc_adaptive_replay(n, peak_p2p, m, tk.ctypes.data, tc.ctypes.data, ws.ctypes.data,
                                 out.ctypes.data), "jacc_adaptive_replay")
    return out.tolist()


def jacc_adaptive_history(loop_id, cap=4096):
    tk, tc, ws = (np.zeros(cap) for _ in range(3))
    st = np.zeros(cap, dtype=np.int32)
    ln, now = ctypes.c_int(), ctypes.c_int()
    _ck(lib.jacc_adaptive_history(loop_id, cap, tk.ctypes.data, tc.ctypes.data, ws.ctypes.data,
                                  st.ctypes.data, ctypes.byref(ln), ctypes.byref(now)),
        "jacc_adaptive_history")
    m = min(ln.value, cap)
    return list(zip(tk[:m], tc[:m], ws[:m])), st[:m].tolist(), now.value


# ---- CUDA graphs of launch sequences ------------------------------------------
def jacc_graph_begin():
    return _ck(lib.jacc_graph_begin(), "jacc_graph_begin")


def jacc_graph_end():
    g = ctypes.c_int()
    _ck(lib.jacc_graph_end(ctypes.byref(g)), "jacc_graph_end")
    return g.value


def jacc_graph_replay(graph_id, count=1):
    return _ck(lib.jacc_graph_replay(graph_id, count), "jacc_graph_replay")


def jacc_graph_destroy(graph_id):
    return _ck(lib.jacc_graph_destroy(graph_id), "jacc_graph_destroy")


# ---- A18 / A19 division of multidimensional arrays ---------------------------
def jacc_select_split_dim(n_parallel, n_sequential, fortran=False):
    nd = len(n_parallel)
    par = (ctypes.c_int * nd)(*n_parallel)
    seq = (ctypes.c_int * nd)(*n_sequential)
    d = ctypes.c_int()
    _ck(lib.jacc_select_split_dim(nd, par, seq, 1 if fortran else 0, ctypes.byref(d)),
        "jacc_select_split_dim")
    return d.value


def jacc_exchange_plan(extents, elem, split_dim, n, d):
    ext = (ctypes.c_int64 * len(extents))(*extents)
    out = jacc_copy2d_plan()
    _ck(lib.jacc_exchange_plan(len(extents), ext, elem, split_dim, n, d, ctypes.byref(out)),
        "jacc_exchange_plan")
    return {k: getattr(out, k) for k, _ in jacc_copy2d_plan._fields_}


# ---- NEXT-4 automated async queues -------------------------------------------
def jacc_set_queues(nq):
    return _ck(lib.jacc_set_queues(nq), "jacc_set_queues")


def jacc_queue_replay(nq, trace):
    """trace: list of (reads, writes, requested or None) -> [(queue, waits)]"""
    m = len(trace)
    nr = np.array([len(t[0]) for t in trace] or [0], dtype=np.int32)
    nw = np.array([len(t[1]) for t in trace] or [0], dtype=np.int32)
    rd = np.array([x for t in trace for x in t[0]] or [0], dtype=np.int64)
    wr = np.array([x for t in trace for x in t[1]] or [0], dtype=np.int64)
    rq = np.array([(-1 if t[2] is None else t[2]) for t in trace] or [0], dtype=np.int32)
    qo = np.zeros(max(m, 1), dtype=np.int32)
    wo = np.zeros(max(m, 1) * nq, dtype=np.int32)
    _ck(lib.jacc_queue_replay(nq, m, nr.ctypes.data, rd.ctypes.data, nw.ctypes.data, wr.ctypes.data,
                              rq.ctypes.data, qo.ctypes.data, wo.ctypes.data), "jacc_queue_replay")
    return [(int(qo[l]), [q for q in range(nq) if wo[l * nq + q]]) for l in range(m)]
