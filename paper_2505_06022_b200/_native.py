"""ctypes binding of ``libcq.so`` (include/cq.h).

Every call is checked: a non-zero status raises ``NativeError`` (or the
reference error type it corresponds to) with ``cq_last_error()``'s message.
There is deliberately no fallback -- if the library is missing or no GPU is
visible, the executor fails loudly.
"""

import ctypes
import os

from .errors import EvalError, MapperViolationError, NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CQ_LIB", os.path.join(HERE, "libcq.so"))

CQ_OK, CQ_ERR_CUDA, CQ_ERR_NCCL, CQ_ERR_NVML, CQ_ERR_ARG = 0, 1, 2, 3, 4
CQ_ERR_PERMISSION, CQ_ERR_UNSUPPORTED, CQ_ERR_EVAL, CQ_ERR_MAPPER, CQ_ERR_P2P = 5, 6, 7, 8, 9
CQ_F64, CQ_F32, CQ_I64 = 0, 1, 2
STREAM_COMPUTE, STREAM_BOUNDARY, STREAM_COMM = 0, 1, 2
STREAM_LANE0, NUM_LANES = 3, 8
ALL_STREAMS = tuple(range(STREAM_LANE0 + NUM_LANES))
SIDE_STREAMS = ALL_STREAMS[1:]   # joined to / forked from the compute stream
SGEMM_FFMA, SGEMM_3XTF32 = 0, 1

KIND_CODE = {"float64": CQ_F64, "float32": CQ_F32, "int64": CQ_I64}

MAX_CODE, MAX_CONST, MAX_SLOTS, MAX_VIEWS, MAX_OUT, MAX_CHECK = 192, 64, 24, 8, 4, 8

i64 = ctypes.c_int64
i32 = ctypes.c_int32
u64 = ctypes.c_uint64
vp = ctypes.c_void_p


class CqBox(ctypes.Structure):
    _fields_ = [("lo", i64 * 3), ("hi", i64 * 3)]


class CqView(ctypes.Structure):
    _fields_ = [("ptr", vp), ("alloc", CqBox), ("stride", i64 * 3)]


class CqPeerSync(ctypes.Structure):
    """cq_peer_sync_t: in-pass ordering with the neighbouring ranks."""
    _fields_ = [("slot", ctypes.c_void_p * 2), ("count", ctypes.c_void_p), ("done", ctypes.c_void_p),
                ("peer_slot", ctypes.c_void_p * 2), ("peer_amax", ctypes.c_void_p * 2),
                ("timeout_ns", ctypes.c_int64)]


class CqMirror(ctypes.Structure):
    """cq_mirror_t: peer allocations that also receive some output rows of a fused pass."""
    _fields_ = [("last", ctypes.c_void_p), ("prev", ctypes.c_void_p), ("row0", ctypes.c_int64),
                ("col0", ctypes.c_int64), ("stride", ctypes.c_int64), ("row_lo", ctypes.c_int64),
                ("row_hi", ctypes.c_int64)]


class CqExpr(ctypes.Structure):
    _fields_ = [
        ("kind", i32), ("dims", i32), ("box", CqBox),
        ("n_out", i32), ("out_code_begin", i32 * MAX_OUT), ("out_code_end", i32 * MAX_OUT),
        ("out", CqView * MAX_OUT),
        ("n_code", i32), ("code_op", ctypes.c_int16 * MAX_CODE), ("code_arg", ctypes.c_int16 * MAX_CODE),
        ("n_const", i32), ("consts", i64 * MAX_CONST),
        ("n_slots", i32), ("slot_view", i32 * MAX_SLOTS), ("slot_off", (i32 * 3) * MAX_SLOTS),
        ("n_views", i32), ("views", CqView * MAX_VIEWS), ("view_extent", CqBox * MAX_VIEWS),
        ("view_dims", i32 * MAX_VIEWS), ("view_n_check", i32 * MAX_VIEWS),
        ("view_check", (CqBox * MAX_CHECK) * MAX_VIEWS),
    ]


P = ctypes.POINTER
_SIGS = {
    "cq_last_error": (ctypes.c_char_p, []),
    "cq_version": (i32, [P(i32)]),
    "cq_device_count": (i32, [P(i32)]),
    "cq_init_device": (i32, [i32]),
    "cq_device_props": (i32, [i32, P(i32), P(i64), P(i32), P(i64)]),
    "cq_enable_peer": (i32, [i32, i32, P(i32)]),
    "cq_shutdown": (i32, []),
    "cq_malloc": (i32, [i32, i64, P(vp)]),
    "cq_free": (i32, [i32, vp]),
    "cq_pool_trim": (i32, [i32]),
    "cq_host_register": (i32, [vp, i64]),
    "cq_host_alloc": (i32, [i64, P(vp)]),
    "cq_host_free": (i32, [vp]),
    "cq_host_unregister": (i32, [vp]),
    "cq_copy_h2d": (i32, [i32, i32, vp, vp, i64]),
    "cq_copy_d2h": (i32, [i32, i32, vp, vp, i64]),
    "cq_copy_box": (i32, [i32, i32, i32, P(CqView), i32, P(CqView), i32, P(CqBox)]),
    "cq_copy_box_h2d": (i32, [i32, i32, i32, P(CqView), vp, P(CqBox), P(CqBox)]),
    "cq_copy_box_d2h": (i32, [i32, i32, i32, vp, P(CqBox), P(CqView), P(CqBox)]),
    "cq_pack_box": (i32, [i32, i32, i32, vp, P(CqView), P(CqBox)]),
    "cq_unpack_box": (i32, [i32, i32, i32, P(CqView), vp, P(CqBox)]),
    "cq_event_create": (i32, [i32, i32, P(u64)]),
    "cq_event_destroy": (i32, [u64]),
    "cq_event_record": (i32, [u64, i32, i32]),
    "cq_event_record_timed": (i32, [u64, i32, i32]),
    "cq_stream_wait_event": (i32, [i32, i32, u64]),
    "cq_event_synchronize": (i32, [u64]),
    "cq_event_elapsed_ms": (i32, [u64, u64, P(ctypes.c_float)]),
    "cq_stream_synchronize": (i32, [i32, i32]),
    "cq_device_synchronize": (i32, [i32]),
    "cq_graph_begin": (i32, [i32]),
    "cq_graph_end": (i32, [i32, P(u64)]),
    "cq_graph_launch": (i32, [u64, i32]),
    "cq_graph_destroy": (i32, [u64]),
    "cq_nccl_unique_id": (i32, [ctypes.c_char_p]),
    "cq_nccl_init": (i32, [i32, i32, i32, ctypes.c_char_p]),
    "cq_nccl_group_start": (i32, []),
    "cq_nccl_group_end": (i32, []),
    "cq_nccl_send": (i32, [i32, i32, vp, i64, i32]),
    "cq_nccl_recv": (i32, [i32, i32, vp, i64, i32]),
    "cq_nccl_allgather": (i32, [i32, i32, vp, vp, i64]),
    "cq_nccl_bcast": (i32, [i32, i32, vp, i64, i32]),
    "cq_ipc_handle": (i32, [vp, vp]),
    "cq_ipc_open": (i32, [i32, vp, P(vp)]),
    "cq_ipc_close": (i32, [i32, vp]),
    "cq_p2p_wait": (i32, [i32, i32, vp, vp, vp, i64]),
    "cq_p2p_signal": (i32, [i32, i32, vp, vp, vp]),
    "cq_nccl_destroy": (i32, []),
    "cq_fill": (i32, [i32, i32, i32, P(CqView), P(CqBox), P(CqBox), i32, ctypes.c_double, i64]),
    "cq_saxpy": (i32, [i32, i32, i32, ctypes.c_double, i64, vp, vp, vp, i64]),
    "cq_wave5": (i32, [i32, i32, i32, P(CqView), P(CqView), P(CqView), P(CqBox), P(CqBox),
                       ctypes.c_double, ctypes.c_double, ctypes.c_double]),
    "cq_wave5_fused": (i32, [i32, i32, i32, i32, P(CqView), P(CqView), P(CqView), P(CqView), i64, i64, i64, i64,
                             P(CqBox), ctypes.c_double, ctypes.c_double, ctypes.c_double]),
    "cq_wave5_fused_bounded": (i32, [i32, i32, i32, i32, P(CqView), P(CqView), P(CqView), P(CqView), i64, i64,
                                     i64, i64, P(CqBox), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     vp, vp]),
    "cq_wave5_fused_ex": (i32, [i32, i32, i32, i32, P(CqView), P(CqView), P(CqView), P(CqView), i64, i64,
                                i64, i64, P(CqBox), ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                vp, vp, i64, i64, vp, i32, vp]),
    "cq_wave5_fused_geometry": (i32, [i32, i32, i32, i64, i64, P(i64)]),
    "cq_expr_eval": (i32, [i32, i32, P(CqExpr)]),
    "cq_error_flag": (i32, [i32, P(i32), P(i64), i32]),
    "cq_error_flag_async": (i32, [i32, i32, vp]),
    "cq_nbody_kick": (i32, [i32, i32, vp, i64, vp, vp, i64, i64, ctypes.c_float, ctypes.c_float]),
    "cq_nbody_drift": (i32, [i32, i32, vp, vp, vp, i64, ctypes.c_float]),
    "cq_nbody_jcols": (i32, [P(i32)]),
    "cq_nbody_kick_partial": (i32, [i32, i32, vp, i64, vp, i64, i64, ctypes.c_float, i32, i32]),
    "cq_nbody_kick_finalize": (i32, [i32, i32, vp, vp, vp, i64, ctypes.c_float]),
    "cq_sgemm": (i32, [i32, i32, i32, vp, i64, vp, i64, vp, i64, i64, i64, i64]),
    "cq_jit_compile": (i32, [ctypes.c_char_p, ctypes.c_char_p, i32, P(ctypes.c_char_p),
                             P(ctypes.c_char_p), P(u64)]),
    "cq_jit_launch": (i32, [u64, i32, i32, P(CqExpr)]),
    "cq_plan_generate": (i32, [P(i64), i64, i32, P(P(i64)), P(i64)]),
    "cq_plan_free": (i32, [P(i64)]),
    "cq_nvml_init": (i32, []),
    "cq_nvml_energy_mj": (i32, [i32, P(u64)]),
    "cq_nvml_power_mw": (i32, [i32, P(ctypes.c_uint)]),
    "cq_nvml_sm_clock_mhz": (i32, [i32, P(ctypes.c_uint), P(ctypes.c_uint)]),
    "cq_nvml_throttle_reasons": (i32, [i32, P(ctypes.c_ulonglong)]),
    "cq_nvml_supported_sm_clocks": (i32, [i32, P(ctypes.c_uint), P(i32)]),
    "cq_nvml_lock_sm_clock": (i32, [i32, ctypes.c_uint]),
    "cq_nvml_reset_sm_clock": (i32, [i32]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """The loaded library (raises NativeError when it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"libcq.so not found at {LIB_PATH}; run "
                          f"`python -m paper_2505_06022_b200.build` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_host_lib = None


def load_host():
    """The real libcq for host-only entry points (the planner): never the
    device-side test double a CPU test may install as ``_lib``."""
    global _host_lib
    if _host_lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"libcq.so not found at {LIB_PATH}")
        lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name in ("cq_plan_generate", "cq_plan_free", "cq_last_error", "cq_jit_compile"):
            res, args = _SIGS[name]
            getattr(lib, name).restype = res
            getattr(lib, name).argtypes = args
        _host_lib = lib
    return _host_lib


def check(status, what=""):
    if status == CQ_OK:
        return
    msg = load().cq_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == CQ_ERR_EVAL:
        raise EvalError(text)
    if status == CQ_ERR_MAPPER:
        raise MapperViolationError(text)
    raise NativeError(text, status)


def call(name, *args):
    """Call ``cq_<name>`` and raise on failure."""
    check(getattr(load(), name)(*args), name)


def box3(lo, hi):
    """Pad a 1..3-D box to the C-ABI's 3-D form (leading unit axes)."""
    pad = 3 - len(lo)
    b = CqBox()
    b.lo[:] = [0] * pad + list(lo)
    b.hi[:] = [1] * pad + list(hi)
    return b
