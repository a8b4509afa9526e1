"""ctypes binding of libprune_b200.so (declarations in include/prune_b200.h).

The library is built in-tree by `paper_1802_06625_b200.build`; there is no
fallback: if it cannot be loaded every device entry point raises
`DeviceUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import (ActorPanic, DeviceUnavailable, EndOfStream, InvalidParams, Poisoned, Timeout,
                     ProtocolError, UnsupportedGraph)

# PB_LIB_PATH selects an alternative build of the same library (profiling
# experiments with different compile-time tunings); default: the in-tree build
LIB_PATH = Path(os.environ.get("PB_LIB_PATH") or
                Path(__file__).resolve().parent / "libprune_b200.so")

PB_OK = 0
PB_E_INVALID = -1
PB_E_PROTOCOL = -2
PB_E_EOS = -3
PB_E_POISONED = -4
PB_E_CUDA = -5
PB_E_NOMEM = -6
PB_E_UNSUPPORTED = -7
PB_E_ACTOR = -8
PB_E_TIMEOUT = -9

PB_TAPS = 10
PB_FIR_EXACT = 0
PB_FIR_EXACT_PAIRED = 1
PB_FIR_FMA = 2
PB_FIR_MERGED = 3
PB_CONV_BF16X3 = 0
PB_CONV_I8 = 1
PB_MAX_BRANCHES = 32
PB_MAX_PORTS = 16
PB_POLICY_STATE_BYTES = 2560

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64


class Plan(C.Structure):
    _fields_ = [("rate", i32), ("token_bytes", i32), ("delay", i32), ("factor", i32),
                ("aligned", i32), ("pad_", i32), ("slots", i64), ("nbytes", i64),
                ("copy_src", i64), ("copy_dst", i64), ("copy_count", i64)]


class Condition(C.Structure):
    _fields_ = [("tokens", vp), ("stream_stride", i64), ("token_stride", i32),
                ("element", i32), ("slots", i32), ("base", i32)]


class Resolved(C.Structure):
    _fields_ = [("act", vp), ("prefix", vp), ("count", vp), ("worklist", vp),
                ("n_cond", i32), ("n_streams", i32), ("n_iter", i32), ("cap", i32)]


class Eq1Port(C.Structure):
    _fields_ = [("own_cond", i32), ("moved_cond", i32), ("actor_cond", i32), ("pad_", i32)]


class RingAdvance(C.Structure):
    _fields_ = [("counters", vp), ("cond", i32), ("rate", i32), ("delay", i32), ("pad_", i32)]


class SpanRef(C.Structure):
    _fields_ = [("data", vp), ("stream_stride", i64), ("span_bytes", i64), ("base", vp),
                ("slots", i32), ("index_cond", i32), ("act_cond", i32), ("offset", i32)]


class FirActor(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("taps", vp), ("state", vp),
                ("cond", i32), ("pad_", i32)]


class FilterBank(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("branches", vp), ("n_branches", i32),
                ("actor_cond", i32), ("sched", vp), ("math", i32), ("pad_", i32)]


class SumActor(C.Structure):
    _fields_ = [("in_", SpanRef * PB_MAX_PORTS), ("out", SpanRef), ("n_in", i32), ("cond", i32)]


class BytesActor(C.Structure):
    _fields_ = [("in_", SpanRef * PB_MAX_PORTS), ("out", SpanRef * PB_MAX_PORTS),
                ("n_in", i32), ("n_out", i32), ("offset", i32), ("cond", i32)]


class MatmulActor(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("weights", vp), ("n", i32), ("cond", i32)]


class MatmulChainActor(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("weights", vp), ("n", i32),
                ("layers", i32), ("cond", i32), ("pad_", i32)]


class PathMergeActor(C.Structure):
    _fields_ = [("in_", SpanRef * PB_MAX_PORTS), ("out", SpanRef), ("n_in", i32),
                ("bypass_index", i32), ("marker", C.c_float), ("cond", i32),
                ("error_flag", vp)]


class ImageActor(C.Structure):
    _fields_ = [("in_", SpanRef * 2), ("out", SpanRef * PB_MAX_PORTS), ("n_out", i32),
                ("op", i32), ("side", i32), ("threshold", i32), ("cond", i32), ("pad_", i32)]


PB_IMG_BLUR, PB_IMG_DIFF, PB_IMG_MEDIAN = 0, 1, 2


class BypassRegion(C.Structure):
    _fields_ = [("chain_in", SpanRef), ("bypass_in", SpanRef), ("out", SpanRef), ("weights", vp),
                ("layers", i32), ("chain_live", i32), ("cond", i32), ("marker", C.c_float),
                ("error_flag", vp)]


class MotionRegion(C.Structure):
    _fields_ = [("in_", SpanRef), ("prev_in", SpanRef), ("prev_out", SpanRef), ("out", SpanRef),
                ("side", i32), ("threshold", i32)]


class ConvActor(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("weights", vp), ("bias", vp),
                ("frames", i32), ("h", i32), ("w", i32), ("cin", i32), ("cout", i32),
                ("pad", i32), ("cond", i32), ("debug", i32), ("math", i32),
                ("weights_i8", vp), ("absmax_out", vp), ("absmax_in", vp)]


class DenseActor(C.Structure):
    _fields_ = [("in_", SpanRef), ("out", SpanRef), ("weights", vp), ("bias", vp),
                ("frames", i32), ("nin", i32), ("nout", i32), ("cond", i32)]


class ClassifyActor(C.Structure):
    _fields_ = [("chain", SpanRef), ("bypass", SpanRef), ("out", SpanRef), ("w4", vp),
                ("b4", vp), ("w5", vp), ("b5", vp), ("frames", i32), ("nin", i32),
                ("nhid", i32), ("nout", i32), ("marker", C.c_float), ("cond", i32),
                ("error_flag", vp)]


# name -> (restype, argtypes); every symbol include/prune_b200.h declares
SIGNATURES = {
    "pb_abi_version": (C.c_int, []),
    "pb_last_error": (C.c_char_p, []),
    "pb_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "pb_set_device": (C.c_int, [C.c_int]),
    "pb_device_sync": (C.c_int, []),
    "pb_sm_count": (C.c_int, [C.POINTER(C.c_int)]),
    "pb_malloc": (C.c_int, [C.POINTER(vp), C.c_size_t]),
    "pb_free": (C.c_int, [vp]),
    "pb_host_alloc": (C.c_int, [C.POINTER(vp), C.c_size_t]),
    "pb_host_free": (C.c_int, [vp]),
    "pb_host_register": (C.c_int, [vp, C.c_size_t]),
    "pb_host_unregister": (C.c_int, [vp]),
    "pb_memcpy_h2d": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "pb_memcpy_d2h": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "pb_memcpy_d2d": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "pb_memset": (C.c_int, [vp, C.c_int, C.c_size_t, vp]),
    "pb_memcpy_2d": (C.c_int, [vp, C.c_size_t, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int,
                               vp]),
    "pb_stream_create": (C.c_int, [C.POINTER(vp)]),
    "pb_stream_destroy": (C.c_int, [vp]),
    "pb_stream_sync": (C.c_int, [vp]),
    "pb_event_create": (C.c_int, [C.POINTER(vp)]),
    "pb_event_destroy": (C.c_int, [vp]),
    "pb_event_record": (C.c_int, [vp, vp]),
    "pb_event_elapsed_ms": (C.c_int, [vp, vp, C.POINTER(C.c_float)]),
    "pb_event_sync": (C.c_int, [vp]),
    "pb_stream_wait": (C.c_int, [vp, vp]),
    "pb_launch_count": (i64, []),
    "pb_layout_plan": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(Plan)]),
    "pb_writer_gate": (i64, [i64, C.c_int, C.c_int, C.c_int, C.c_int]),
    "pb_reader_gate": (i64, [i64, C.c_int, C.c_int]),
    "pb_copy_gate": (i64, [i64, C.c_int, C.c_int, C.c_int]),
    "pb_ring_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                                 C.POINTER(vp)]),
    "pb_ring_destroy": (C.c_int, [vp]),
    "pb_ring_plan": (C.c_int, [vp, C.POINTER(Plan)]),
    "pb_ring_storage": (C.c_int, [vp, C.POINTER(vp), C.POINTER(i64), C.POINTER(vp)]),
    "pb_ring_push_host": (C.c_int, [vp, C.c_int, vp, i64, vp]),
    "pb_ring_pop_host": (C.c_int, [vp, C.c_int, vp, i64, vp]),
    "pb_ring_push_host_wait": (C.c_int, [vp, C.c_int, vp, i64, vp, i64]),
    "pb_ring_pop_host_wait": (C.c_int, [vp, C.c_int, vp, i64, vp, i64]),
    "pb_ring_counters": (C.c_int, [vp, C.c_int, C.POINTER(i64), C.POINTER(i64),
                                   C.POINTER(i64)]),
    "pb_ring_close": (C.c_int, [vp]),
    "pb_ring_poison": (C.c_int, [vp, C.c_char_p]),
    "pb_resolve": (C.c_int, [C.POINTER(Condition), Resolved, vp]),
    "pb_eq1_check": (C.c_int, [C.POINTER(Eq1Port), C.c_int, Resolved, vp, vp]),
    "pb_rings_advance": (C.c_int, [C.POINTER(RingAdvance), C.c_int, Resolved, vp]),
    "pb_epoch_close": (C.c_int, [C.POINTER(Eq1Port), C.c_int, vp, C.POINTER(RingAdvance),
                                 C.c_int, Resolved, vp]),
    "pb_fire_fir": (C.c_int, [vp, C.c_int, Resolved, i64, C.c_int, vp]),
    "pb_fir_carry": (C.c_int, [vp, C.c_int, Resolved, i64, vp]),
    "pb_fire_filter_bank": (C.c_int, [FilterBank, Resolved, i64, vp]),
    "pb_fire_branch_sum": (C.c_int, [SumActor, Resolved, i64, vp]),
    "pb_fire_bytes": (C.c_int, [BytesActor, Resolved, vp]),
    "pb_fire_matmul": (C.c_int, [MatmulActor, Resolved, vp]),
    "pb_fire_matmul_chain": (C.c_int, [MatmulChainActor, Resolved, vp]),
    "pb_fire_motion_region": (C.c_int, [MotionRegion, Resolved, vp]),
    "pb_fire_bypass_region": (C.c_int, [BypassRegion, Resolved, vp]),
    "pb_fire_path_merge": (C.c_int, [PathMergeActor, Resolved, vp]),
    "pb_fire_image": (C.c_int, [ImageActor, Resolved, vp]),
    "pb_fire_conv_pool": (C.c_int, [ConvActor, Resolved, vp]),
    "pb_conv_debug_counters": (C.c_int, [vp, C.c_int]),
    "pb_fire_dense": (C.c_int, [DenseActor, Resolved, vp]),
    "pb_fire_classify": (C.c_int, [ClassifyActor, Resolved, vp]),
    "pb_policy_init": (C.c_int, [vp, i64]),
    "pb_policy_tokens": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, i64, i64, vp, C.c_int]),
    "pb_policy_tokens_streams": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, i64, i64,
                                           vp, C.c_int, C.c_int]),
    "pb_crc32": (C.c_uint32, [vp, C.c_size_t]),
}

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load libprune_b200.so and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DeviceUnavailable(
            f"{LIB_PATH} is missing; build it with `python -m paper_1802_06625_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pb_abi_version() != 1:
        raise DeviceUnavailable("libprune_b200 ABI version mismatch")
    _lib = lib
    return lib


def error_text() -> str:
    msg = load().pb_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "") -> int:
    """Map a PB_E_* status onto the reference's exception types."""
    if rc == PB_OK:
        return rc
    text = error_text()
    if what:
        text = f"{what}: {text}"
    if rc == PB_E_INVALID:
        raise InvalidParams(text)
    if rc == PB_E_PROTOCOL:
        raise ProtocolError(text)
    if rc == PB_E_EOS:
        raise EndOfStream(text)
    if rc == PB_E_POISONED:
        raise Poisoned("ring", text)
    if rc == PB_E_UNSUPPORTED:   # shape / size outside what the kernels implement
        raise UnsupportedGraph(text)
    if rc == PB_E_ACTOR:
        raise ActorPanic(what or "device", RuntimeError(text))
    if rc == PB_E_TIMEOUT:
        raise Timeout(None, [], text)
    raise DeviceUnavailable(text or f"libprune_b200 status {rc}")


def call(name: str, *args) -> int:
    return check(getattr(load(), name)(*args), name)


def device_count() -> int:
    n = C.c_int(0)
    rc = load().pb_device_count(C.byref(n))
    return n.value if rc == PB_OK else 0
