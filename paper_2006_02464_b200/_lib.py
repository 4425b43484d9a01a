"""ctypes binding of libcw.so (include/cw.h).

The library is built in-tree by `paper_2006_02464_b200.build`. There is no
fallback: if the library is missing the import of this module raises, and every
device call raises `CwError` with the library's own message on failure.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcw.so")
if os.environ.get("CW_LIB"):  # experiments only: a variant built with CW_BUILD_TAG
    LIB_PATH = os.path.join(_HERE, os.environ["CW_LIB"])

MAX_BATCH = 16


class CwError(RuntimeError):
    pass


class cw_op(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "layer", "in_buf", "out_buf", "res_buf", "cin", "cout", "kh", "kw", "stride",
        "pad", "relu", "in_h", "in_w", "out_h", "out_w", "kpad", "pad_w", "in_ctot",
        "out_ctot", "out_coff", "cout_pad", "flags", "pre_layer")]


class cw_tensor_loc(C.Structure):
    _fields_ = [("w_off", C.c_int64), ("b_off", C.c_int64), ("rows", C.c_int32), ("k", C.c_int32),
                ("s_off", C.c_int64)]


class cw_model_info(C.Structure):
    _fields_ = [
        ("blob_id", C.c_int32), ("arch_id", C.c_int32), ("pages_needed", C.c_int32),
        ("n_batches", C.c_int32), ("batch_sizes", C.c_int32 * 8), ("exec_ns", C.c_int64 * 8),
        ("weights_transfer_ns", C.c_int64), ("input_size", C.c_int64), ("output_size", C.c_int64),
        ("input_transfer_ns", C.c_int64), ("output_transfer_ns", C.c_int64)]


class cw_engine_config(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("worker_id", C.c_int32), ("gpu_count", C.c_int32),
        ("n_models", C.c_int32), ("pages_per_gpu", C.c_int64), ("page_bytes", C.c_int64),
        ("io_capacity", C.c_int64), ("epoch_ns", C.c_int64),
        ("devices", C.POINTER(C.c_int32)), ("models", C.POINTER(cw_model_info)),
        ("io_slots", C.c_int64), ("in_bytes_max", C.c_int64), ("out_bytes_max", C.c_int64),
        ("executor_cpu", C.c_int32), ("executor_rt_prio", C.c_int32), ("peer_load", C.c_int32)]


class cw_action(C.Structure):
    _fields_ = [
        ("action_id", C.c_uint64), ("kind", C.c_int32), ("model_id", C.c_uint32),
        ("gpu_index", C.c_int32), ("batch_size", C.c_int32), ("earliest", C.c_int64),
        ("latest", C.c_int64), ("expected_duration", C.c_int64),
        ("request_ids", C.c_uint64 * MAX_BATCH)]


class cw_result(C.Structure):
    _fields_ = [
        ("action_id", C.c_uint64), ("status", C.c_int32), ("kind", C.c_int32),
        ("start", C.c_int64), ("end", C.c_int64), ("device_duration", C.c_int64),
        ("output_ref", C.c_int64), ("pages_free", C.c_int64)]


class cw_net_record(C.Structure):
    _fields_ = [
        ("action_id", C.c_uint64), ("kind", C.c_int32), ("model_id", C.c_uint32),
        ("gpu_index", C.c_int32), ("batch_size", C.c_int32), ("status", C.c_int32),
        ("pad_", C.c_int32), ("start", C.c_int64), ("end", C.c_int64),
        ("device_duration", C.c_int64)]


# (name, restype, argtypes) for every symbol include/cw.h declares.
_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
SIGNATURES = [
    ("cw_abi_version", C.c_int, []),
    ("cw_last_error", C.c_char_p, []),
    ("cw_device_count", C.c_int, []),
    ("cw_rt_open", _P, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    ("cw_rt_close", None, [_P]),
    ("cw_rt_register_arch", C.c_int, [_P, C.c_int, C.POINTER(cw_op), C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.c_int, _I32P, C.c_int]),
    ("cw_rt_register_blob", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int64,
                                      C.POINTER(cw_tensor_loc), C.c_int]),
    ("cw_rt_build", C.c_int, [_P]),
    ("cw_rt_set_input_pool", C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int64]),
    ("cw_rt_clock_offset", C.c_int64, [_P]),
    ("cw_rt_plan_info", C.c_int, [_P, C.c_int, C.c_int, _I32P, C.POINTER(C.c_double)]),
    ("cw_rt_load_sync", C.c_int, [_P, C.c_int, _I32P, C.c_int, _I64P]),
    ("cw_rt_infer_sync", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, _P, _P, _I64P]),
    ("cw_rt_exec_many", C.c_int, [_P, C.c_int, C.c_int, _I32P, C.c_int, _I64P, _I64P]),
    ("cw_rt_exec_closed", C.c_int, [_P, C.c_int, C.c_int, _I32P, C.c_int, _I64P, _I64P]),
    ("cw_rt_profile_layers", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, _P, _I32P, C.c_int]),
    ("cw_rt_last_trace", C.c_int64, [_P, _P, C.c_int64]),
    ("cw_rt_plan_layers", C.c_int, [_P, C.c_int, C.c_int, _I32P, C.c_int]),
    ("cw_rt_plan_launch", C.c_int, [_P, C.c_int, C.c_int, _I32P, _I32P]),
    ("cw_rt_buffer_io", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int64, C.c_int]),
    ("cw_rt_exec_window", C.c_int, [_P, C.c_int, C.c_int, C.c_int32, C.c_int64, C.c_int64,
                                    _I32P, _I64P, _I64P]),
    ("cw_engine_open", _P, [C.POINTER(cw_engine_config)]),
    ("cw_engine_runtime", _P, [_P, C.c_int]),
    ("cw_engine_start", C.c_int, [_P]),
    ("cw_engine_close", None, [_P]),
    ("cw_engine_submit", C.c_int, [_P, C.POINTER(cw_action), C.c_int64]),
    ("cw_engine_poll", C.c_int, [_P, C.POINTER(cw_result), C.c_int, C.c_int64]),
    ("cw_engine_sim_run", C.c_int, [_P, C.c_int64]),
    ("cw_engine_now", C.c_int64, [_P]),
    ("cw_engine_next_time", C.c_int64, [_P]),
    ("cw_engine_failed", C.c_int, [_P]),
    ("cw_engine_executor_info", C.c_int, [_P, _I32P, _I32P]),
    ("cw_engine_stats", C.c_int, [_P, C.c_int, _I64P, C.c_int]),
    ("cw_engine_clock_drift", C.c_int, [_P, C.c_int, _I64P]),
    ("cw_engine_sim_deliver", C.c_int, [_P, C.POINTER(cw_action), C.c_int64]),
    ("cw_engine_sim_take_new", C.c_int, [_P, _I64P, C.POINTER(C.c_uint64), C.c_int]),
    ("cw_engine_sim_run_to", C.c_int, [_P, C.c_int64, C.c_uint64]),
    ("cw_engine_pages", C.c_int, [_P, C.c_int, _I64P, _I32P, _I32P, C.c_int, _I32P]),
    ("cw_engine_io_in_use", C.c_int64, [_P, C.c_int]),
    ("cw_engine_output", C.c_int, [_P, C.c_int, C.c_int64, _P, C.c_int, C.c_int]),
    ("cw_wire_decode_action", C.c_int, [C.c_char_p, C.c_int64, C.POINTER(cw_action)]),
    ("cw_wire_encode_result", C.c_int, [C.POINTER(cw_result), C.c_char_p]),
    ("cw_wire_encode_handshake", C.c_int64, [C.c_uint32, C.c_uint32, C.c_uint64,
                                             C.POINTER(C.c_uint32), C.c_int32, C.c_char_p,
                                             C.c_int64]),
    ("cw_sched_create", _P, [C.c_int32, _I32P, _I32P, _I64P, _I64P, _I64P, _I64P, _I32P,
                             _I64P, C.c_double]),
    ("cw_sched_destroy", None, [_P]),
    ("cw_sched_handshake", C.c_int, [_P, C.c_int32, C.c_int32, C.c_int64]),
    ("cw_sched_request", C.c_int, [_P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64]),
    ("cw_sched_result", C.c_int, [_P, C.c_int64, C.c_uint64, C.c_int32, C.c_int64, C.c_int64,
                                  C.c_int64]),
    ("cw_sched_timer", C.c_int, [_P, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64]),
    ("cw_sched_records", _I64P, [_P]),
    ("cw_sched_ids", C.POINTER(C.c_uint64), [_P, _I64P]),
    ("cw_sched_live", C.c_int64, [_P]),
    ("cw_sched_fsum", C.c_double, [C.POINTER(C.c_double), C.c_int64]),
    ("cw_net_serve", C.c_int, [_P, C.c_int, C.c_char_p, C.c_int64, C.c_int64,
                               C.POINTER(cw_net_record), C.c_int64, _I64P, _I64P]),
]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2006_02464_b200.build` "
            "(there is no CPU fallback for the worker's device path)")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        if os.environ.get("CW_LIB") and not hasattr(lib, name):
            continue  # experiments: an older variant library may predate a symbol
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    return (lib.cw_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise CwError(f"{what}: {last_error()}")
    return rc
