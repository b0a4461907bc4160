"""ctypes binding of libqcs_b200.so (the C ABI declared in include/qcs_abi.h).

There is no fallback: if the shared library is missing or cannot be loaded, importing the
package's compute API raises ``ImportError``; if no CUDA device is present, calls fail with
``CudaError`` (QCS_ERR_CUDA).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QCS_B200_LIB", os.path.join(HERE, "libqcs_b200.so"))

QCS_OK, QCS_ERR_CAPACITY, QCS_ERR_DIMENSION, QCS_ERR_ENCODING, QCS_ERR_PARSE, QCS_ERR_SIM, \
    QCS_ERR_CUDA, QCS_ERR_NCCL, QCS_ERR_ARG = range(9)
QCS_MEM_HOST, QCS_MEM_DEVICE = 0, 1
QCS_STEP_GATES, QCS_STEP_DIAG = 0, 1
MAX_ARITY = 3


# pointer members as void* (same ABI): plain integer addresses assign without ctypes casts
class qcs_placement(C.Structure):
    _fields_ = [("arity", C.c_int), ("qubits", C.c_void_p), ("matrix", C.c_void_p), ("name", C.c_char_p)]


class qcs_step(C.Structure):
    _fields_ = [("kind", C.c_int), ("stage", C.c_int), ("placements", C.c_void_p), ("num_placements", C.c_int),
                ("flipped", C.c_void_p), ("num_flipped", C.c_uint64), ("flip_rest", C.c_int)]


class qcs_sim_options(C.Structure):
    _fields_ = [("sign_method", C.c_int), ("block_size", C.c_uint64), ("fuse", C.c_int), ("reset", C.c_int),
                ("initial", C.c_uint64)]


class qcs_step_report(C.Structure):
    _fields_ = [("structure", C.c_int), ("stage", C.c_int), ("matrix_bytes", C.c_uint64),
                ("dense_bytes", C.c_uint64), ("entry_count", C.c_uint64), ("sign_count", C.c_uint64),
                ("madd_count", C.c_uint64)]


class qcs_plan_info(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("ops", "passes", "tile_passes", "single_passes", "rounds",
                                         "smem_rounds", "reg_ops", "max_tile_bits", "alt_passes",
                                         "skip_passes", "paired_passes", "fp64_ops", "sweep_amps")]


_P = C.c_void_p
_PS = C.POINTER(_P)
_D = C.POINTER(C.c_double)
_U64 = C.POINTER(C.c_uint64)
_U8 = C.POINTER(C.c_uint8)
_I = C.POINTER(C.c_int)

# name -> (restype, argtypes)
SIGNATURES = {
    "qcs_last_error": (C.c_char_p, []),
    "qcs_version": (C.c_char_p, []),
    "qcs_device_count": (C.c_int, [_I]),
    "qcs_set_dense_cap": (C.c_int, [C.c_uint64]),
    "qcs_dense_cap": (C.c_uint64, []),
    "qcs_gate_catalog_size": (C.c_int, []),
    "qcs_gate_catalog_entry": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), _I, _I, _D]),
    "qcs_gate_lookup": (C.c_int, [C.c_char_p, _D, C.c_int, _D, _I, C.POINTER(C.c_char_p)]),
    "qcs_canonical_params": (C.c_int, [C.c_char_p, _D, _I]),
    "qcs_state_create": (C.c_int, [C.c_int, C.c_int, C.c_uint64, _PS]),
    "qcs_state_wrap": (C.c_int, [C.c_int, C.c_int, _P, _P, _PS]),
    "qcs_state_destroy": (C.c_int, [_P]),
    "qcs_state_info": (C.c_int, [_P, _I, _I, _PS, _PS]),
    "qcs_state_set_basis": (C.c_int, [_P, C.c_uint64]),
    "qcs_state_upload": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64]),
    "qcs_state_download": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64]),
    "qcs_state_download_async": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64]),
    "qcs_state_wait": (C.c_int, [_P, _P]),
    "qcs_state_copy": (C.c_int, [_P, _P]),
    "qcs_state_sync": (C.c_int, [_P]),
    "qcs_state_random": (C.c_int, [_P, C.c_uint64]),
    "qcs_host_alloc": (C.c_int, [C.c_size_t, _PS]),
    "qcs_host_free": (C.c_int, [_P]),
    "qcs_apply_step": (C.c_int, [_P, C.POINTER(qcs_placement), C.c_int]),
    "qcs_apply_diag": (C.c_int, [_P, _U64, C.c_uint64, C.c_int]),
    "qcs_apply_rh": (C.c_int, [_P]),
    "qcs_norm": (C.c_int, [_P, _D]),
    "qcs_probabilities": (C.c_int, [_P, _P, C.c_int]),
    "qcs_argmax": (C.c_int, [_P, _U64, _D]),
    "qcs_topk": (C.c_int, [_P, C.c_int, _U64, _D]),
    "qcs_gather": (C.c_int, [_P, _U64, C.c_uint64, _D]),
    "qcs_state_distance": (C.c_int, [_P, _P, _D, _D]),
    "qcs_summary": (C.c_int, [_P, C.c_int, _D, _U64, _D]),
    "qcs_summary_begin": (C.c_int, [_P, C.c_int]),
    "qcs_summary_end": (C.c_int, [_P, _D, _U64, _D]),
    "qcs_sample": (C.c_int, [_P, C.c_uint64, C.c_uint64, _U64, _D]),
    "qcs_rh_mvm": (C.c_int, [_P, C.c_int, C.c_double, C.c_int, C.c_uint64, _U64, _U64]),
    "qcs_simulate": (C.c_int, [_P, C.POINTER(qcs_step), C.c_int, C.c_int, C.POINTER(qcs_sim_options),
                               C.POINTER(qcs_step_report)]),
    "qcs_memory_report": (C.c_int, [C.c_int, C.POINTER(qcs_step), C.c_int, C.c_int, C.POINTER(qcs_step_report)]),
    "qcs_apply_split": (C.c_int, [_P, _P, C.c_int, C.c_int, _I, _D, C.c_uint32]),
    "qcs_swap_peer": (C.c_int, [_P, C.c_uint64, _P, C.c_uint64]),
    "qcs_plan_stats": (C.c_int, [C.c_int, C.POINTER(qcs_step), C.c_int, C.c_int, C.POINTER(qcs_sim_options),
                                 C.POINTER(qcs_plan_info)]),
    "qcs_set_jit_mode": (C.c_int, [C.c_int]),
    "qcs_get_jit_mode": (C.c_int, []),
    "qcs_set_pipeline_mode": (C.c_int, [C.c_int]),
    "qcs_get_pipeline_mode": (C.c_int, []),
    "qcs_plan_compile": (C.c_int, [C.c_int, C.POINTER(qcs_step), C.c_int, C.c_int, C.POINTER(qcs_sim_options),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "qcs_plan_verify": (C.c_int, [C.c_int, C.POINTER(qcs_step), C.c_int, C.c_int, C.POINTER(qcs_sim_options),
                                  C.POINTER(C.c_int64)]),
    "qcs_step_dax": (C.c_int, [C.c_int, C.POINTER(qcs_placement), C.c_int, C.c_int, _P, _P, _P, C.c_uint64,
                               C.c_int, _U64]),
    "qcs_step_das": (C.c_int, [C.c_int, C.POINTER(qcs_placement), C.c_int, C.c_int, _P, _P, _P, C.c_uint64,
                               C.c_int, _U64]),
    "qcs_dax_mvm": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int, _P, _P]),
    "qcs_das_mvm": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int, _P, _P]),
    "qcs_kernel_launches": (C.c_uint64, []),
    "qcs_event_record": (C.c_int, [_P, C.c_int]),
    "qcs_event_elapsed_ms": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "qcs_timing_enable": (C.c_int, [_P, C.c_int]),
    "qcs_timing_reset": (C.c_int, [_P]),
    "qcs_timing_count": (C.c_int, [_P, _I]),
    "qcs_timing_entry": (C.c_int, [_P, C.c_int, C.POINTER(C.c_char_p), _U64, _D, _D]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2411_15332_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load()
    return _lib
