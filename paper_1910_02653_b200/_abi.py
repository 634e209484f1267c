"""ctypes declarations of include/cm.h (argument marshalling only).

The shared library is built in-tree (paper_1910_02653_b200/build.py).  There is
no fallback: if the library is missing or fails to load, importing the binding
raises, so nothing can silently run on the CPU."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CM_LIB: load another build of the same library (kernel-variant tuning); never a fallback
LIB_PATH = os.environ.get("CM_LIB") or os.path.join(_HERE, "libcheckmate_b200.so")

CM_OK, CM_EINVAL, CM_ETOPO, CM_EDUP, CM_ERANGE, CM_ECUDA, CM_ENOMEM = range(7)
CM_NMAX = 1024
CM_EMAX = 8192
CM_LAYOUT_DENSE = 0
CM_LAYOUT_TRI4 = 1
CM_LAYOUT_BLK = 2
CM_KEY_NONE = (1 << 63) - 1
CM_ROUND_THRESHOLD = 0
CM_ROUND_RANDOMIZED = 1
CM_EVAL_INIT_KEYS = 1
CM_EVAL_OVERLAP = 2

EXPORTS = ("cm_graph_create", "cm_graph_destroy", "cm_graph_n", "cm_graph_cost_bound",
           "cm_round_and_evaluate", "cm_workspace_bytes", "cm_sstar_floats", "cm_debug_trace", "cm_debug_last_launches", "cm_debug_cta_trace", "cm_debug_cta_trace_at",
           "cm_last_call_seq", "cm_stream_wait_call", "cm_key_idx_bits", "cm_decode_key", "cm_decode_batch_key", "cm_status_string", "cm_emit_plan", "cm_plan_last_error",
           "cm_policy_checkpoints", "cm_policy_sstar", "cm_policy_last_error",
           "cm_mc_supported", "cm_mc_create", "cm_mc_export_fd", "cm_mc_import_fd", "cm_mc_size", "cm_mc_handle_type",
           "cm_mc_add_device", "cm_mc_bind", "cm_mc_destroy", "cm_mc_last_error",
           "cm_last_error")


class EvalArgs(ctypes.Structure):
    _fields_ = [
        ("n_sstar", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("sstar", ctypes.c_void_p),
        ("ld", ctypes.c_int64),
        ("sstar_stride", ctypes.c_int64),
        ("n_theta", ctypes.c_int32),
        ("theta", ctypes.c_void_p),
        ("n_budget", ctypes.c_int32),
        ("budget", ctypes.c_void_p),
        ("index_base", ctypes.c_int64),
        ("total_candidates", ctypes.c_int64),
        ("peak", ctypes.c_void_p),
        ("cost", ctypes.c_void_p),
        ("best_key", ctypes.c_void_p),
        ("r_mask", ctypes.c_void_p),
        ("s_mask", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_int64),
        ("rounding", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("best_batch_key", ctypes.c_void_p),
        ("cost_limit", ctypes.c_int64),
        ("flags", ctypes.c_int32),
        ("best_key_mc", ctypes.c_void_p),
        ("best_batch_key_mc", ctypes.c_void_p),
    ]


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_1910_02653_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.cm_graph_create.argtypes = [ctypes.c_int32, P, P, P, P, ctypes.c_int64, ctypes.POINTER(P)]
    lib.cm_graph_create.restype = ctypes.c_int
    lib.cm_graph_destroy.argtypes = [P]
    lib.cm_graph_destroy.restype = None
    lib.cm_graph_n.argtypes = [P]
    lib.cm_graph_n.restype = ctypes.c_int32
    lib.cm_graph_cost_bound.argtypes = [P]
    lib.cm_graph_cost_bound.restype = ctypes.c_int64
    lib.cm_round_and_evaluate.argtypes = [P, ctypes.POINTER(EvalArgs), P]
    lib.cm_round_and_evaluate.restype = ctypes.c_int
    lib.cm_sstar_floats.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64]
    lib.cm_sstar_floats.restype = ctypes.c_int64
    lib.cm_workspace_bytes.argtypes = [P, ctypes.c_int64]
    lib.cm_workspace_bytes.restype = ctypes.c_int64
    lib.cm_debug_trace.argtypes = [P, ctypes.c_int32]
    lib.cm_debug_trace.restype = ctypes.c_int32
    lib.cm_debug_last_launches.argtypes = []
    lib.cm_debug_last_launches.restype = ctypes.c_int32
    lib.cm_debug_cta_trace.argtypes = [P, ctypes.c_int32]
    lib.cm_debug_cta_trace.restype = ctypes.c_int32
    lib.cm_debug_cta_trace_at.argtypes = [ctypes.c_int32, P, ctypes.c_int32]
    lib.cm_debug_cta_trace_at.restype = ctypes.c_int32
    lib.cm_last_call_seq.argtypes = [P]
    lib.cm_last_call_seq.restype = ctypes.c_uint32
    lib.cm_stream_wait_call.argtypes = [P, ctypes.c_uint32, P]
    lib.cm_stream_wait_call.restype = ctypes.c_int
    lib.cm_key_idx_bits.argtypes = [ctypes.c_int64]
    lib.cm_key_idx_bits.restype = ctypes.c_int32
    lib.cm_decode_key.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_int64)]
    lib.cm_decode_key.restype = None
    lib.cm_decode_batch_key.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int64)]
    lib.cm_decode_batch_key.restype = None
    lib.cm_emit_plan.argtypes = [ctypes.c_int32, P, P, P, ctypes.c_int64, P, P, ctypes.c_int32, P,
                                 ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.cm_emit_plan.restype = ctypes.c_int
    lib.cm_plan_last_error.argtypes = []
    lib.cm_plan_last_error.restype = ctypes.c_char_p
    lib.cm_policy_checkpoints.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P, ctypes.c_int32, ctypes.c_int64, P]
    lib.cm_policy_checkpoints.restype = ctypes.c_int
    lib.cm_policy_sstar.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, P, ctypes.c_int64, P]
    lib.cm_policy_sstar.restype = ctypes.c_int
    lib.cm_policy_last_error.argtypes = []
    lib.cm_policy_last_error.restype = ctypes.c_char_p
    lib.cm_status_string.argtypes = [ctypes.c_int]
    lib.cm_status_string.restype = ctypes.c_char_p
    lib.cm_last_error.argtypes = []
    lib.cm_last_error.restype = ctypes.c_char_p
    # NVLS multicast buffers (a8 in the reduce step)
    lib.cm_mc_supported.argtypes = []
    lib.cm_mc_supported.restype = ctypes.c_int32
    lib.cm_mc_create.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(P)]
    lib.cm_mc_create.restype = ctypes.c_int
    lib.cm_mc_export_fd.argtypes = [P, ctypes.POINTER(ctypes.c_int32)]
    lib.cm_mc_export_fd.restype = ctypes.c_int
    lib.cm_mc_import_fd.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(P)]
    lib.cm_mc_import_fd.restype = ctypes.c_int
    lib.cm_mc_size.argtypes = [P]
    lib.cm_mc_size.restype = ctypes.c_int64
    lib.cm_mc_handle_type.argtypes = [P]
    lib.cm_mc_handle_type.restype = ctypes.c_int32
    lib.cm_mc_add_device.argtypes = [P]
    lib.cm_mc_add_device.restype = ctypes.c_int
    lib.cm_mc_bind.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P)]
    lib.cm_mc_bind.restype = ctypes.c_int
    lib.cm_mc_destroy.argtypes = [P]
    lib.cm_mc_destroy.restype = None
    lib.cm_mc_last_error.argtypes = []
    lib.cm_mc_last_error.restype = ctypes.c_char_p
    return lib
