"""ctypes binding of the C-ABI in include/streamconv_b200.h (libstreamconv_b200.so).

The library is the product: every GPU computation of this package goes through it.  There is
no Python or CPU fallback — if the shared library is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["SC_LIB_PATH"]) if os.environ.get("SC_LIB_PATH") else PKG / "lib" / "libstreamconv_b200.so"

# streamconv::ErrCode (proj/include/streamconv/error.hpp:8-29); status = 1 + ordinal
ERR_NAMES = [
    "InvalidArgument", "InputTooShort", "ChannelMismatch", "CycleDetected", "DanglingNode",
    "RateMismatchAtSum", "MalformedGraph", "NotCausal", "PaddingNotStreamable",
    "InternalNonIntegerDelay", "BufferNotMultipleOfRatio", "LengthNotMultipleOfRatio",
    "ChunkTooSmall", "LengthMismatch", "ZeroEnergy", "VersionMismatch", "CorruptBlob",
    "SchemaError", "UnsupportedFormat", "MalformedHeader",
]

NODE_CONV, NODE_CONVT, NODE_ACT, NODE_RES_BEGIN, NODE_RES_END, NODE_GATE, NODE_SLICE = range(7)
ACT_IDENTITY, ACT_TANH, ACT_LEAKY_RELU = range(3)
PREC_FP32, PREC_BF16 = 0, 1
HINT_NONE, HINT_PQMF = 0, 1


class StreamconvError(RuntimeError):
    """Mirror of streamconv::Error (error.hpp:57-70): `.code` is the ErrCode name."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        if 1 <= status <= len(ERR_NAMES):
            self.code = ERR_NAMES[status - 1]
        elif status >= 1000:
            self.code = "CudaError"
        else:
            self.code = "UnknownError"


class SCNode(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("in_channels", C.c_int32), ("out_channels", C.c_int32),
        ("taps", C.c_int32), ("stride", C.c_int32), ("dilation", C.c_int32),
        ("pad_left", C.c_int64), ("pad_right", C.c_int64), ("act", C.c_int32),
        ("alpha", C.c_float), ("weight_offset", C.c_int64), ("slice_begin", C.c_int32),
        ("slice_count", C.c_int32), ("hint", C.c_int32),
    ]


(G_SOURCE, G_SINK, G_CONV, G_ZERO_UPSAMPLE, G_ACTIVATION, G_DELAY, G_SUM, G_FANOUT, G_GATE,
 G_SLICE) = range(10)
GKIND_NAMES = ["Source", "Sink", "Conv", "ZeroUpsample", "Activation", "Delay", "Sum", "Fanout",
               "Gate", "Slice"]


class SCGNode(C.Structure):
    """sc_gnode: one SPEC graph_ir node."""
    _fields_ = [
        ("kind", C.c_int32), ("in_channels", C.c_int32), ("out_channels", C.c_int32),
        ("taps", C.c_int32), ("stride", C.c_int32), ("dilation", C.c_int32),
        ("pad_left", C.c_int64), ("pad_right", C.c_int64), ("shift", C.c_int64),
        ("factor", C.c_int32), ("act", C.c_int32), ("alpha", C.c_float), ("arity", C.c_int32),
        ("samples", C.c_int64), ("weight_offset", C.c_int64), ("slice_begin", C.c_int32),
        ("slice_count", C.c_int32), ("hint", C.c_int32), ("inserted", C.c_int32),
    ]


class SCEdge(C.Structure):
    """sc_edge: (from, to, input port)."""
    _fields_ = [("from_", C.c_int32), ("to", C.c_int32), ("port", C.c_int32)]


_LIB = None

_SIGS = {
    "sc_last_error": (C.c_char_p, []),
    "sc_version": (C.c_char_p, []),
    "sc_status_name": (C.c_char_p, [C.c_int]),
    "sc_delay_for_stride": (C.c_int64, [C.c_int64, C.c_int64, C.c_int64]),
    "sc_branch_alignment": (C.c_int, [C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int64)]),
    "sc_plan_create": (C.c_int, [C.POINTER(SCNode), C.c_int32, C.POINTER(C.c_float), C.c_int64,
                                 C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "sc_plan_create_graph": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                       C.POINTER(C.c_float), C.c_int64, C.c_int32, C.c_int32,
                                       C.c_int32, C.POINTER(C.c_void_p)]),
    "sc_graph_validate": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                    C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "sc_graph_compression_ratio": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge),
                                             C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "sc_graph_receptive_field": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge),
                                           C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]),
    "sc_graph_causalize": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                     C.c_int32, C.POINTER(SCGNode), C.c_int32,
                                     C.POINTER(C.c_int32), C.POINTER(SCEdge), C.c_int32,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "sc_graph_mac_count": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                     C.c_int32, C.c_int64, C.POINTER(C.c_int64)]),
    "sc_graph_latency": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                   C.c_int32, C.POINTER(C.c_int64)]),
    "sc_model_load": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "sc_model_graph": (C.c_int, [C.c_void_p, C.POINTER(C.POINTER(SCGNode)), C.POINTER(C.c_int32),
                                 C.POINTER(C.POINTER(SCEdge)), C.POINTER(C.c_int32),
                                 C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int32)]),
    "sc_model_destroy": (C.c_int, [C.c_void_p]),
    "sc_model_save": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(SCGNode), C.c_int32,
                                C.POINTER(SCEdge), C.c_int32, C.POINTER(C.c_float), C.c_int64,
                                C.c_int32]),
    "sc_ola_create": (C.c_int, [C.POINTER(SCGNode), C.c_int32, C.POINTER(SCEdge), C.c_int32,
                                C.POINTER(C.c_float), C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.POINTER(C.c_void_p)]),
    "sc_ola_process": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "sc_ola_destroy": (C.c_int, [C.c_void_p]),
    "sc_ola_describe": (C.c_char_p, [C.c_void_p]),
    "sc_ola_window": (C.c_int, [C.c_int64, C.c_int32, C.POINTER(C.c_float)]),
    "sc_ola_redundancy": (C.c_double, [C.c_int32]),
    "sc_fidelity": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double),
                              C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]),
    "sc_best_lag": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                              C.POINTER(C.c_int64), C.c_void_p]),
    "sc_plan_destroy": (C.c_int, [C.c_void_p]),
    "sc_plan_ratio": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_plan_sink_rate": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32)]),
    "sc_plan_latency": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_plan_state_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_plan_macs_per_sample": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "sc_plan_describe": (C.c_char_p, [C.c_void_p]),
    "sc_plan_num_ops": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "sc_plan_op_macs": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double)]),
    "sc_state_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_void_p)]),
    "sc_state_destroy": (C.c_int, [C.c_void_p]),
    "sc_state_reset": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p]),
    "sc_state_device_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_state_cache_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_state_redzone_check": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_process": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "sc_process_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "sc_process_host_wait": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sc_process_host_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "sc_process_launches": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int32)]),
    "sc_state_launch_total": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "sc_state_set_graphs": (C.c_int, [C.c_void_p, C.c_int32]),
    "sc_state_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.POINTER(C.c_float), C.c_void_p]),
    "sc_launch_name": (C.c_char_p, [C.c_void_p, C.c_int64, C.c_int32]),
    "sc_conv1d": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                            C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "sc_conv_output_length": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
    "sc_pqmf_filters": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                  C.POINTER(C.c_float), C.POINTER(C.c_double)]),
}

EXPORTED = tuple(_SIGS)


def lib() -> C.CDLL:
    """Load the engine library (built in-tree by paper_2204_07064_b200.build)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -m paper_2204_07064_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            if os.environ.get("SC_LIB_PATH") and not hasattr(L, name):
                continue  # A/B experiments against an older build: newer entry points absent
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def check(status: int) -> None:
    if status != 0:
        msg = lib().sc_last_error().decode(errors="replace")
        raise StreamconvError(status, msg)
