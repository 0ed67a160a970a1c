"""ctypes view of the nb200 C ABI (include/nb200.h).

The shared library is built in-tree (``paper_2102_06599_b200/libnb200.so``,
see ``Makefile`` / ``__graft_entry__.build``).  There is no fallback: if the
library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnb200.so")
# A/B experiments only: load another in-tree build of the same ABI
if os.environ.get("NB200_LIB"):
    LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ["NB200_LIB"])

# nb_status (include/nb200.h) -- values map 1:1 onto nestopt exception classes.
NB_OK = 0
STATUS_NAMES = {
    1: "InvalidSpec", 2: "ConfigError", 3: "ShapeMismatch", 4: "CapExceeded",
    5: "TransformError", 6: "ParseError", 7: "IoError", 8: "Error",
    100: "CudaError", 101: "NoDevice", 102: "OutOfMemory", 103: "Unsupported",
    199: "InternalError",
}

PREC_FP32, PREC_TF32, PREC_SIMT = 0, 1, 2


class ChannelSplitC(C.Structure):
    _fields_ = [("begin", C.c_int64), ("end", C.c_int64), ("groups", C.c_int64)]


class ConvSpecC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "ci", "co", "h", "w", "kh", "kw", "stride", "pad", "groups",
        "bottleneck_out", "spatial_div_h", "spatial_div_w", "num_splits")] + [
        ("splits", C.POINTER(ChannelSplitC))]


class LayerC(C.Structure):
    _fields_ = [("spec", ConvSpecC), ("relu", C.c_int32), ("reserved", C.c_int32)]


class NetworkC(C.Structure):
    _fields_ = [("num_layers", C.c_int64), ("layers", C.POINTER(LayerC)),
                ("num_classes", C.c_int64), ("seed", C.c_uint64)]


class WeightsC(C.Structure):
    _fields_ = [("layer", C.POINTER(C.POINTER(C.c_double))), ("head", C.POINTER(C.c_double))]


class BatchC(C.Structure):
    _fields_ = [("n", C.c_int64), ("inputs", C.POINTER(C.c_double)),
                ("labels", C.POINTER(C.c_int32)), ("seed", C.c_uint64)]


class FisherOutC(C.Structure):
    _fields_ = [("per_channel", C.POINTER(C.c_double)), ("per_layer", C.POINTER(C.c_double)),
                ("total", C.c_double), ("seed", C.c_uint64), ("loss", C.c_double),
                ("probs", C.POINTER(C.c_double))]


class KernelStatC(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


class EvalStatsC(C.Structure):
    _fields_ = [("evaluated", C.c_int64), ("deduplicated", C.c_int64),
                ("requeued", C.c_int64), ("failed_sessions", C.c_int32),
                ("reserved", C.c_int32), ("est_flops", C.POINTER(C.c_double)),
                ("busy_ms", C.POINTER(C.c_double)), ("evaluations", C.POINTER(C.c_int64))]


P = C.POINTER
vp = C.c_void_p
dp = P(C.c_double)

# name -> (restype, argtypes); the exported symbol set of include/nb200.h.
class NestExprC(C.Structure):
    _fields_ = [("nops", C.c_int32), ("code", C.POINTER(C.c_int64))]


class NestAccessC(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("zero_pad", C.c_int32), ("rank", C.c_int32),
                ("idx", C.POINTER(NestExprC))]


class NestStmtC(C.Structure):
    _fields_ = [("depth", C.c_int32), ("extents", C.POINTER(C.c_int64)),
                ("ndomain", C.c_int32), ("coord", C.POINTER(NestExprC)),
                ("naccess", C.c_int32), ("access", C.POINTER(NestAccessC))]


class LegalAccessC(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("mode", C.c_int32), ("rank", C.c_int32),
                ("idx", C.POINTER(NestExprC)), ("lo", C.POINTER(C.c_int64)),
                ("hi", C.POINTER(C.c_int64))]


class LegalStmtC(C.Structure):
    _fields_ = [("sid", C.c_int32), ("gid", C.c_int32), ("depth", C.c_int32),
                ("extents", C.POINTER(C.c_int64)), ("rank_base", C.c_int64),
                ("rank_stride", C.POINTER(C.c_int64)), ("ndomain", C.c_int32),
                ("coord", C.POINTER(NestExprC)), ("lo", C.POINTER(C.c_int64)),
                ("hi", C.POINTER(C.c_int64)), ("naccess", C.c_int32),
                ("access", C.POINTER(LegalAccessC))]


class LegalNestC(C.Structure):
    _fields_ = [("num_stmts", C.c_int64), ("stmts", C.POINTER(LegalStmtC))]


class LegalOutC(C.Structure):
    _fields_ = [("verdict", C.c_int32), ("src_inst", C.c_int64), ("dst_inst", C.c_int64),
                ("src_stmt", C.c_int32), ("dst_stmt", C.c_int32),
                ("src_coord", C.c_int64 * 8), ("dst_coord", C.c_int64 * 8), ("pairs", C.c_int64)]


class NestC(C.Structure):
    _fields_ = [("num_stmts", C.c_int64), ("stmts", C.POINTER(NestStmtC)),
                ("out_shape", C.c_int64 * 4), ("in_shape", C.c_int64 * 4),
                ("w_shape", C.c_int64 * 4), ("out_rank", C.c_int32), ("in_rank", C.c_int32),
                ("w_rank", C.c_int32)]


SIGNATURES = {
    "nb_version": (C.c_char_p, []),
    "nb_abi_version": (C.c_int, []),
    "nb_device_count": (C.c_int, []),
    "nb_last_error": (C.c_char_p, []),
    "nb_validate_spec": (C.c_int, [P(ConvSpecC)]),
    "nb_validate_network": (C.c_int, [P(NetworkC)]),
    "nb_conv_macs": (C.c_int, [P(ConvSpecC), P(C.c_int64)]),
    "nb_network_macs": (C.c_int, [P(NetworkC), P(C.c_int64)]),
    "nb_repair_network": (C.c_int, [C.c_int64, P(LayerC)]),
    "nb_schedule_lpt": (C.c_int, [dp, C.c_int64, C.c_int32, P(C.c_int32)]),
    "nb_fisher_flops": (C.c_int, [P(NetworkC), C.c_int64, dp]),
    "nb_init_weights": (C.c_int, [P(NetworkC), dp, dp]),
    "nb_make_batch": (C.c_int, [P(NetworkC), C.c_int64, C.c_uint64, dp, P(C.c_int32)]),
    "nb_ctx_create": (C.c_int, [C.c_int, P(vp)]),
    "nb_ctx_destroy": (C.c_int, [vp]),
    "nb_ctx_stream": (vp, [vp]),
    "nb_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
    "nb_ctx_kernel_stats": (C.c_int, [vp, P(KernelStatC), C.c_int32, P(C.c_int32)]),
    "nb_ctx_reset_stats": (C.c_int, [vp]),
    "nb_ctx_clear_caches": (C.c_int, [vp]),
    "nb_ctx_launch_count": (C.c_int64, [vp]),
    "nb_conv_forward": (C.c_int, [vp, P(ConvSpecC), C.c_int64, dp, dp, dp, C.c_int32, C.c_int]),
    "nb_conv_dgrad": (C.c_int, [vp, P(ConvSpecC), C.c_int64, dp, dp, dp, C.c_int]),
    "nb_nest_execute": (C.c_int, [vp, P(NestC), C.c_int32, vp, vp, vp]),
    "nb_nest_cells": (C.c_int, [vp, P(NestC), P(C.c_int32), P(C.c_int32), P(C.c_int64)]),
    "nb_conv_band": (C.c_int, [vp, P(ConvSpecC), C.c_int64, dp, dp, C.c_int32, C.c_int32, dp,
                               C.c_int]),
    "nb_semantic_legality": (C.c_int, [vp, P(LegalNestC), P(LegalNestC), P(LegalOutC)]),
    "nb_ctx_device": (C.c_int, [vp]),
    "nb_forward": (C.c_int, [vp, P(NetworkC), P(WeightsC), P(BatchC), C.c_int, dp, dp, dp]),
    "nb_activation_gradients": (C.c_int, [vp, P(NetworkC), P(WeightsC), P(BatchC), C.c_int,
                                          dp, dp]),
    "nb_fisher_potential": (C.c_int, [vp, P(NetworkC), P(WeightsC), P(BatchC), C.c_int,
                                      P(FisherOutC)]),
    "nb_fisher_accepts": (C.c_int, [P(FisherOutC), P(FisherOutC)]),
    "nb_session_create": (C.c_int, [vp, P(NetworkC), P(BatchC), P(vp)]),
    "nb_session_destroy": (C.c_int, [vp]),
    "nb_session_ctx": (vp, [vp]),
    "nb_session_fisher": (C.c_int, [vp, P(NetworkC), P(WeightsC), C.c_int, P(FisherOutC)]),
    "nb_session_forward": (C.c_int, [vp, P(NetworkC), P(WeightsC), C.c_int, dp, dp]),
    "nb_fisher_sharded": (C.c_int, [P(vp), C.c_int32, P(NetworkC), P(WeightsC), C.c_int,
                                    P(FisherOutC)]),
    "nb_evaluate": (C.c_int, [P(vp), C.c_int32, P(NetworkC), C.c_int64, C.c_int,
                              P(FisherOutC), P(EvalStatsC)]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libnb200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"nb200 native library missing at {LIB_PATH}: run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
