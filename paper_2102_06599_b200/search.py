"""The GPU search driver (run_search, I/search.hpp:364) from Python.

It is the reference's own search pipeline -- draw_candidates, the semantic
legality gate, derived_spec, rank_survivors and the report writer, compiled
from the unmodified nestopt headers -- with fisher_potential / evaluate_all
replaced by the nb200 scheduler (integration/nestopt_b200.hpp), loaded from
integration/_build/libnb200_nestopt.so.  The report is the reference's
search_report_to_json schema plus a "gpu" block.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional

from . import abi
from .api import Precision, _STATUS, Error

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(os.path.dirname(_HERE), "integration", "_build", "libnb200_nestopt.so")
_lib: Optional[C.CDLL] = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise Error(f"nestopt integration library not built: {SO} (make -C integration)")
        abi.load()  # libnb200.so first (the integration library links it)
        lib = C.CDLL(SO)
        lib.nbi_last_error.restype = C.c_char_p
        lib.nbi_free.argtypes = [C.c_void_p]
        lib.nbi_run_search.restype = C.c_int
        lib.nbi_run_search.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_void_p)]
        lib.nbi_near_threshold.restype = C.c_int
        lib.nbi_near_threshold.argtypes = [C.c_double, C.c_double, C.c_int]
        lib.nbi_execute_boxes.restype = C.c_int
        lib.nbi_execute_boxes.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int,
                                          C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                          C.POINTER(C.c_longlong)]
        lib.nbi_execute.restype = C.c_int
        lib.nbi_execute.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        lib.nbi_gate_candidates.restype = C.c_int
        lib.nbi_gate_candidates.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        lib.nbi_legality_nests.restype = C.c_int
        lib.nbi_legality_nests.argtypes = [C.c_char_p, C.c_char_p, C.c_longlong, C.c_int,
                                           C.POINTER(C.c_double), C.POINTER(C.c_void_p)]
        lib.nbi_draw_candidates.restype = C.c_int
        lib.nbi_draw_candidates.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        lib.nbi_nest_json.restype = C.c_int
        lib.nbi_nest_json.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]
        lib.nbi_legality.restype = C.c_int
        lib.nbi_legality.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_longlong, C.c_int,
                                     C.POINTER(C.c_double), C.POINTER(C.c_void_p)]
        _lib = lib
    return _lib


def run_search_gpu(cfg: dict, devices: str = "0", precision: int = Precision.FP32,
                   jobs: int = 0) -> dict:
    """cfg: the reference's search config (schema v1) with an embedded
    "network" (P/samples/search_toy.json).  devices: comma-separated GPU
    indices, one session each (repeats allowed)."""
    lib = load()
    p = C.c_void_p()
    rc = lib.nbi_run_search(json.dumps(cfg).encode(), devices.encode(), int(precision),
                            int(jobs), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        return json.loads(C.cast(p, C.c_char_p).value.decode())
    finally:
        lib.nbi_free(p)


def near_threshold(cand: float, origin: float, precision: int) -> bool:
    """Whether the search driver re-scores this candidate in SIMT before the
    accept decision (integration/nestopt_b200.hpp near_threshold)."""
    return bool(load().nbi_near_threshold(cand, origin, int(precision)))


def gate_candidates(cfg: dict, legal_device: int = -1, with_counts: bool = False):
    """The host half of a search: the reference's draw_candidates and
    evaluate_candidate's gates (I/search.hpp:187-293).  legal_device >= 0
    checks semantic runs on that GPU (nb_semantic_legality), -1 (no GPU
    needed) with the reference's host check.  Returns one dict per
    candidate: status ("fisher" = a neural candidate that needs a Fisher
    score, else the reference's final status), reason, macs, and the
    repaired network JSON of "fisher" candidates.  with_counts: also return
    {"gpu": n, "host": m}, the semantic runs each side checked."""
    lib = load()
    p = C.c_void_p()
    rc = lib.nbi_gate_candidates(json.dumps(cfg).encode(), int(legal_device), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        out = json.loads(C.cast(p, C.c_char_p).value.decode())
        return (out["candidates"], out["legality"]) if with_counts else out["candidates"]
    finally:
        lib.nbi_free(p)


def legality(spec, seq: str, pre: str = "", cap: int = 1_000_000, device: int = -1):
    """check_semantic_legality (I/transforms.hpp:598-663) of the semantic run
    `seq` applied to conv_nest(spec) rewritten by `pre`: device -1 = the
    reference's host function, else the GPU check on that device (no host
    fallback).  Returns ({"verdict", "reason", "path": "gpu"|"host"} or
    {"error": "CapExceeded", "what"}, elapsed ms)."""
    lib = load()
    p = C.c_void_p()
    ms = C.c_double()
    sj = spec if isinstance(spec, dict) else spec.to_json()
    rc = lib.nbi_legality(json.dumps(sj).encode(), pre.encode(), seq.encode(), int(cap),
                          int(device), C.byref(ms), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        return json.loads(C.cast(p, C.c_char_p).value.decode()), ms.value
    finally:
        lib.nbi_free(p)


def legality_nests(original: dict, transformed: dict, cap: int = 1_000_000, device: int = -1):
    """check_semantic_legality of two explicit nests (nest JSON of
    nbi_nest_json: {"parts": [{"spine": [[name, extent, unroll, kernel]],
    "stmts": [...]}]}), e.g. the reference tests' hand-injected rewrites."""
    lib = load()
    p = C.c_void_p()
    ms = C.c_double()
    rc = lib.nbi_legality_nests(json.dumps(original).encode(), json.dumps(transformed).encode(),
                                int(cap), int(device), C.byref(ms), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        return json.loads(C.cast(p, C.c_char_p).value.decode()), ms.value
    finally:
        lib.nbi_free(p)


def draw_candidates(cfg: dict, threads: int = 0) -> list:
    """draw_candidates (I/search.hpp:188-214): threads 0 = the reference's
    serial loop, else the bridge's index-parallel version.  Returns per
    candidate {"neural", "layers": [DSL per layer]}."""
    lib = load()
    p = C.c_void_p()
    rc = lib.nbi_draw_candidates(json.dumps(cfg).encode(), int(threads), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        return json.loads(C.cast(p, C.c_char_p).value.decode())
    finally:
        lib.nbi_free(p)


def nest_json(spec, dsl: str = "") -> dict:
    """conv_nest(spec) (I/ir.hpp:427-470) rewritten by `dsl`, as nest JSON."""
    lib = load()
    p = C.c_void_p()
    sj = spec if isinstance(spec, dict) else spec.to_json()
    rc = lib.nbi_nest_json(json.dumps(sj).encode(), dsl.encode(), C.byref(p))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    try:
        return json.loads(C.cast(p, C.c_char_p).value.decode())
    finally:
        lib.nbi_free(p)


def execute_gpu(spec, dsl: str, x, w):
    """execute (I/interp.hpp:67-145) on the GPU of conv_nest(spec) rewritten
    by the DSL sequence `dsl` -- any rewritten nest, including those with no
    ConvSpec such as the paper's Sequence 1.  Integer inputs run in int64
    (exact), floating inputs in fp64.  Returns (Co_eff, out_h, out_w)."""
    import numpy as np
    lib = load()
    is_int = np.asarray(x).dtype.kind in "iu"
    dt = np.int64 if is_int else np.float64
    x = np.ascontiguousarray(x, dt)
    w = np.ascontiguousarray(w, dt)
    y = np.zeros(spec.output_shape(), dt)
    rc = lib.nbi_execute(json.dumps(spec.to_json()).encode(), dsl.encode(), int(is_int),
                         x.ctypes.data, w.ctypes.data, y.ctypes.data)
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    return y


def execute_boxes_gpu(spec, dsl: str, x, w, precision: int = None):
    """The masked box executor (integration/nestopt_b200.hpp execute_boxes):
    execute (I/interp.hpp:67-145) of conv_nest(spec) rewritten by `dsl` as
    tensor-core implicit GEMMs over (output-channel range x row band x
    input-channel range) boxes found by a GPU cell pass.  Integer inputs
    come back as int64 (exact while sums stay small), floating ones as
    float64 within the precision tier's tolerance.  Returns (y, stats) with
    stats = {"boxes", "box_macs", "nest_macs"}; raises Unsupported for a
    nest that does not decompose into boxes."""
    import numpy as np
    from .api import Precision
    lib = load()
    prec = Precision.FP32 if precision is None else precision
    is_int = np.asarray(x).dtype.kind in "iu"
    dt = np.int64 if is_int else np.float64
    x = np.ascontiguousarray(x, dt)
    w = np.ascontiguousarray(w, dt)
    y = np.zeros(spec.output_shape(), dt)
    nb_, bm, nm = C.c_longlong(), C.c_longlong(), C.c_longlong()
    rc = lib.nbi_execute_boxes(json.dumps(spec.to_json()).encode(), dsl.encode(), int(is_int),
                               x.ctypes.data, w.ctypes.data, y.ctypes.data, int(prec),
                               C.byref(nb_), C.byref(bm), C.byref(nm))
    if rc != 0:
        raise _STATUS.get(rc, Error)(lib.nbi_last_error().decode(errors="replace"))
    return y, {"boxes": nb_.value, "box_macs": bm.value, "nest_macs": nm.value}
