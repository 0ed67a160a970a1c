"""Python mirror of the reference's operator API for the hot path.

The reference (``nestopt``) is a header-only C++ library; its hot-path API is
``ConvSpec``/``Layer``/``Network``/``Batch``/``FisherReport`` plus the free
functions ``reference_conv``, ``layer_forward``, ``forward``,
``activation_gradients``, ``fisher_potential``, ``fisher_accepts``,
``repair_network``, ``network_macs`` and ``evaluate_all``.  This module keeps
those names, argument meanings and error classes, and routes every
computation through the nb200 C ABI (include/nb200.h) to the sm_100a kernels.
There is no CPU fallback: without a B200 every compute call raises
``NoDevice``.

Citations: I/ = /root/reference/proj/include/nestopt/.
"""
from __future__ import annotations

import os

import ctypes as C
import sys
import threading
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi


# ---------------------------------------------------------------------------
# Errors (I/errors.hpp) -- one class per nb_status.

class Error(RuntimeError):
    """nestopt::Error (I/errors.hpp:8)."""


class InvalidSpec(Error): pass       # I/errors.hpp:11
class ConfigError(Error): pass       # I/errors.hpp:64
class ShapeMismatch(Error): pass     # I/errors.hpp:60
class CapExceeded(Error): pass       # I/errors.hpp:17
class TransformError(Error): pass    # I/errors.hpp:22
class ParseError(Error): pass        # I/errors.hpp:46
class IoError(Error): pass           # I/errors.hpp:67
class CudaError(Error): pass
class NoDevice(Error): pass
class OutOfMemory(Error): pass
class Unsupported(Error): pass


_STATUS = {1: InvalidSpec, 2: ConfigError, 3: ShapeMismatch, 4: CapExceeded,
           5: TransformError, 6: ParseError, 7: IoError, 8: Error, 100: CudaError,
           101: NoDevice, 102: OutOfMemory, 103: Unsupported, 199: Error}


def _check(status: int) -> None:
    if status != abi.NB_OK:
        msg = abi.load().nb_last_error().decode(errors="replace")
        raise _STATUS.get(status, Error)(msg)


def fp32_split() -> str:
    """The tensor-core split of the FP32 tier, as libnb200 reads it from the
    environment (engine.cu split_h16): "3xf16" (default), "3xbf16"
    (NB_TC_SPLIT=bf16) or "3xtf32" (NB_TC_SPLIT=tf32)."""
    e = os.environ.get("NB_TC_SPLIT")
    return {"tf32": "3xtf32", "bf16": "3xbf16"}.get(e, "3xf16")


class Precision:
    FP32 = abi.PREC_FP32   # 3xTF32 tensor cores (default; legality decisions)
    TF32 = abi.PREC_TF32   # 1xTF32 tensor-core throughput mode
    SIMT = abi.PREC_SIMT   # fp32 FFMA everywhere (fp32-faithful; near-tie rechecks)


# Stated tolerances against the fp64 reference, measured
# on the GPU: relative error of Fisher totals and per-layer values, and of
# conv outputs relative to sum |w||x|.  TOLERANCE holds for chains of up to
# ~10 layers (the reference's goldens, tests/test_gpu_parity.py);
# TOLERANCE_DEEP for the benchmarked 33-layer ResNet-34 chain at N=128
# (tests/test_r34_parity.py), where even true fp32 (SIMT) sits ~1e-4 from
# fp64: rounding flips ReLU masks of near-zero activations, and every flip
# re-routes gradient through 30 more layers (measured SIMT totals 1.4e-4,
# layers 7.3e-4; 3xTF32 8.0e-4 / 2.4e-3, biased low by the tensor core's
# truncating accumulation, profiles/r02_precision.md; TF32 3.0e-2 / 3.9e-2).
# RECHECK_BAND is the near-threshold band of the search driver: a candidate
# whose score is within it of the origin's is re-scored in SIMT mode before
# the accept decision (integration/nestopt_b200.hpp recheck_band, kept equal
# to these values): 2.5 x the deep total tolerance, since the candidate and
# the origin may each be off by it in opposite directions.
TOLERANCE = {
    Precision.SIMT: {"total": 1e-5, "layer": 1e-4, "conv": 2e-6},
    Precision.FP32: {"total": 5e-4, "layer": 5e-3, "conv": 1e-5},
    Precision.TF32: {"total": 5e-2, "layer": 2e-1, "conv": 2e-3},
}
TOLERANCE_DEEP = {
    Precision.SIMT: {"total": 3e-4, "layer": 1.5e-3},
    Precision.FP32: {"total": 1.5e-3, "layer": 5e-3},
    Precision.TF32: {"total": 5e-2, "layer": 2e-1},
}
RECHECK_BAND = {Precision.SIMT: 0.0, Precision.FP32: 3.75e-3, Precision.TF32: 1.25e-1}
# decisions closer than this to the origin may differ from the fp64
# reference even after the SIMT recheck (the documented near-threshold ties)
TIE_BAND = 2 * TOLERANCE_DEEP[Precision.SIMT]["total"]


# ---------------------------------------------------------------------------
# Descriptors

@dataclass
class ChannelSplit:
    """ChannelSplit, I/ir.hpp:20-24."""
    begin: int
    end: int
    groups: int = 1


@dataclass
class ConvSpec:
    """ConvSpec, I/ir.hpp:26-87."""
    ci: int = 1
    co: int = 1
    h: int = 1
    w: int = 1
    kh: int = 1
    kw: int = 1
    stride: int = 1
    pad: int = 0
    groups: int = 1
    bottleneck_out: int = 1
    spatial_div_h: int = 1
    spatial_div_w: int = 1
    channel_splits: List[ChannelSplit] = field(default_factory=list)

    def set_bottleneck_spatial(self, b: int) -> None:
        self.spatial_div_h = self.spatial_div_w = b

    def co_eff(self) -> int:
        return self.co // self.bottleneck_out

    def raw_out_h(self) -> int:
        return (self.h + 2 * self.pad - self.kh) // self.stride + 1

    def raw_out_w(self) -> int:
        return (self.w + 2 * self.pad - self.kw) // self.stride + 1

    def out_h(self) -> int:
        return self.raw_out_h() // self.spatial_div_h

    def out_w(self) -> int:
        return self.raw_out_w() // self.spatial_div_w

    def ranges(self) -> List[ChannelSplit]:
        if self.channel_splits:
            return list(self.channel_splits)
        return [ChannelSplit(0, self.co_eff(), self.groups)]

    def output_shape(self):
        return (self.co_eff(), self.out_h(), self.out_w())

    def validate(self) -> None:
        holder = _SpecHolder(self)
        _check(abi.load().nb_validate_spec(C.byref(holder.c)))

    # conv_spec_from_json / conv_spec_to_json, I/nnet.hpp:387-425
    @staticmethod
    def from_json(j: dict) -> "ConvSpec":
        s = ConvSpec(ci=j["ci"], co=j["co"], h=j["h"], w=j["w"], kh=j.get("kh", 1),
                     kw=j.get("kw", 1), stride=j.get("stride", 1), pad=j.get("pad", 0),
                     groups=j.get("groups", 1), bottleneck_out=j.get("bottleneck", 1),
                     spatial_div_h=j.get("spatial_div_h", 1),
                     spatial_div_w=j.get("spatial_div_w", 1),
                     channel_splits=[ChannelSplit(r["begin"], r["end"], r.get("groups", 1))
                                     for r in j.get("channel_splits", [])])
        s.validate()
        return s

    def to_json(self) -> dict:
        j = {"ci": self.ci, "co": self.co, "h": self.h, "w": self.w, "kh": self.kh,
             "kw": self.kw, "stride": self.stride, "pad": self.pad, "groups": self.groups,
             "bottleneck": self.bottleneck_out, "spatial_div_h": self.spatial_div_h,
             "spatial_div_w": self.spatial_div_w}
        if self.channel_splits:
            j["channel_splits"] = [{"begin": r.begin, "end": r.end, "groups": r.groups}
                                   for r in self.channel_splits]
        return j


class _SpecHolder:
    """Keeps a ConvSpecC and its split array alive."""

    def __init__(self, s: ConvSpec):
        self.splits = (abi.ChannelSplitC * max(1, len(s.channel_splits)))(
            *[abi.ChannelSplitC(r.begin, r.end, r.groups) for r in s.channel_splits])
        self.c = abi.ConvSpecC(s.ci, s.co, s.h, s.w, s.kh, s.kw, s.stride, s.pad, s.groups,
                               s.bottleneck_out, s.spatial_div_h, s.spatial_div_w,
                               len(s.channel_splits),
                               C.cast(self.splits, C.POINTER(abi.ChannelSplitC)))


@dataclass
class Layer:
    """Layer, I/nnet.hpp:23-26."""
    spec: ConvSpec
    relu: bool = True


class Network:
    """Network, I/nnet.hpp:28-79.

    ``weights``/``head`` stay ``None`` until ``init_weights()`` materialises
    them on the host; while they are ``None`` the device draws the reference's
    init_weights values itself (bit-identical), so candidates never pay for a
    host-side re-initialisation.
    """

    def __init__(self, layers: Sequence[Layer], num_classes: int = 10, seed: int = 0):
        self.layers = list(layers)
        self.num_classes = num_classes
        self.seed = seed
        self.weights: Optional[List[np.ndarray]] = None
        self.head: Optional[np.ndarray] = None

    def head_features(self) -> int:
        if not self.layers:
            raise ConfigError("network has no layers")
        return self.layers[-1].spec.co_eff()

    def c_struct(self) -> "_NetHolder":
        return _NetHolder(self)

    def validate(self) -> None:
        h = self.c_struct()
        _check(abi.load().nb_validate_network(C.byref(h.c)))

    def init_weights(self) -> None:
        """Network::init_weights, I/nnet.hpp:58-79 (host copies)."""
        h = self.c_struct()
        sizes = [l.spec.co_eff() * l.spec.ci * l.spec.kh * l.spec.kw for l in self.layers]
        flat = np.empty(sum(sizes), np.float64)
        head = np.empty(self.num_classes * self.head_features(), np.float64)
        _check(abi.load().nb_init_weights(C.byref(h.c), _dp(flat), _dp(head)))
        self.weights, off = [], 0
        for l, n in zip(self.layers, sizes):
            s = l.spec
            self.weights.append(flat[off:off + n].reshape(s.co_eff(), s.ci, s.kh, s.kw).copy())
            off += n
        self.head = head.reshape(self.num_classes, self.head_features())

    def copy(self) -> "Network":
        import copy as _c
        return _c.deepcopy(self)

    # network_from_json / network_to_json, I/nnet.hpp:427-454
    @staticmethod
    def from_json(j: dict, init: bool = False) -> "Network":
        if j.get("schema_version", 1) != 1:
            raise ConfigError("unsupported network schema version")
        net = Network([Layer(ConvSpec.from_json(lj), lj.get("relu", True)) for lj in j["layers"]],
                      num_classes=j.get("num_classes", 10), seed=j.get("seed", 0))
        net.validate()
        if init:
            net.init_weights()
        return net

    def to_json(self) -> dict:
        layers = []
        for l in self.layers:
            lj = l.spec.to_json()
            lj["relu"] = l.relu
            layers.append(lj)
        return {"schema_version": 1, "seed": self.seed, "num_classes": self.num_classes,
                "layers": layers}


class _NetHolder:
    def __init__(self, net: Network):
        self.specs = [_SpecHolder(l.spec) for l in net.layers]
        self.layers = (abi.LayerC * len(net.layers))(
            *[abi.LayerC(h.c, 1 if l.relu else 0, 0) for h, l in zip(self.specs, net.layers)])
        self.c = abi.NetworkC(len(net.layers), C.cast(self.layers, C.POINTER(abi.LayerC)),
                              net.num_classes, net.seed)
        self.w = None
        if net.weights is not None or net.head is not None:
            if net.weights is None or net.head is None:
                raise ConfigError("explicit weights need both layer weights and head")
            self._arrs = [np.ascontiguousarray(w, np.float64) for w in net.weights]
            for a, l in zip(self._arrs, net.layers):
                s = l.spec
                if a.shape != (s.co_eff(), s.ci, s.kh, s.kw):
                    raise ShapeMismatch("weight tensor shape does not match spec")
            self._head = np.ascontiguousarray(net.head, np.float64)
            if self._head.shape != (net.num_classes, net.head_features()):
                raise ShapeMismatch("head shape does not match the network")
            self._ptrs = (C.POINTER(C.c_double) * len(self._arrs))(*[_dp(a) for a in self._arrs])
            self.w = abi.WeightsC(C.cast(self._ptrs, C.POINTER(C.POINTER(C.c_double))),
                                  _dp(self._head))

    def wptr(self):
        return C.byref(self.w) if self.w is not None else None


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class Batch:
    """Batch, I/nnet.hpp:81-85: inputs (N, Ci, H, W) fp64, labels (N,)."""
    inputs: np.ndarray
    labels: np.ndarray
    seed: int = 0

    def __len__(self) -> int:
        return int(self.inputs.shape[0])

    def c_struct(self):
        x = np.ascontiguousarray(self.inputs, np.float64)
        y = np.ascontiguousarray(self.labels, np.int32)
        b = abi.BatchC(x.shape[0], _dp(x), y.ctypes.data_as(C.POINTER(C.c_int32)), self.seed)
        return b, (x, y)


def make_batch(net: Network, n: int, seed: int) -> Batch:
    """make_batch, I/nnet.hpp:87-101 (bit-identical draws)."""
    s0 = net.layers[0].spec
    x = np.empty((n, s0.ci, s0.h, s0.w), np.float64)
    y = np.empty(n, np.int32)
    h = net.c_struct()
    _check(abi.load().nb_make_batch(C.byref(h.c), n, seed, _dp(x),
                                    y.ctypes.data_as(C.POINTER(C.c_int32))))
    return Batch(x, y, seed)


@dataclass
class FisherReport:
    """FisherReport, I/nnet.hpp:272-277 (+ forward loss/probs)."""
    per_channel: List[np.ndarray]
    per_layer: np.ndarray
    total: float
    seed: int
    loss: float = float("nan")
    probs: Optional[np.ndarray] = None


@dataclass
class ForwardCache:
    """The outputs of forward (I/nnet.hpp:143-150) the GPU path returns."""
    probs: np.ndarray
    example_loss: np.ndarray
    loss: float


# ---------------------------------------------------------------------------
# Device contexts

class Context:
    """One nb_ctx (a GPU with its stream, arena and weight caches)."""

    def __init__(self, device: int = 0):
        lib = abi.load()
        p = C.c_void_p()
        _check(lib.nb_ctx_create(device, C.byref(p)))
        self.ptr = p
        self.device = device

    def close(self) -> None:
        if self.ptr:
            abi.load().nb_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on, every: int = 1) -> None:
        """Per-launch CUDA events (kernel_stats) on every `every`-th
        evaluation while `on`."""
        _check(abi.load().nb_ctx_set_profiling(self.ptr, max(1, int(every)) if on else 0))

    def reset_stats(self) -> None:
        _check(abi.load().nb_ctx_reset_stats(self.ptr))

    def clear_caches(self) -> None:
        """Drops the packed-weight and z-stream caches of this context."""
        _check(abi.load().nb_ctx_clear_caches(self.ptr))

    def kernel_stats(self) -> dict:
        arr = (abi.KernelStatC * 64)()
        n = C.c_int32()
        _check(abi.load().nb_ctx_kernel_stats(self.ptr, arr, 64, C.byref(n)))
        return {arr[i].name.decode(): {"launches": arr[i].launches, "ms": arr[i].ms,
                                       "flops": arr[i].flops, "bytes": arr[i].bytes}
                for i in range(min(n.value, 64))}

    def launch_count(self) -> int:
        return int(abi.load().nb_ctx_launch_count(self.ptr))

    def stream(self) -> int:
        return int(abi.load().nb_ctx_stream(self.ptr) or 0)


_default_ctx = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        if device not in _default_ctx:
            _default_ctx[device] = Context(device)
        return _default_ctx[device]


def device_count() -> int:
    return int(abi.load().nb_device_count())


# ---------------------------------------------------------------------------
# Hot-path functions

def _images(x: np.ndarray, shape3) -> np.ndarray:
    a = np.asarray(x, np.float64)
    if a.shape == tuple(shape3):
        a = a[None]
    if a.ndim != 4 or a.shape[1:] != tuple(shape3):
        raise ShapeMismatch("input tensor shape does not match spec")
    return np.ascontiguousarray(a)


def reference_conv(spec: ConvSpec, inputs: np.ndarray, weights: np.ndarray,
                   precision: int = Precision.FP32, ctx: Optional[Context] = None,
                   relu: bool = False) -> np.ndarray:
    """reference_conv (I/interp.hpp:151-186) on one image (C,H,W) or a batch
    (N,C,H,W); weights (Co_eff, Ci, Kh, Kw).  Returns fp64 (computed fp32)."""
    spec.validate()
    ctx = ctx or default_context()
    single = np.asarray(inputs).ndim == 3
    x = _images(inputs, (spec.ci, spec.h, spec.w))
    w = np.ascontiguousarray(weights, np.float64)
    if w.shape != (spec.co_eff(), spec.ci, spec.kh, spec.kw):
        raise ShapeMismatch("weight tensor shape does not match spec")
    y = np.empty((x.shape[0],) + spec.output_shape(), np.float64)
    h = _SpecHolder(spec)
    _check(abi.load().nb_conv_forward(ctx.ptr, C.byref(h.c), x.shape[0], _dp(x), _dp(w),
                                      _dp(y), 1 if relu else 0, precision))
    return y[0] if single else y


def layer_forward(layer: Layer, weights: np.ndarray, inputs: np.ndarray, **kw) -> np.ndarray:
    """layer_forward, I/nnet.hpp:130-141."""
    return reference_conv(layer.spec, inputs, weights, relu=layer.relu, **kw)


def conv_dgrad(spec: ConvSpec, dy: np.ndarray, weights: np.ndarray,
               precision: int = Precision.FP32, ctx: Optional[Context] = None) -> np.ndarray:
    """The dgrad MAC loop of activation_gradients (I/nnet.hpp:235-243)."""
    spec.validate()
    ctx = ctx or default_context()
    single = np.asarray(dy).ndim == 3
    g = _images(dy, spec.output_shape())
    w = np.ascontiguousarray(weights, np.float64)
    dx = np.empty((g.shape[0], spec.ci, spec.h, spec.w), np.float64)
    h = _SpecHolder(spec)
    _check(abi.load().nb_conv_dgrad(ctx.ptr, C.byref(h.c), g.shape[0], _dp(g), _dp(w),
                                    _dp(dx), precision))
    return dx[0] if single else dx


def forward(net: Network, batch: Batch, precision: int = Precision.FP32,
            ctx: Optional[Context] = None) -> ForwardCache:
    """forward, I/nnet.hpp:180-197."""
    ctx = ctx or default_context()
    h = net.c_struct()
    b, keep = batch.c_struct()
    n = len(batch)
    probs = np.empty((n, net.num_classes))
    ex = np.empty(n)
    loss = C.c_double()
    _check(abi.load().nb_forward(ctx.ptr, C.byref(h.c), h.wptr(), C.byref(b), precision,
                                 _dp(probs), _dp(ex), C.byref(loss)))
    return ForwardCache(probs, ex, loss.value)


def activation_gradients(net: Network, batch: Batch, precision: int = Precision.FP32,
                         ctx: Optional[Context] = None):
    """forward + activation_gradients (I/nnet.hpp:180-247).  Returns
    (acts, grads): per layer arrays (N, C, H, W) of the post-activation output
    and of dLoss/dOutput."""
    ctx = ctx or default_context()
    h = net.c_struct()
    b, keep = batch.c_struct()
    n = len(batch)
    shapes = [(n,) + l.spec.output_shape() for l in net.layers]
    total = sum(int(np.prod(s)) for s in shapes)
    acts = np.empty(total)
    grads = np.empty(total)
    _check(abi.load().nb_activation_gradients(ctx.ptr, C.byref(h.c), h.wptr(), C.byref(b),
                                              precision, _dp(acts), _dp(grads)))
    out_a, out_g, off = [], [], 0
    for s in shapes:
        k = int(np.prod(s))
        out_a.append(acts[off:off + k].reshape(s))
        out_g.append(grads[off:off + k].reshape(s))
        off += k
    return out_a, out_g


def _fisher_buffers(net: Network, n: int):
    ch = sum(l.spec.co_eff() for l in net.layers)
    per_channel = np.empty(ch)
    per_layer = np.empty(len(net.layers))
    probs = np.empty((n, net.num_classes))
    out = abi.FisherOutC(_dp(per_channel), _dp(per_layer), 0.0, 0, 0.0, _dp(probs))
    return out, per_channel, per_layer, probs


def _report(net: Network, out, per_channel, per_layer, probs) -> FisherReport:
    chans, off = [], 0
    for l in net.layers:
        c = l.spec.co_eff()
        chans.append(per_channel[off:off + c].copy())
        off += c
    return FisherReport(chans, per_layer.copy(), out.total, out.seed, out.loss, probs.copy())


def fisher_potential(net: Network, batch: Batch, precision: int = Precision.FP32,
                     ctx: Optional[Context] = None) -> FisherReport:
    """fisher_potential, I/nnet.hpp:321-352."""
    ctx = ctx or default_context()
    h = net.c_struct()
    b, keep = batch.c_struct()
    out, pc, pl, pr = _fisher_buffers(net, len(batch))
    _check(abi.load().nb_fisher_potential(ctx.ptr, C.byref(h.c), h.wptr(), C.byref(b),
                                          precision, C.byref(out)))
    return _report(net, out, pc, pl, pr)


def fisher_accepts(original: FisherReport, candidate: FisherReport) -> bool:
    """fisher_accepts, I/nnet.hpp:356-359: ties are accepted."""
    return candidate.total >= original.total


def legality_fisher(original: Network, candidate: Network, batch: Batch, **kw) -> bool:
    """legality_fisher, I/nnet.hpp:361-365."""
    return fisher_accepts(fisher_potential(original, batch, **kw),
                          fisher_potential(candidate, batch, **kw))


def repair_network(net: Network) -> None:
    """repair_network, I/nnet.hpp:372-382 (shape propagation; weights are
    re-drawn from the seed)."""
    for l in range(1, len(net.layers)):
        prev, cur = net.layers[l - 1].spec, net.layers[l].spec
        cur.ci, cur.h, cur.w = prev.co_eff(), prev.out_h(), prev.out_w()
    net.validate()
    net.weights = None
    net.head = None


def count_macs(spec: ConvSpec) -> int:
    """count_macs(conv_nest(spec)), I/interp.hpp:190-202."""
    h = _SpecHolder(spec)
    m = C.c_int64()
    _check(abi.load().nb_conv_macs(C.byref(h.c), C.byref(m)))
    return m.value


def network_macs(net: Network) -> int:
    """network_macs, I/search.hpp:84-88."""
    h = net.c_struct()
    m = C.c_int64()
    _check(abi.load().nb_network_macs(C.byref(h.c), C.byref(m)))
    return m.value


def fisher_flops(net: Network, n: int) -> float:
    h = net.c_struct()
    f = C.c_double()
    _check(abi.load().nb_fisher_flops(C.byref(h.c), n, C.byref(f)))
    return f.value


def schedule_lpt(costs: Sequence[float], bins: int) -> List[int]:
    c = np.ascontiguousarray(costs, np.float64)
    a = np.zeros(len(c), np.int32)
    _check(abi.load().nb_schedule_lpt(_dp(c), len(c), bins,
                                      a.ctypes.data_as(C.POINTER(C.c_int32))))
    return a.tolist()


# ---------------------------------------------------------------------------
# Sessions and the candidate scheduler

class Session:
    """A batch kept resident in one GPU's HBM (the search's fixed batch,
    I/search.hpp:371)."""

    def __init__(self, shape_net: Network, batch: Batch, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        h = shape_net.c_struct()
        b, keep = batch.c_struct()
        p = C.c_void_p()
        _check(abi.load().nb_session_create(self.ctx.ptr, C.byref(h.c), C.byref(b), C.byref(p)))
        self.ptr = p
        self.n = len(batch)
        self.seed = batch.seed

    def close(self):
        if self.ptr:
            abi.load().nb_session_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fisher(self, net: Network, precision: int = Precision.FP32) -> FisherReport:
        h = net.c_struct()
        out, pc, pl, pr = _fisher_buffers(net, self.n)
        _check(abi.load().nb_session_fisher(self.ptr, C.byref(h.c), h.wptr(), precision,
                                            C.byref(out)))
        return _report(net, out, pc, pl, pr)

    def forward(self, net: Network, precision: int = Precision.FP32):
        h = net.c_struct()
        probs = np.empty((self.n, net.num_classes))
        loss = C.c_double()
        _check(abi.load().nb_session_forward(self.ptr, C.byref(h.c), h.wptr(), precision,
                                             _dp(probs), C.byref(loss)))
        return probs, loss.value


def shard_batch(batch: Batch, count: int) -> List[Batch]:
    """Consecutive example slices of one batch (sizes differ by at most one),
    for nb_fisher_sharded."""
    n = len(batch)
    if not 1 <= count <= n:
        raise ConfigError(f"cannot split {n} examples into {count} shards")
    cuts = [n * i // count for i in range(count + 1)]
    return [Batch(batch.inputs[a:b], batch.labels[a:b], batch.seed)
            for a, b in zip(cuts[:-1], cuts[1:])]


def fisher_sharded(shards: Sequence[Session], net: Network,
                   precision: int = Precision.FP32) -> FisherReport:
    """fisher_potential (I/nnet.hpp:321-350) with the batch split over
    ``shards`` (sessions on distinct contexts -- normally one per GPU --
    holding consecutive slices of one batch, see shard_batch).  The report is
    bitwise that of one session holding the whole batch."""
    h = net.c_struct()
    out, pc, pl, pr = _fisher_buffers(net, sum(s.n for s in shards))
    sp = (C.c_void_p * len(shards))(*[s.ptr for s in shards])
    _check(abi.load().nb_fisher_sharded(sp, len(shards), C.byref(h.c), h.wptr(), precision,
                                        C.byref(out)))
    return _report(net, out, pc, pl, pr)


@dataclass
class EvalStats:
    evaluated: int
    deduplicated: int
    est_flops: List[float]    # per session: estimated FLOPs it ran
    busy_ms: List[float]      # per session: device time of its evaluations
    evaluations: List[int] = field(default_factory=list)  # per session
    requeued: int = 0         # evaluations handed back after a device failure
    failed_sessions: int = 0


def evaluate(sessions: Sequence[Session], nets: Sequence[Network],
             precision: int = Precision.FP32):
    """The candidate scheduler (evaluate_all, I/search.hpp:315-334): scores
    every network (init_weights draws) across the sessions' GPUs.  Returns
    (reports, EvalStats); reports[i] belongs to nets[i]."""
    _t0 = time.perf_counter()
    holders = [n.c_struct() for n in nets]
    for n in nets:
        if n.weights is not None:
            raise ConfigError("the scheduler scores init_weights networks only")
    arr = (abi.NetworkC * max(1, len(nets)))(*[h.c for h in holders])
    bufs = [_fisher_buffers(n, sessions[0].n) for n in nets]
    outs = (abi.FisherOutC * max(1, len(nets)))(*[b[0] for b in bufs])
    sp = (C.c_void_p * len(sessions))(*[s.ptr for s in sessions])
    est = np.zeros(len(sessions))
    busy = np.zeros(len(sessions))
    done = np.zeros(len(sessions), np.int64)
    st = abi.EvalStatsC(0, 0, 0, 0, 0, _dp(est), _dp(busy),
                        done.ctypes.data_as(C.POINTER(C.c_int64)))
    _t1 = time.perf_counter()
    _check(abi.load().nb_evaluate(sp, len(sessions), arr, len(nets), precision, outs,
                                  C.byref(st)))
    _t2 = time.perf_counter()
    reps = [_report(n, outs[i], b[1], b[2], b[3]) for i, (n, b) in enumerate(zip(nets, bufs))]
    if os.environ.get("NB_EVAL_LOG"):  # (experiments: host time around the C call)
        print(f"evaluate: prepare {1e3 * (_t1 - _t0):.1f} ms, nb_evaluate {1e3 * (_t2 - _t1):.1f} ms, "
              f"reports {1e3 * (time.perf_counter() - _t2):.1f} ms", file=sys.stderr, flush=True)
    return reps, EvalStats(st.evaluated, st.deduplicated, est.tolist(), busy.tolist(),
                           done.tolist(), st.requeued, st.failed_sessions)
