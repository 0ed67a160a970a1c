"""TEST INFRASTRUCTURE ONLY: Python bindings of the parity checker.

* ``Restatement`` -- oracle/_build/libnb_oracle.so, our CPU restatement of the
  reference's fp64 engine (oracle/nb_oracle.cpp); it takes the same nb200.h
  descriptors as the product.
* ``Reference`` -- oracle/_ref/libnestopt_ref.so, the UNMODIFIED reference
  (nestopt headers compiled in place by oracle/Makefile) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
legs may use this module, and only as the checker / baseline.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from paper_2102_06599_b200 import abi
from paper_2102_06599_b200.api import Network, _dp

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libnb_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnestopt_ref.so")

P = C.POINTER
dp = P(C.c_double)


class OracleError(RuntimeError):
    pass


class Restatement:
    """fp64 restatement of I/nnet.hpp + I/interp.hpp (oracle/nb_oracle.cpp)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise OracleError(f"oracle not built: {path} (make -C oracle)")
        lib = C.CDLL(path)
        lib.orc_last_error.restype = C.c_char_p
        for name, args in {
            "orc_validate_spec": [P(abi.ConvSpecC)],
            "orc_init_weights": [P(abi.NetworkC), dp, dp],
            "orc_make_batch": [P(abi.NetworkC), C.c_int64, C.c_uint64, dp, P(C.c_int32)],
            "orc_conv": [P(abi.ConvSpecC), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p],
            "orc_conv_dgrad": [P(abi.ConvSpecC), dp, dp, dp],
            "orc_fisher": [P(abi.NetworkC), P(abi.WeightsC), P(abi.BatchC), P(abi.FisherOutC),
                           dp, dp],
            "orc_forward": [P(abi.NetworkC), P(abi.WeightsC), P(abi.BatchC), dp, dp],
        }.items():
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = args
        self.lib = lib

    def _ok(self, rc):
        if rc != 0:
            raise OracleError(self.lib.orc_last_error().decode())

    def conv(self, spec, x, w):
        from paper_2102_06599_b200.api import _SpecHolder
        is_int = np.asarray(x).dtype.kind in "iu"
        dt = np.int64 if is_int else np.float64
        x = np.ascontiguousarray(x, dt)
        w = np.ascontiguousarray(w, dt)
        y = np.zeros(spec.output_shape(), dt)
        h = _SpecHolder(spec)
        self._ok(self.lib.orc_conv(C.byref(h.c), int(is_int), x.ctypes.data, w.ctypes.data,
                                   y.ctypes.data))
        return y

    def conv_dgrad(self, spec, dy, w):
        from paper_2102_06599_b200.api import _SpecHolder
        dy = np.ascontiguousarray(dy, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        dx = np.zeros((spec.ci, spec.h, spec.w))
        h = _SpecHolder(spec)
        self._ok(self.lib.orc_conv_dgrad(C.byref(h.c), _dp(dy), _dp(w), _dp(dx)))
        return dx

    def fisher(self, net: Network, n: int, batch_seed: int = 1, batch=None, grads=False):
        """Returns dict(per_channel, per_layer, total, loss, probs[, acts, grads])."""
        h = net.c_struct()
        if batch is not None:
            b, keep = batch.c_struct()
            n = len(batch)
        else:
            b = abi.BatchC(n, None, None, batch_seed)
        ch = sum(l.spec.co_eff() for l in net.layers)
        pc, pl, pr = np.empty(ch), np.empty(len(net.layers)), np.empty((n, net.num_classes))
        out = abi.FisherOutC(_dp(pc), _dp(pl), 0.0, 0, 0.0, _dp(pr))
        acts = grd = None
        if grads:
            tot = n * sum(int(np.prod(l.spec.output_shape())) for l in net.layers)
            acts, grd = np.empty(tot), np.empty(tot)
        self._ok(self.lib.orc_fisher(C.byref(h.c), h.wptr(), C.byref(b), C.byref(out),
                                     _dp(acts), _dp(grd)))
        r = dict(per_channel=pc, per_layer=pl, total=out.total, loss=out.loss, probs=pr)
        if grads:
            r["acts"], r["grads"] = acts, grd
        return r

    def make_batch(self, net: Network, n: int, seed: int):
        s0 = net.layers[0].spec
        x = np.empty((n, s0.ci, s0.h, s0.w))
        y = np.empty(n, np.int32)
        h = net.c_struct()
        self._ok(self.lib.orc_make_batch(C.byref(h.c), n, seed, _dp(x),
                                         y.ctypes.data_as(P(C.c_int32))))
        return x, y

    def init_weights(self, net: Network):
        sizes = [l.spec.co_eff() * l.spec.ci * l.spec.kh * l.spec.kw for l in net.layers]
        w = np.empty(sum(sizes))
        hd = np.empty(net.num_classes * net.head_features())
        h = net.c_struct()
        self._ok(self.lib.orc_init_weights(C.byref(h.c), _dp(w), _dp(hd)))
        return w, hd


class Reference:
    """The unmodified reference library (oracle/_ref/libnestopt_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"reference shim not built: {path} (make -C oracle)")
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_free.argtypes = [C.c_void_p]
        sig = {
            "ref_init_weights": [C.c_char_p, dp, dp],
            "ref_make_batch": [C.c_char_p, C.c_int64, C.c_uint64, dp, P(C.c_int32)],
            "ref_fisher": [C.c_char_p, dp, dp, C.c_int64, dp, P(C.c_int32), C.c_uint64, dp,
                           dp, dp, dp, dp, dp, dp],
            "ref_forward": [C.c_char_p, C.c_int64, C.c_uint64, dp, dp, dp],
            "ref_conv": [C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p],
            "ref_layer_forward": [C.c_char_p, C.c_int, dp, dp, dp],
            "ref_execute": [C.c_char_p, C.c_char_p, C.c_int, C.c_void_p, C.c_void_p,
                            C.c_void_p],
            "ref_count_macs": [C.c_char_p, C.c_char_p, P(C.c_int64)],
            "ref_derived_spec": [C.c_char_p, C.c_char_p, P(C.c_void_p)],
            "ref_search": [C.c_char_p, C.c_int, P(C.c_void_p)],
        }
        for name, args in sig.items():
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = args
        self.lib = lib

    def _ok(self, rc):
        if rc != 0:
            raise OracleError(f"[{rc}] " + self.lib.ref_last_error().decode())

    def _str(self, fn, *args) -> str:
        p = C.c_void_p()
        self._ok(fn(*args, C.byref(p)))
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.ref_free(p)
        return s

    @staticmethod
    def _j(obj) -> bytes:
        return json.dumps(obj if isinstance(obj, dict) else obj.to_json()).encode()

    def fisher(self, net: Network, n: int, batch_seed: int = 1, batch=None, grads=False,
               explicit_weights=False):
        js = self._j(net)
        x = y = None
        if batch is not None:
            x = np.ascontiguousarray(batch.inputs, np.float64)
            y = np.ascontiguousarray(batch.labels, np.int32)
            n = x.shape[0]
            batch_seed = batch.seed
        wflat = head = None
        if explicit_weights:
            wflat = np.concatenate([np.ravel(w) for w in net.weights])
            head = np.ascontiguousarray(net.head, np.float64).ravel()
        ch = sum(l.spec.co_eff() for l in net.layers)
        pc, pl, pr = np.empty(ch), np.empty(len(net.layers)), np.empty((n, net.num_classes))
        tot, loss = C.c_double(), C.c_double()
        acts = grd = None
        if grads:
            t = n * sum(int(np.prod(l.spec.output_shape())) for l in net.layers)
            acts, grd = np.empty(t), np.empty(t)
        self._ok(self.lib.ref_fisher(js, _dp(wflat), _dp(head), n, _dp(x),
                                     None if y is None else y.ctypes.data_as(P(C.c_int32)),
                                     batch_seed, _dp(pc), _dp(pl), C.byref(tot),
                                     C.byref(loss), _dp(pr), _dp(acts), _dp(grd)))
        r = dict(per_channel=pc, per_layer=pl, total=tot.value, loss=loss.value, probs=pr)
        if grads:
            r["acts"], r["grads"] = acts, grd
        return r

    def make_batch(self, net: Network, n: int, seed: int):
        s0 = net.layers[0].spec
        x = np.empty((n, s0.ci, s0.h, s0.w))
        y = np.empty(n, np.int32)
        self._ok(self.lib.ref_make_batch(self._j(net), n, seed, _dp(x),
                                         y.ctypes.data_as(P(C.c_int32))))
        return x, y

    def init_weights(self, net: Network):
        sizes = [l.spec.co_eff() * l.spec.ci * l.spec.kh * l.spec.kw for l in net.layers]
        w = np.empty(sum(sizes))
        hd = np.empty(net.num_classes * net.head_features())
        self._ok(self.lib.ref_init_weights(self._j(net), _dp(w), _dp(hd)))
        return w, hd

    def conv(self, spec, x, w):
        is_int = np.asarray(x).dtype.kind in "iu"
        dt = np.int64 if is_int else np.float64
        x = np.ascontiguousarray(x, dt)
        w = np.ascontiguousarray(w, dt)
        y = np.zeros(spec.output_shape(), dt)
        self._ok(self.lib.ref_conv(self._j(spec), int(is_int), x.ctypes.data, w.ctypes.data,
                                   y.ctypes.data))
        return y

    def execute(self, spec, dsl: str, x, w):
        is_int = np.asarray(x).dtype.kind in "iu"
        dt = np.int64 if is_int else np.float64
        x = np.ascontiguousarray(x, dt)
        w = np.ascontiguousarray(w, dt)
        y = np.zeros(spec.output_shape(), dt)
        self._ok(self.lib.ref_execute(self._j(spec), dsl.encode(), int(is_int), x.ctypes.data,
                                      w.ctypes.data, y.ctypes.data))
        return y

    def count_macs(self, spec, dsl: str = "") -> int:
        m = C.c_int64()
        self._ok(self.lib.ref_count_macs(self._j(spec), dsl.encode(), C.byref(m)))
        return m.value

    def derived_spec(self, spec, dsl: str):
        return json.loads(self._str(self.lib.ref_derived_spec, self._j(spec), dsl.encode()))

    def search(self, cfg: dict, jobs: int = 0) -> dict:
        return json.loads(self._str(self.lib.ref_search, json.dumps(cfg).encode(), jobs))
