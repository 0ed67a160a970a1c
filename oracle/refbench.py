"""BENCH BASELINE ONLY: the reference CPU path of bench.py.

Runs the UNMODIFIED reference (oracle/_ref/libnestopt_ref.so, compiled in
place from /root/reference by oracle/Makefile) on the bench's candidate pool
without importing or loading the nb200 product: the pool is rebuilt from
tests/golden/r34_candidates.json in plain Python (repair_network's shape
propagation, I/nnet.hpp:372-380), and the timing entry point is
ref_fisher_jobs (oracle/ref_shim.cpp), i.e. evaluate_all's own thread pool
(I/search.hpp:315-334) running fisher_potential (I/nnet.hpp:321).

Only bench.py (its --impl reference arm and its cpu_baseline leg) uses this
module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import List, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_SO = os.path.join(HERE, "_ref", "libnestopt_ref.so")
POOL = os.path.join(ROOT, "tests", "golden", "r34_candidates.json")


def _out(l: dict) -> Tuple[int, int, int]:
    """(co_eff, out_h, out_w) of a layer JSON (ConvSpec, I/ir.hpp:40-50)."""
    p, k, s = l.get("pad", 0), (l.get("kh", 1), l.get("kw", 1)), l.get("stride", 1)
    oh = ((l["h"] + 2 * p - k[0]) // s + 1) // l.get("spatial_div_h", 1)
    ow = ((l["w"] + 2 * p - k[1]) // s + 1) // l.get("spatial_div_w", 1)
    return l["co"] // l.get("bottleneck", 1), oh, ow


def rebuild(origin: dict, diff) -> dict:
    """The origin network JSON with layer diff[0] replaced by diff[1] and the
    downstream shapes repaired (repair_network, I/nnet.hpp:372-380)."""
    layers = [dict(l) for l in origin["layers"]]
    layers[diff[0]] = dict(diff[1])
    for l in range(1, len(layers)):
        layers[l]["ci"], layers[l]["h"], layers[l]["w"] = _out(layers[l - 1])
    return dict(origin, layers=layers)


def layer_macs(l: dict) -> int:
    """count_macs(conv_nest(spec)) (I/interp.hpp:190-202): padded taps
    included, summed over the channel ranges."""
    co_eff, oh, ow = _out(l)
    ranges = l.get("channel_splits") or [{"begin": 0, "end": co_eff,
                                          "groups": l.get("groups", 1)}]
    return sum((r["end"] - r["begin"]) * oh * ow * (l["ci"] // r.get("groups", 1))
               * l.get("kh", 1) * l.get("kw", 1) for r in ranges)


def fisher_macs(net: dict, n: int) -> int:
    """fprop of every layer + dgrad of layers >= 1 (I/nnet.hpp:225), x n."""
    m = [layer_macs(l) for l in net["layers"]]
    return n * (sum(m) + sum(m[1:]))


def bench_pool(steps: int, warmup: int, world: int):
    """The bench's candidate selection (both arms use it): the reference's
    R34 per-layer pool in a fixed shuffled order; the first max(1, W) are the
    warm-up networks, the next K x world the timed ones.  Returns (origin,
    warm, timed) as network JSON dicts."""
    data = json.load(open(POOL))
    origin = data["origin"]
    pool = [rebuild(origin, c["diff"]) for c in data["candidates"]]
    order = np.random.default_rng(0).permutation(len(pool))
    pool = [pool[i] for i in order]
    warm = pool[:max(1, warmup)]
    timed = pool[len(warm):]
    need = steps * world
    if need > len(timed):
        raise SystemExit(f"--steps x gpus = {need} exceeds the {len(timed)} distinct candidates")
    return origin, warm, timed[:need], timed[need:]


class RefArm:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"reference library not built: {path} (make -C oracle)")
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        P = C.POINTER
        lib.ref_fisher_jobs.restype = C.c_int
        lib.ref_fisher_jobs.argtypes = [P(C.c_char_p), C.c_int, C.c_int64, C.c_uint64, C.c_int,
                                        P(C.c_double), P(C.c_double), P(C.c_double)]
        lib.ref_layer_forward.restype = C.c_int
        lib.ref_layer_forward.argtypes = [C.c_char_p, C.c_int, P(C.c_double), P(C.c_double),
                                          P(C.c_double)]
        self.lib = lib

    def fisher_jobs(self, nets: List[dict], n: int, jobs: int, batch_seed: int = 1):
        """fisher_potential of every network at batch size n on `jobs`
        threads (evaluate_all's scheduler).  Returns (totals, per-job
        seconds, wall seconds)."""
        enc = [json.dumps(x).encode() for x in nets]
        arr = (C.c_char_p * len(enc))(*enc)
        tot = (C.c_double * len(enc))()
        sec = (C.c_double * len(enc))()
        wall = C.c_double()
        rc = self.lib.ref_fisher_jobs(arr, len(enc), n, batch_seed, jobs, tot, sec,
                                      C.byref(wall))
        if rc != 0:
            raise RuntimeError(f"reference: {self.lib.ref_last_error().decode()}")
        return list(tot), list(sec), wall.value

    def layer_forward_seconds(self, layer: dict, reps: int = 1) -> float:
        """Time of the reference's layer_forward (I/nnet.hpp:130-141) on one
        image of the layer's input shape."""
        import time
        x = np.random.default_rng(0).standard_normal(layer["ci"] * layer["h"] * layer["w"])
        co, oh, ow = _out(layer)
        w = np.random.default_rng(1).standard_normal(
            co * layer["ci"] * layer.get("kh", 1) * layer.get("kw", 1))
        y = np.empty(co * oh * ow)
        dp = C.POINTER(C.c_double)
        js = json.dumps(layer).encode()
        t = time.perf_counter()
        for _ in range(reps):
            rc = self.lib.ref_layer_forward(js, 1, x.ctypes.data_as(dp), w.ctypes.data_as(dp),
                                            y.ctypes.data_as(dp))
            if rc != 0:
                raise RuntimeError(f"reference: {self.lib.ref_last_error().decode()}")
        return (time.perf_counter() - t) / reps


def slices(net: dict, parts: int) -> List[Tuple[int, int]]:
    """Contiguous layer slices [a, b] balanced by Fisher MACs; every slice
    but the first starts one layer early (its layer a-1 is forward-only), so
    the slices together run every layer's forward and every dgrad of the
    whole network (activation_gradients' l >= 1 loop, I/nnet.hpp:225-243)."""
    L = len(net["layers"])
    m = [layer_macs(l) for l in net["layers"]]
    cost = [m[0]] + [2 * v for v in m[1:]]
    parts = max(1, min(parts, L))
    total, acc, cuts = sum(cost), 0, []
    for i, c in enumerate(cost):
        acc += c
        if len(cuts) < parts - 1 and acc >= total * (len(cuts) + 1) / parts and i < L - 1:
            cuts.append(i + 1)
    bounds = [0] + cuts + [L]
    return [(a, b - 1) for a, b in zip(bounds[:-1], bounds[1:])]


def candidate_seconds_by_slices(arm: RefArm, net: dict, threads: int):
    """A bounded sample of one candidate's reference Fisher cost at N=1:
    the network is cut into `threads` slices (above), each slice scored as
    its own network by fisher_potential, all slices at once on `threads`
    threads; the overlap layers' extra forwards are timed with layer_forward
    and subtracted.  Returns (thread-seconds of one N=1 evaluation, wall
    seconds of the sample, slice count)."""
    sl = slices(net, threads)
    nets = []
    for i, (a, b) in enumerate(sl):
        lo = a - 1 if i > 0 else a
        nets.append({"schema_version": 1, "seed": net.get("seed", 42),
                     "num_classes": net.get("num_classes", 10),
                     "layers": [dict(l) for l in net["layers"][lo:b + 1]]})
    _, sec, wall = arm.fisher_jobs(nets, 1, threads)
    extra = sum(arm.layer_forward_seconds(net["layers"][a - 1]) for a, _ in sl[1:])
    return sum(sec) - extra, wall, len(sl)
