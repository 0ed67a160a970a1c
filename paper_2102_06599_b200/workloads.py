"""Benchmark networks and candidate sets.

The reference can only express conv(+ReLU) chains followed by GAP + linear
head (I/nnet.hpp:23-79), so each benchmark architecture is its chain of conv
shapes.  Candidate sets are the rewritten networks a per-layer search
produces (neural rewrites: bottleneck, group, depthwise, spatial crop),
lowered to ConvSpecs and shape-repaired exactly as evaluate_candidate does
(I/search.hpp:270-292).
"""
from __future__ import annotations

import json
import os
from typing import List

import numpy as np

from .api import ConvSpec, Layer, Network, repair_network


def conv3(ci, co, hw, stride=1, groups=1):
    return Layer(ConvSpec(ci, co, hw, hw, 3, 3, stride, 1, groups=groups))


def conv1(ci, co, hw):
    return Layer(ConvSpec(ci, co, hw, hw, 1, 1, 1, 0))


def resnet34_chain(seed: int = 42) -> Network:
    """The 33-conv ResNet-34 CIFAR chain: 1,153,105,920 MACs
    per image."""
    L = [conv3(3, 64, 32)] + [conv3(64, 64, 32) for _ in range(6)]
    L += [conv3(64, 128, 32, 2)] + [conv3(128, 128, 16) for _ in range(7)]
    L += [conv3(128, 256, 16, 2)] + [conv3(256, 256, 8) for _ in range(11)]
    L += [conv3(256, 512, 8, 2)] + [conv3(512, 512, 4) for _ in range(5)]
    return Network(L, num_classes=10, seed=seed)


def resnext29_chain(seed: int = 42) -> Network:
    """ResNeXt-29 (2x64d) CIFAR chain, 28 convs."""
    L = [conv3(3, 64, 32)]
    cin, hw = 64, 32
    for inner, out, stride in [(128, 256, 1), (256, 512, 2), (512, 1024, 2)]:
        for b in range(3):
            s = stride if b == 0 else 1
            L.append(conv1(cin, inner, hw))
            L.append(conv3(inner, inner, hw, s, groups=2))
            hw //= s
            L.append(conv1(inner, out, hw))
            cin = out
    return Network(L, num_classes=10, seed=seed)


def densenet161_layer_chains(seed: int = 42) -> List[Network]:
    """DenseNet-161 CIFAR: every dense layer as its own 2-conv chain
    [1x1 c->192, 3x3 192->48] (concatenation is not chain-expressible)."""
    nets = []
    c, hw = 96, 32
    for bi, nl in enumerate([6, 12, 36, 24]):
        for i in range(nl):
            cin = c + 48 * i
            nets.append(Network([conv1(cin, 192, hw), conv3(192, 48, hw)], num_classes=10,
                                seed=seed))
        c = c + 48 * nl
        if bi < 3:
            c //= 2
            hw //= 2
    return nets


def c1_network(groups: int = 1, bottleneck: int = 1, seed: int = 42) -> Network:
    """configs[0]: single 3x3 conv 64->64, 32x32."""
    return Network([Layer(ConvSpec(64, 64, 32, 32, 3, 3, 1, 1, groups=groups,
                                   bottleneck_out=bottleneck))], num_classes=10, seed=seed)


# ---------------------------------------------------------------------------
# candidate sets

def _variant(origin: Network, layer: int, *, b=1, g=1, dw=False, crop=(1, 1)):
    net = origin.copy()
    s = net.layers[layer].spec
    s.bottleneck_out = b
    s.groups = s.ci if dw else g
    s.spatial_div_h, s.spatial_div_w = crop
    if dw and s.co_eff() != s.ci:
        return None
    try:
        repair_network(net)
    except Exception:
        return None
    return net


def per_layer_candidates(origin: Network, count: int, seed: int = 7) -> List[Network]:
    """A deterministic mix shaped like the reference's per-layer neural
    search (SURVEY finding 12: ~50% depthwise, ~40% dense+crop/bottleneck,
    ~10% grouped): one rewritten layer per candidate, repaired downstream."""
    rng = np.random.default_rng(seed)
    out: List[Network] = []
    L = len(origin.layers)
    while len(out) < count:
        l = int(rng.integers(1, L))
        s = origin.layers[l].spec
        kind = rng.random()
        oh, ow = s.raw_out_h(), s.raw_out_w()
        divs = [d for d in (1, 2, 4) if oh % d == 0 and ow % d == 0]
        crop = int(rng.choice(divs))
        if kind < 0.5:
            v = _variant(origin, l, dw=True, crop=(crop, crop))
        elif kind < 0.9:
            v = _variant(origin, l, b=int(rng.choice([1, 2, 4])), crop=(crop, crop))
        else:
            v = _variant(origin, l, g=int(rng.choice([2, 4, 8])))
        if v is not None:
            out.append(v)
    return out


def load_candidates(path: str, origin: Network) -> List[Network]:
    """Candidate networks of tests/golden/r34_candidates.json (written by
    oracle/gen_r34_candidates.py from the reference's draw_candidates and
    evaluate_candidate's host gates): each is the origin with one layer's
    spec replaced, shapes repaired downstream (repair_network)."""
    with open(path) as f:
        data = json.load(f)
    nets = []
    for c in data["candidates"]:
        l, sj = c["diff"]
        n = origin.copy()
        n.layers[l] = Layer(ConvSpec.from_json(dict(sj, ci=sj["ci"])), sj.get("relu", True))
        repair_network(n)
        nets.append(n)
    return nets


def shard_lpt(costs: List[float], world: int, per_rank: int) -> List[int]:
    """Candidate sharding of the multi-GPU run (no collective on the data
    path): longest-processing-time-first on the estimated Fisher FLOPs,
    each rank taking exactly `per_rank` candidates (ties by index), so every
    rank's assignment is computed identically and independently."""
    if len(costs) != world * per_rank:
        raise ValueError("need exactly world * per_rank candidates")
    loads, counts = [0.0] * world, [0] * world
    assign = [0] * len(costs)
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min((r for r in range(world) if counts[r] < per_rank), key=lambda r: (loads[r], r))
        assign[i] = r
        loads[r] += costs[i]
        counts[r] += 1
    return assign


def fixture_path(name: str) -> str:
    return os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                        "golden", name)
