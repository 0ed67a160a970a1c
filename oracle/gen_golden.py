"""TEST INFRASTRUCTURE: generates tests/golden/*.json from the UNMODIFIED
reference (oracle/_ref/libnestopt_ref.so, built from /root/reference by
oracle/Makefile).  Run here (where /root/reference exists):

    make -C oracle && python oracle/gen_golden.py

The fixtures are small and committed; the GPU box never needs the reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2102_06599_b200.api import ChannelSplit, ConvSpec, Layer, Network  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SAMPLES = "/root/reference/proj/samples"


def conv_cases():
    """Specs covering every ConvSpec feature; inputs are small ints drawn by
    numpy from the case index (regenerable in the tests)."""
    S = ConvSpec
    specs = [
        S(1, 1, 1, 1),                                        # 1x1 KAT shape
        S(4, 4, 1, 1, groups=2),                              # grouped KAT shape
        S(1, 1, 2, 2, 3, 3, 1, 1),                            # padded KAT shape
        S(8, 8, 8, 8, 3, 3, 1, 1),                            # conv_small.json
        S(8, 16, 8, 8, 3, 3, 1, 1, groups=2),                 # conv_grouped.json
        S(4, 8, 4, 4, 3, 3, 1, 1, groups=4, bottleneck_out=2),
        S(8, 8, 7, 9, 3, 3, 2, 1),                            # stride 2, odd sizes
        S(6, 6, 8, 8, 3, 3, 1, 1, groups=6),                  # depthwise
        S(8, 8, 8, 8, 3, 3, 1, 1, spatial_div_h=2, spatial_div_w=4),  # crop
        S(8, 8, 8, 8, 3, 3, 1, 1, channel_splits=[ChannelSplit(0, 4, 2), ChannelSplit(4, 8, 4)]),
        S(8, 16, 6, 6, 1, 1, 1, 0, bottleneck_out=16),        # Co_eff = 1
        S(16, 16, 5, 5, 3, 3, 1, 1, groups=16, spatial_div_h=5),
        S(12, 12, 8, 8, 5, 5, 1, 2, groups=3),
        S(8, 8, 9, 9, 3, 3, 2, 0, spatial_div_h=2, spatial_div_w=2),
        S(8, 12, 6, 6, 3, 1, 1, 0, channel_splits=[ChannelSplit(0, 6, 2), ChannelSplit(6, 12, 1)]),
    ]
    return specs


def inputs_for(i, spec):
    rng = np.random.default_rng(1000 + i)
    x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
    return x, w


def nets():
    j = json.load(open(os.path.join(SAMPLES, "network_toy.json")))
    toy = Network.from_json(j)
    s = json.load(open(os.path.join(SAMPLES, "search_toy.json")))
    search_net = Network.from_json(s["network"])
    mixed = Network([
        Layer(ConvSpec(3, 8, 9, 9, 3, 3, 2, 1)),
        Layer(ConvSpec(8, 8, 5, 5, 3, 3, 1, 1, groups=2, spatial_div_h=5)),
        Layer(ConvSpec(8, 6, 1, 5, 1, 3, 1, 0,
                       channel_splits=[ChannelSplit(0, 2, 2), ChannelSplit(2, 6, 1)])),
        Layer(ConvSpec(6, 6, 1, 3, 3, 3, 1, 1, groups=6)),
    ], num_classes=5, seed=3)
    norelu = Network([
        Layer(ConvSpec(2, 4, 5, 5, 3, 3, 1, 1), relu=True),
        Layer(ConvSpec(4, 4, 5, 5, 3, 3, 1, 1), relu=False),
        Layer(ConvSpec(4, 3, 5, 5, 1, 1, 1, 0), relu=True),
    ], num_classes=4, seed=42)
    mid = Network([Layer(ConvSpec(3, 16, 16, 16, 3, 3, 1, 1))] +
                  [Layer(ConvSpec(16, 16, 16, 16, 3, 3, 1, 1)) for _ in range(3)] +
                  [Layer(ConvSpec(16, 32, 16, 16, 3, 3, 2, 1))] +
                  [Layer(ConvSpec(32, 32, 8, 8, 3, 3, 1, 1)) for _ in range(4)] +
                  [Layer(ConvSpec(32, 32, 8, 8, 3, 3, 1, 1, bottleneck_out=2))],
                  num_classes=10, seed=42)
    c1 = lambda g, b: Network([Layer(ConvSpec(64, 64, 32, 32, 3, 3, 1, 1, groups=g,
                                              bottleneck_out=b))], num_classes=10, seed=42)
    return [
        ("network_toy", toy, 8, 1),
        ("search_toy_origin", search_net, 4, 1),
        ("mixed_features", mixed, 3, 5),
        ("norelu_toy", norelu, 4, 9),
        ("mid10", mid, 2, 1),
        ("c1_std_n1", c1(1, 1), 1, 1),
        ("c1_g4_n1", c1(4, 1), 1, 1),
        ("c1_b2_n1", c1(1, 2), 1, 1),
    ]


def main():
    R = Reference()
    os.makedirs(OUT, exist_ok=True)

    # ---- conv outputs: reference_conv<int64> and <double>
    cases = []
    for i, spec in enumerate(conv_cases()):
        x, w = inputs_for(i, spec)
        yi = R.conv(spec, x, w)
        yf = R.conv(spec, x.astype(np.float64) * 0.37, w.astype(np.float64) * 1.3)
        cases.append({"spec": spec.to_json(), "seed": 1000 + i,
                      "out_int": yi.ravel().tolist(), "out_f64": yf.ravel().tolist(),
                      "macs": R.count_macs(spec, "")})
    json.dump({"generator": "oracle/gen_golden.py (reference_conv, I/interp.hpp:151)",
               "cases": cases}, open(os.path.join(OUT, "conv_cases.json"), "w"))

    # ---- named sequences (Sequence 1/2/3, I/transforms.hpp:531-582) and rewrites
    seq = []
    base = ConvSpec(4, 16, 4, 4, 3, 3, 1, 1)
    for dsl in ["", "sequence1", "sequence2", "sequence3", "group(co,ci,2)", "bottleneck(co,2)",
                "bottleneck(h,2)", "spatial_bottleneck(2)", "depthwise",
                "interchange(co,ci) | unroll(co,4)", "sequence3(2,4)"]:
        spec = ConvSpec(8, 8, 4, 4, 3, 3, 1, 1) if dsl == "depthwise" else base
        rng = np.random.default_rng(7)
        x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
        w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
        ds = R.derived_spec(spec, dsl)
        entry = {"spec": spec.to_json(), "dsl": dsl, "derived_spec": ds,
                 "macs": R.count_macs(spec, dsl)}
        if ds is not None:
            d = ConvSpec.from_json(ds)
            if d.ci == spec.ci and (d.h, d.w) == (spec.h, spec.w):
                wd = w[:d.co_eff()] if d.co_eff() <= w.shape[0] else None
                if wd is not None:
                    entry["execute_int"] = R.execute(spec, dsl, x, w).ravel().tolist()
        else:
            entry["execute_int"] = R.execute(spec, dsl, x, w).ravel().tolist()
        seq.append(entry)
    json.dump({"generator": "oracle/gen_golden.py (apply/derived_spec/execute)", "cases": seq},
              open(os.path.join(OUT, "sequences.json"), "w"))

    # ---- Fisher potential of whole networks (fisher_potential, I/nnet.hpp:321)
    fis = []
    for name, net, n, bseed in nets():
        r = R.fisher(net, n, bseed)
        fis.append({"name": name, "network": net.to_json(), "n": n, "batch_seed": bseed,
                    "per_channel": r["per_channel"].tolist(), "per_layer": r["per_layer"].tolist(),
                    "total": r["total"], "loss": r["loss"], "probs": r["probs"].ravel().tolist()})
        print(name, r["total"], flush=True)
    json.dump({"generator": "oracle/gen_golden.py (fisher_potential, I/nnet.hpp:321)",
               "nets": fis}, open(os.path.join(OUT, "fisher_nets.json"), "w"))

    # ---- the reference's own 100-candidate sample search (P/samples/search_toy.json)
    cfg = json.load(open(os.path.join(SAMPLES, "search_toy.json")))
    rep = R.search(cfg, jobs=8)
    rep.pop("timing", None)
    json.dump(rep, open(os.path.join(OUT, "search_toy_100.json"), "w"))
    print("search_toy_100", rep["stats"], flush=True)


if __name__ == "__main__":
    main()
