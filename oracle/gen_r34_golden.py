"""TEST INFRASTRUCTURE: goldens at the benchmarked configuration (BASELINE
configs[1]): the 33-conv ResNet-34 CIFAR chain at batch
N=128 (make_batch seed 1, init_weights seed 42).

Two outputs, both from oracle/nb_oracle.cpp (the fp64 restatement of
I/nnet.hpp:58-352, pinned to the unmodified reference by tests/test_oracle.py
to 1e-12).  The reference itself needs about 7 h per network per core at
N=128 (SURVEY finding 2), so the restatement -- same loops, same summation
order, OpenMP over examples -- stands in for it at this size:

1. tests/golden/r34_n128.json + r34_n128.npz: the origin and a fixed set of
   bench-pool candidates (tests/golden/r34_candidates.json) covering the
   kernel families the pool's candidates lower to: depthwise, crop,
   bottleneck (down to co_eff = 1), grouped G <= 8 (densified tensor-core
   plans), G > 8 (FFMA), and masks on the stem, a stride-2 layer and the
   512-channel stage.  per_layer / total / loss in JSON; per_channel and
   probs in the npz.

2. tests/golden/r34_search_m{M}.json: the reference's run_search report
   (I/search.hpp:364-393) of the per-layer neural search on layer M --
   draw_candidates (reference, serial), evaluate_candidate's host gates
   (integration bridge over the reference's own apply /
   check_semantic_legality / derived_spec / repair_network), then, for
   every neural candidate, fisher_potential of its network at N=128 with
   fisher_accepts (>=) against the origin, and rank_survivors (macs asc,
   fisher desc, index asc).  Identical networks are scored once.

    python oracle/gen_r34_golden.py [pool|search M ...]
"""
import collections
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.oracle import Restatement  # noqa: E402
from paper_2102_06599_b200.api import Network  # noqa: E402
from paper_2102_06599_b200.workloads import (fixture_path, load_candidates,  # noqa: E402
                                             resnet34_chain)

N = 128
GOLD = os.path.join(ROOT, "tests", "golden")

# (masked layer, kind label) -> the first pool candidate of that kind
PICKS = [(1, "dw"), (1, "g8"), (1, "g2+b4"), (1, "g16+b4+crop2x4"), (0, "b2"),
         (0, "crop1x2"), (0, "b64"), (7, "dw*"), (7, "g*"), (15, "b*"), (27, "crop*"),
         (32, "*"), (16, "g*")]


def kind(s):
    k = []
    g = s.get("groups", 1)
    if g == s["ci"] and g == s["co"] // s.get("bottleneck", 1):
        k.append("dw")
    elif g > 1:
        k.append(f"g{g}")
    if s.get("bottleneck", 1) > 1:
        k.append(f"b{s['bottleneck']}")
    if s.get("spatial_div_h", 1) > 1 or s.get("spatial_div_w", 1) > 1:
        k.append(f"crop{s.get('spatial_div_h', 1)}x{s.get('spatial_div_w', 1)}")
    return "+".join(k)


def match(label, k):
    if label.endswith("*"):
        return k.startswith(label[:-1])
    return k == label


def pool_golden():
    R = Restatement()
    raw = json.load(open(fixture_path("r34_candidates.json")))["candidates"]
    origin = resnet34_chain()
    nets = load_candidates(fixture_path("r34_candidates.json"), origin)
    chosen = []
    for m, label in PICKS:
        for i, c in enumerate(raw):
            if c["diff"][0] == m and match(label, kind(c["diff"][1])) and i not in chosen:
                chosen.append(i)
                break
        else:
            raise SystemExit(f"no pool candidate for {m} {label}")
    entries, arrays = [], {}
    for name, idx, net in [("origin", -1, origin)] + [(f"pool{i}", i, nets[i]) for i in chosen]:
        t = time.time()
        r = R.fisher(net, N, 1)
        print(f"{name}: {kind(raw[idx]['diff'][1]) if idx >= 0 else 'origin'} "
              f"total {r['total']:.17g} ({time.time() - t:.0f} s)", flush=True)
        entries.append({"name": name, "pool_index": idx,
                        "mask": raw[idx]["diff"][0] if idx >= 0 else None,
                        "kind": kind(raw[idx]["diff"][1]) if idx >= 0 else "origin",
                        "total": r["total"], "loss": r["loss"],
                        "per_layer": r["per_layer"].tolist()})
        arrays[name + "_per_channel"] = r["per_channel"]
        arrays[name + "_probs"] = r["probs"]
    json.dump({"generator": "oracle/gen_r34_golden.py pool (nb_oracle restatement, fp64)",
               "n": N, "batch_seed": 1, "weight_seed": 42, "networks": entries},
              open(os.path.join(GOLD, "r34_n128.json"), "w"), indent=1)
    np.savez_compressed(os.path.join(GOLD, "r34_n128.npz"), **arrays)


def search_config(mask, count=200):
    o = resnet34_chain().to_json()
    L = len(o["layers"])
    return {"schema_version": 1, "candidate_count": count, "max_seq_len": 6, "seed": 7,
            "kinds": ["bottleneck", "group", "depthwise"], "batch": {"n": N, "seed": 1},
            "layer_mask": [l == mask for l in range(L)], "network": o}


def fmt_g(v):
    """std::ostream << double (default precision 6, %g-like)."""
    return f"{v:g}"


def search_golden(mask):
    from paper_2102_06599_b200 import search as S
    from paper_2102_06599_b200.api import network_macs
    R = Restatement()
    cfg = search_config(mask)
    draws = S.draw_candidates(cfg, 0)
    gated = S.gate_candidates(cfg)
    origin = resnet34_chain()
    t = time.time()
    o = R.fisher(origin, N, 1)
    print(f"mask {mask}: origin total {o['total']:.17g} ({time.time() - t:.0f} s)", flush=True)
    cache = {json.dumps(origin.to_json()["layers"], sort_keys=True): o}
    cands = []
    for i, (d, g) in enumerate(zip(draws, gated)):
        c = {"index": i, "macs": g["macs"], "neural": g["neural"], "sequences": d["layers"]}
        if g["status"] == "fisher":
            key = json.dumps(g["network"]["layers"], sort_keys=True)
            if key not in cache:
                t = time.time()
                cache[key] = R.fisher(Network.from_json(g["network"]), N, 1)
                print(f"  cand {i}: total {cache[key]['total']:.6g} ({time.time() - t:.0f} s,"
                      f" {len(cache)} distinct)", flush=True)
            r = cache[key]
            c["fisher_total"] = r["total"]
            c["fisher_per_layer"] = r["per_layer"].tolist()
            if r["total"] >= o["total"]:
                c["status"] = "survivor"
            else:
                c["status"] = "rejected_fisher"
                c["reason"] = (f"fisher potential dropped: {fmt_g(r['total'])} < "
                               f"{fmt_g(o['total'])}")
            c["relative_margin"] = (r["total"] - o["total"]) / o["total"]
        elif g["status"] == "survivor":
            c["status"] = "survivor"
            c["fisher_total"] = o["total"]
            c["fisher_per_layer"] = o["per_layer"].tolist()
        else:
            c["status"] = g["status"]
            c["reason"] = g.get("reason", "")
        cands.append(c)
    surv = [c["index"] for c in cands if c["status"] == "survivor"]
    ranked = sorted(surv, key=lambda i: (cands[i]["macs"], -cands[i]["fisher_total"], i))
    st = collections.Counter(c["status"] for c in cands)
    rep = {"generator": "oracle/gen_r34_golden.py search (reference draw + host gates, "
                        "nb_oracle fp64 Fisher at N=128)",
           "config": cfg, "origin": {"fisher_total": o["total"],
                                     "macs": network_macs(origin)},
           "candidates": cands, "survivors_ranked": ranked,
           "stats": {"survivors": st["survivor"], "rejected_semantic": st["rejected_semantic"],
                     "rejected_fisher": st["rejected_fisher"]},
           "distinct_networks": len(cache)}
    json.dump(rep, open(os.path.join(GOLD, f"r34_search_m{mask}.json"), "w"),
              separators=(",", ":"))
    print(f"mask {mask}: {rep['stats']} best {ranked[:3]}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "pool"
    if what == "pool":
        pool_golden()
    else:
        for m in sys.argv[2:]:
            search_golden(int(m))
