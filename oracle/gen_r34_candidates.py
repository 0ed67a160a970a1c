"""TEST/BENCH INFRASTRUCTURE: the candidate pool of the R34 per-layer search
(BASELINE configs[1]): for each masked layer, the reference's
draw_candidates with neural kinds {bottleneck, group, depthwise},
max_seq_len 6, seed 7, 200 candidates, through evaluate_candidate's host
gates (integration/_build/libnb200_nestopt.so, compiled from the unmodified
reference headers).  The distinct networks that need a Fisher score are
written to tests/golden/r34_candidates.json as (masked layer, its rewritten
spec) -- the other layers follow from the origin by repair_network's shape
propagation (I/nnet.hpp:372-380) -- with the per-mask draw statistics."""
import collections, json, os, sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2102_06599_b200 import search as S  # noqa: E402
from paper_2102_06599_b200.workloads import resnet34_chain  # noqa: E402

def rebuild(origin, diff):
    """origin layers with layer diff[0] replaced by diff[1], shapes repaired."""
    layers = [dict(l) for l in origin["layers"]]
    layers[diff[0]] = dict(diff[1])
    for l in range(1, len(layers)):
        p = layers[l - 1]
        co_eff = p["co"] // p.get("bottleneck", 1)
        oh = ((p["h"] + 2 * p.get("pad", 0) - p.get("kh", 1)) // p.get("stride", 1) + 1) \
            // p.get("spatial_div_h", 1)
        ow = ((p["w"] + 2 * p.get("pad", 0) - p.get("kw", 1)) // p.get("stride", 1) + 1) \
            // p.get("spatial_div_w", 1)
        layers[l]["ci"], layers[l]["h"], layers[l]["w"] = co_eff, oh, ow
    return layers


MASKS = [0, 1, 3, 7, 8, 12, 15, 16, 22, 27, 28, 32]


def main():
    origin = resnet34_chain().to_json()
    L = len(origin["layers"])
    seen, pool, stats = set(), [], {}
    for m in MASKS:
        cfg = {"schema_version": 1, "candidate_count": 200, "max_seq_len": 6, "seed": 7,
               "kinds": ["bottleneck", "group", "depthwise"], "batch": {"n": 128, "seed": 1},
               "layer_mask": [l == m for l in range(L)], "network": origin}
        g = S.gate_candidates(cfg)
        c = collections.Counter(x["status"] for x in g)
        new = 0
        for x in g:
            if x["status"] != "fisher":
                continue
            net = x["network"]
            diff = [m, net["layers"][m]]  # the rest follows by repair_network
            assert rebuild(origin, diff) == net["layers"]
            key = json.dumps(net["layers"], sort_keys=True)
            if key in seen:
                continue
            seen.add(key)
            pool.append({"mask": m, "macs": x["macs"], "diff": diff})
            new += 1
        stats[str(m)] = dict(c, distinct_new=new)
        print(m, dict(c), "distinct", new, flush=True)
    out = os.path.join(os.path.dirname(HERE), "tests", "golden", "r34_candidates.json")
    json.dump({"generator": "oracle/gen_r34_candidates.py (draw_candidates + host gates)",
               "origin": origin, "masks": MASKS, "stats": stats, "candidates": pool},
              open(out, "w"), separators=(",", ":"))
    print(len(pool), "distinct candidate networks ->", out)


if __name__ == "__main__":
    main()
