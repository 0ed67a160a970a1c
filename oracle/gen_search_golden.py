"""TEST INFRASTRUCTURE: generates tests/golden/search_toy_1000.json from the
UNMODIFIED reference (oracle/_ref/libnestopt_ref.so -> run_search,
I/search.hpp:364) with the configuration of acceptance criterion 7
(T/acceptance.cpp:406-433: the 4-layer search network, 1000 candidates,
max_seq_len 4, seed 7, batch n=4 seed 1, default kinds and cap).  The
digest keeps per-candidate status / macs / fisher_total / reason, the ranked
survivors and the bucket counts."""
import json, os, sys, time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Reference  # noqa: E402

SAMPLES = "/root/reference/proj/samples"


def criterion7_config():
    net = json.load(open(os.path.join(SAMPLES, "search_toy.json")))["network"]
    return {"schema_version": 1, "candidate_count": 1000, "max_seq_len": 4, "seed": 7,
            "batch": {"n": 4, "seed": 1}, "network": net}


def main():
    cfg = criterion7_config()
    t0 = time.time()
    rep = Reference().search(cfg, jobs=os.cpu_count() or 1)
    dt = time.time() - t0
    digest = {
        "generator": "oracle/gen_search_golden.py (run_search, I/search.hpp:364; "
                     "acceptance criterion 7 config)",
        "config": cfg, "reference_wall_s": dt,
        "origin": rep["origin"], "stats": rep["stats"],
        "survivors_ranked": rep["survivors_ranked"],
        "candidates": [{k: c[k] for k in ("status", "neural", "macs", "fisher_total", "reason")
                        if k in c} for c in rep["candidates"]],
    }
    out = os.path.join(os.path.dirname(HERE), "tests", "golden", "search_toy_1000.json")
    json.dump(digest, open(out, "w"), separators=(",", ":"))
    print(rep["stats"], "best", rep["survivors_ranked"][:1], f"{dt:.1f}s")


if __name__ == "__main__":
    main()
