"""Host gates of an all-kinds R34 search (the reference's default kinds,
semantic runs included) with the reference's host legality check vs the GPU
check: wall time and identical outcomes.  Usage: python scripts/gate_timing.py
[count] [mask_layers...]"""
import collections, json, os, sys, time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_06599_b200 import search as S  # noqa: E402
from paper_2102_06599_b200.workloads import resnet34_chain  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
mask = [int(x) for x in sys.argv[2:]] or [0, 1]
o = resnet34_chain().to_json()
L = len(o["layers"])
cfg = {"schema_version": 1, "candidate_count": count, "max_seq_len": 6, "seed": 7,
       "batch": {"n": 128, "seed": 1}, "layer_mask": [l in mask for l in range(L)], "network": o}
res = {}
S.gate_candidates(dict(cfg, candidate_count=8), legal_device=0)  # CUDA context / module load
for dev in (0, -1):
    t = time.perf_counter()
    g = S.gate_candidates(cfg, legal_device=dev)
    dt = time.perf_counter() - t
    res[dev] = g
    print(json.dumps({"legality": "gpu" if dev >= 0 else "host", "candidates": count,
                      "mask": mask, "threads": os.cpu_count(), "seconds": round(dt, 2),
                      "status": dict(collections.Counter(c["status"] for c in g))}), flush=True)
same = [(c["status"], c.get("reason"), c["macs"]) for c in res[0]] == \
       [(c["status"], c.get("reason"), c["macs"]) for c in res[-1]]
print(json.dumps({"identical": same}))
