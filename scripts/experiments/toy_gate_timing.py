import json, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2102_06599_b200 import search as S
g = json.load(open("tests/golden/search_toy_1000.json"))
cfg = dict(g["config"])
S.gate_candidates(dict(cfg, candidate_count=8), legal_device=0)
for dev in (0, -1):
    t = time.perf_counter(); S.gate_candidates(cfg, legal_device=dev); print(os.environ.get("NB_LEGAL_GPU_MIN"), dev, round(time.perf_counter() - t, 3))
