"""Single-stream time of bench.py's timed candidate pool (64 R34 candidates,
N=128) on one session: steadier than the 4-stream bench for A/B of lowering
switches (NB_TC_*).  Prints the best of 3 passes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
origin = resnet34_chain()
pool = load_candidates(fixture_path("r34_candidates.json"), origin)
order = np.random.default_rng(0).permutation(len(pool))
pool = [pool[i] for i in order]
warm, timed = pool[:8], pool[8:72]
s = nb.Session(origin, nb.make_batch(origin, 128, 1), ctx=nb.Context(0))
nb.evaluate([s], warm)
nb.evaluate([s], timed)
best = 1e9
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    nb.evaluate([s], timed)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t)
print(f"{os.environ.get('TAG', 'default')}: {1e3 * best:.1f} ms for {len(timed)} candidates "
      f"({len(timed) / best:.1f} cand/s single stream)", flush=True)
