"""Where does the e2e time of bench.py go?  Times session creation from a
pinned host batch, the evaluation and the teardown, five times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
origin = resnet34_chain()
pool = load_candidates(fixture_path("r34_candidates.json"), origin)
order = np.random.default_rng(0).permutation(len(pool))
pool = [pool[i] for i in order][8:72]
batch = nb.make_batch(origin, 128, 1)
ctxs = [nb.Context(0) for _ in range(4)]
sess = [nb.Session(origin, batch, ctx=c) for c in ctxs]
nb.evaluate(sess, pool)
xin = torch.from_numpy(batch.inputs).pin_memory()
lab = torch.from_numpy(batch.labels).pin_memory()
hb = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)
for it in range(5):
    t0 = time.perf_counter()
    ss = [nb.Session(origin, hb, ctx=c) for c in ctxs]
    t1 = time.perf_counter()
    nb.evaluate(ss, pool)
    t2 = time.perf_counter()
    for s in ss:
        s.close()
    t3 = time.perf_counter()
    print(f"iter {it}: sessions {1e3*(t1-t0):.1f} ms  evaluate {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms", flush=True)
