"""bench.py's e2e at small K: phase times (sessions / evaluate / close),
synchronised, after the same warm-up and cache reset as bench.py."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
K, W = int(sys.argv[1]), int(sys.argv[2])
origin = resnet34_chain()
pool = load_candidates(fixture_path("r34_candidates.json"), origin)
order = np.random.default_rng(0).permutation(len(pool))
pool = [pool[i] for i in order]
warm, mine = pool[:W], pool[W:W + K]
batch = nb.make_batch(origin, 128, 1)
ctxs = [nb.Context(0) for _ in range(4)]
sess = [nb.Session(origin, batch, ctx=c) for c in ctxs]
nb.evaluate(sess, warm)
for s in sess:
    s.fisher(origin)
def sync():
    torch.cuda.synchronize()
    return time.perf_counter()
t0 = sync(); nb.evaluate(sess, mine); t1 = sync()
print(f"timed-equivalent evaluate {1e3*(t1-t0):.1f} ms", flush=True)
xin = torch.from_numpy(batch.inputs).pin_memory()
lab = torch.from_numpy(batch.labels).pin_memory()
hb = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)
def e2e(p, tag):
    t0 = sync()
    ss = [nb.Session(origin, hb, ctx=c) for c in ctxs]
    t1 = sync()
    nb.evaluate(ss, p)
    t2 = sync()
    for s in ss:
        s.close()
    t3 = sync()
    print(f"{tag}: sessions {1e3*(t1-t0):.1f} ms  evaluate {1e3*(t2-t1):.1f} ms  close {1e3*(t3-t2):.1f} ms", flush=True)
e2e(warm, "e2e warm")
for c in ctxs:
    c.clear_caches()
t0 = sync(); nb.evaluate(sess, warm); t1 = sync()
print(f"re-warm {1e3*(t1-t0):.1f} ms")
e2e(mine, "e2e timed")
e2e(mine, "e2e again")
for i in range(3):
    t0 = sync(); nb.evaluate(sess, mine); t1 = sync()
    print(f"evaluate again {1e3*(t1-t0):.1f} ms", flush=True)
