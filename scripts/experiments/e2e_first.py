"""First vs second pass of the same 40-candidate pool on fresh contexts
(wall time and the device busy time of each session)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2102_06599_b200 as nb
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
origin_j, warm_j, timed_j, _ = bench.timed_pool(steps, 5, 1)
origin = nb.Network.from_json(origin_j)
warm = [nb.Network.from_json(n) for n in warm_j]
timed = [nb.Network.from_json(n) for n in timed_j]
batch = nb.make_batch(origin, 128, 1)
ctxs = [nb.Context(0) for _ in range(4)]
ss = [nb.Session(origin, batch, ctx=c) for c in ctxs]
nb.evaluate(ss, warm)
for s in ss:
    s.fisher(origin)
for p in range(3):
    for c in ctxs:
        c.reset_stats(); c.set_profiling(True, every=1)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r, st = nb.evaluate(ss, timed)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    agg = {}
    for c in ctxs:
        for k, v in c.kernel_stats().items():
            agg[k] = agg.get(k, 0) + v["ms"]
    top = sorted(((v, k) for k, v in agg.items()), reverse=True)[:8]
    print(f"pass {p}: {1e3*(t1-t0):.1f} ms busy {[round(b,1) for b in st.busy_ms]}", [(k, round(v, 1)) for v, k in top], flush=True)
