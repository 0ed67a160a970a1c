"""Host-phase profile of bench.py's value pass vs its e2e pass (40 steps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import time
import torch
import paper_2102_06599_b200 as nb
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
origin_j, warm_j, timed_j, _ = bench.timed_pool(steps, 5, 1)
origin = nb.Network.from_json(origin_j)
warm = [nb.Network.from_json(n) for n in warm_j]
timed = [nb.Network.from_json(n) for n in timed_j]
batch = nb.make_batch(origin, 128, 1)
xin = torch.from_numpy(batch.inputs).pin_memory(); lab = torch.from_numpy(batch.labels).pin_memory()
hb = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)
for label, hostb in (("value", batch), ("e2e", hb), ("value-again", batch)):
    ctxs = [nb.Context(0) for _ in range(4)]
    ws = [nb.Session(origin, batch, ctx=c) for c in ctxs]
    nb.evaluate(ws, warm)
    for s in ws:
        s.fisher(origin)
    for c in ctxs:
        c.reset_stats(); c.set_profiling(True, every=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ss = ws if label.startswith("value") else [nb.Session(origin, hostb, ctx=c) for c in ctxs]
    r, st = nb.evaluate(ss, timed)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    agg = {}
    for c in ctxs:
        for k, v in c.kernel_stats().items():
            if k.startswith("host"):
                agg[k] = agg.get(k, 0) + v["ms"]
    print(label, f"{1e3*(t1-t0):.1f} ms", {k: round(v, 1) for k, v in agg.items()}, "busy", [round(b, 1) for b in st.busy_ms], flush=True)
