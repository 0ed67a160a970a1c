"""Why does bench.py's e2e fall behind the device-timed value at 40 steps?
Times session creation / evaluate / close of the e2e path for 20 and 40
candidates, after the bench's own cache preparation."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2102_06599_b200 as nb
import bench
for steps in (20, 40):
    origin_j, warm_j, timed_j, _ = bench.timed_pool(steps, 5, 1)
    origin = nb.Network.from_json(origin_j)
    warm = [nb.Network.from_json(n) for n in warm_j]
    timed = [nb.Network.from_json(n) for n in timed_j]
    batch = nb.make_batch(origin, 128, 1)
    ctxs = [nb.Context(0) for _ in range(4)]
    sess = [nb.Session(origin, batch, ctx=c) for c in ctxs]
    nb.evaluate(sess, warm)
    xin = torch.from_numpy(batch.inputs).pin_memory(); lab = torch.from_numpy(batch.labels).pin_memory()
    hb = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)
    for rep in range(3):
        for c in ctxs:
            c.clear_caches()
        nb.evaluate(sess, warm)
        for s in sess:
            s.fisher(origin)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ss = [nb.Session(origin, hb, ctx=c) for c in ctxs]
        t1 = time.perf_counter()
        r, st = nb.evaluate(ss, timed)
        t2 = time.perf_counter()
        for s in ss:
            s.close()
        t3 = time.perf_counter()
        t4 = time.perf_counter(); nb.evaluate(sess, timed); t5 = time.perf_counter()
        print(f"steps {steps} rep {rep}: sessions {1e3*(t1-t0):.1f} evaluate {1e3*(t2-t1):.1f} close {1e3*(t3-t2):.1f} | cached re-evaluate {1e3*(t5-t4):.1f} ms", flush=True)
