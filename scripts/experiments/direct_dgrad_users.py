"""Which bench-pool candidates run their dgrad on k_dgrad_direct (FFMA gather),
and how long it takes: per-candidate kernel stats over the 726-network pool."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
import bench
origin, warm, timed, spare = bench.timed_pool(64, 8, 1)
pool = warm + timed + spare
ctx = nb.Context(0)
net0 = nb.Network.from_json(origin)
sess = nb.Session(net0, nb.make_batch(net0, 128, 1), ctx=ctx)
rows = []
for j in pool:
    net = nb.Network.from_json(j)
    ctx.reset_stats(); ctx.set_profiling(True)
    sess.fisher(net, Precision.FP32)
    ctx.set_profiling(False)
    st = ctx.kernel_stats()
    d = st.get("conv_dgrad_direct_fisher")
    if d:
        ch = next((l for l, (a, b) in enumerate(zip(j["layers"], origin["layers"])) if a != b), None)
        rows.append((d["ms"], ch, j["layers"][ch] if ch is not None else None))
rows.sort(key=lambda r: -r[0])
print(len(rows), "candidates with direct dgrad; total ms", round(sum(r[0] for r in rows), 2))
for r in rows[:15]:
    print(round(r[0], 3), r[1], json.dumps(r[2]))
