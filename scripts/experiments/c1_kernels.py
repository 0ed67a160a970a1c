import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import c1_network
for g in (1, 4):
    ctx = nb.Context(0)
    net = c1_network(groups=g)
    s = nb.Session(net, nb.make_batch(net, 8, 1), ctx=ctx)
    for _ in range(3): s.fisher(net)
    ctx.reset_stats(); ctx.set_profiling(True)
    for _ in range(5): s.fisher(net)
    ctx.set_profiling(False)
    print("groups", g)
    for k, v in sorted(ctx.kernel_stats().items()):
        print(f"  {k:32s} {v['launches']:4d} {v['ms']/5:8.4f} ms/eval")
