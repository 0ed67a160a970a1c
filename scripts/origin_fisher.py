"""Runs fisher_potential of the R34 origin chain (N=128) on one session a
few times -- the target of per-layer ncu captures (64 tcgen05 launches per
evaluation: fprop of layers 1..32, then dgrad of layers 32..1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from paper_2102_06599_b200.workloads import resnet34_chain
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prec = {"fp32": Precision.FP32, "tf32": Precision.TF32, "simt": Precision.SIMT}[
    sys.argv[2] if len(sys.argv) > 2 else "fp32"]
net = resnet34_chain()
ctx = nb.Context(0)
N = int(os.environ.get("ORIGIN_N", "128"))
s = nb.Session(net, nb.make_batch(net, N, 1), ctx=ctx)
for i in range(reps):
    t = time.perf_counter()
    r = s.fisher(net, prec)
    print(f"fisher {i}: {1e3 * (time.perf_counter() - t):.2f} ms total {r.total:.6e}", flush=True)
ctx.set_profiling(True)
s.fisher(net, prec)
for k, v in sorted(ctx.kernel_stats().items()):
    print(f"  {k:32s} {v['launches']:4d} {v['ms']:8.3f} ms", flush=True)
