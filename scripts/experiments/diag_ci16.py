"""Localise the pool141/pool135 tensor-core error (GPU experiment): short
chains around the 16-channel layer at several batch sizes vs the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
from oracle.oracle import Restatement
O = Restatement()
pool = load_candidates(fixture_path("r34_candidates.json"), resnet34_chain())
def sub(net, k):
    return Network(net.layers[:k], num_classes=10, seed=net.seed)
cases = {
  "p141[:4]": sub(pool[141], 4), "p135[:4]": sub(pool[135], 4),
  "p141[:3]": sub(pool[141], 3), "p141[:2]": sub(pool[141], 2),
  "c16": Network([Layer(ConvSpec(3, 16, 32, 32, 3, 3, 1, 1)), Layer(ConvSpec(16, 64, 32, 32, 3, 3, 1, 1)),
                  Layer(ConvSpec(64, 64, 32, 32, 3, 3, 1, 1))], num_classes=10, seed=42),
}
for k, v in cases.items():
    print(k, [ (l.spec.ci, l.spec.co, l.spec.h, l.spec.w, l.spec.groups, l.spec.bottleneck_out, l.spec.spatial_div_h, l.spec.spatial_div_w) for l in v.layers])
for n in (4, 32, 128):
    for name, net in cases.items():
        b = nb.make_batch(net, n, 1)
        ref = O.fisher(net, n, batch=b)
        ctx = nb.Context(0)
        out = [f"n={n:3d} {name:9s}"]
        for pn, p in (("simt", Precision.SIMT), ("3x", Precision.FP32), ("tf32", Precision.TF32)):
            r = nb.fisher_potential(net, b, precision=p, ctx=ctx)
            le = (r.per_layer - ref["per_layer"]) / ref["per_layer"]
            out.append(f"{pn}: " + " ".join(f"{x:+.1e}" for x in le))
        print("  ".join(out), flush=True)
