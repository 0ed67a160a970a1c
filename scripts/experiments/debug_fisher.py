"""Per-layer Fisher comparison of every precision mode against the fp64
oracle, with repeat runs to expose nondeterminism.  Test infrastructure."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision
from oracle.oracle import Restatement

O = Restatement()
ctx = nb.Context(0)
gold = json.load(open("tests/golden/fisher_nets.json"))["nets"]
mid10 = Network.from_json([c for c in gold if c["name"] == "mid10"][0]["network"])
tc_chain = Network([
    Layer(ConvSpec(3, 32, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(32, 64, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=2)),
    Layer(ConvSpec(64, 128, 16, 16, 3, 3, 2, 1)),
    Layer(ConvSpec(128, 128, 8, 8, 3, 3, 1, 1, bottleneck_out=2)),
    Layer(ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, spatial_div_h=2, spatial_div_w=2)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1, groups=64)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1)),
], num_classes=10, seed=42)
for name, net, n in [("mid10", mid10, 2), ("mid10", mid10, 4), ("tc_chain", tc_chain, 4)]:
    batch = nb.make_batch(net, n, 1)
    o = O.fisher(net, n, batch=batch, grads=True)
    print(f"== {name} N={n} oracle total {o['total']:.6e}")
    print("   oracle per_layer", " ".join(f"{v:.3e}" for v in o["per_layer"]))
    for pn, p in [("simt", Precision.SIMT), ("fp32", Precision.FP32), ("tf32", Precision.TF32)]:
        reps = [nb.fisher_potential(net, batch, precision=p, ctx=ctx) for _ in range(2)]
        rel = (np.array(reps[0].per_layer) - o["per_layer"]) / o["per_layer"]
        print(f"   {pn}: total rel {(reps[0].total - o['total']) / o['total']:+.2e} "
              f"repeat-equal {reps[0].total == reps[1].total}  per-layer rel "
              + " ".join(f"{v:+.1e}" for v in rel))
        acts, grads = nb.activation_gradients(net, batch, precision=p, ctx=ctx)
        off = 0
        errs = []
        for a, g in zip(acts, grads):
            k = a.size
            ra, rg = o["acts"][off:off + k], o["grads"][off:off + k]
            errs.append((np.abs(a.ravel() - ra).max() / np.abs(ra).max(),
                         np.abs(g.ravel() - rg).max() / np.abs(rg).max()))
            off += k
        print("      act/grad max err rel-to-max: " + " ".join(f"{e[0]:.1e}/{e[1]:.1e}" for e in errs))
