"""Which prior call perturbs a later Fisher evaluation on the same context?"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision
gold = json.load(open("tests/golden/fisher_nets.json"))["nets"]
mid10 = Network.from_json([c for c in gold if c["name"] == "mid10"][0]["network"])
print("mid10 seed", mid10.seed)
tc = Network([
    Layer(ConvSpec(3, 32, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(32, 64, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=2)),
    Layer(ConvSpec(64, 128, 16, 16, 3, 3, 2, 1)),
    Layer(ConvSpec(128, 128, 8, 8, 3, 3, 1, 1, bottleneck_out=2)),
    Layer(ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, spatial_div_h=2, spatial_div_w=2)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1, groups=64)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1)),
], num_classes=10, seed=42)
ctx = nb.Context(0)
bt = nb.make_batch(tc, 4, 1)
bm = nb.make_batch(mid10, 2, 1)
def t(tag):
    r = nb.fisher_potential(tc, bt, precision=Precision.SIMT, ctx=ctx)
    print(f"{tag:40s} tc simt total {r.total:.10e} loss {r.loss:.10f}", flush=True)
t("fresh")
t("again")
nb.fisher_potential(mid10, bm, precision=Precision.SIMT, ctx=ctx); t("after mid10 simt fisher")
nb.fisher_potential(mid10, bm, precision=Precision.FP32, ctx=ctx); t("after mid10 fp32 fisher")
nb.fisher_potential(mid10, bm, precision=Precision.TF32, ctx=ctx); t("after mid10 tf32 fisher")
nb.activation_gradients(mid10, bm, precision=Precision.SIMT, ctx=ctx); t("after mid10 act_grads")
nb.fisher_potential(tc, bt, precision=Precision.FP32, ctx=ctx); t("after tc fp32")
nb.activation_gradients(tc, bt, precision=Precision.SIMT, ctx=ctx); t("after tc act_grads simt")
