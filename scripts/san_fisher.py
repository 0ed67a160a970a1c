"""Small Fisher run for compute-sanitizer (memcheck / racecheck / initcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision
prec = {"simt": Precision.SIMT, "fp32": Precision.FP32, "tf32": Precision.TF32}[sys.argv[1]]
net = Network([
    Layer(ConvSpec(3, 32, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(32, 64, 16, 16, 3, 3, 1, 1)),
    Layer(ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=64)),
    Layer(ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=2)),
    Layer(ConvSpec(64, 128, 16, 16, 3, 3, 2, 1)),
    Layer(ConvSpec(128, 128, 8, 8, 3, 3, 1, 1, bottleneck_out=2)),
    Layer(ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, spatial_div_h=2, spatial_div_w=2)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1, groups=64)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1)),
    Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1, groups=16)),
], num_classes=10, seed=42)
ctx = nb.Context(0)
batch = nb.make_batch(net, 4, 1)
for _ in range(2):
    print(nb.fisher_potential(net, batch, precision=prec, ctx=ctx).total, flush=True)
