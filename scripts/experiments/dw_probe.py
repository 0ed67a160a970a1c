"""One depthwise 3x3 64@56 forward at N=256 (ncu target for the dw kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network
c, hw = int(os.environ.get("DW_C", "64")), int(os.environ.get("DW_HW", "56"))
net = Network([Layer(ConvSpec(c, c, hw, hw, 3, 3, 1, 1, groups=c))], num_classes=10, seed=42)
s = nb.Session(net, nb.make_batch(net, 256, 1), ctx=nb.Context(0))
for _ in range(3):
    s.forward(net)
