"""Fisher evaluation time of 6-layer 64-channel chains at 16x16 and 8x8
(N=128): run under NB_TC_KWF=0/1 to compare kw-fused and N=64 plans."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network
ctx = nb.Context(0)
for hw in (32, 16, 8):
    net = Network([Layer(ConvSpec(3, 64, hw, hw, 3, 3, 1, 1))] +
                  [Layer(ConvSpec(64, 64, hw, hw, 3, 3, 1, 1)) for _ in range(6)],
                  num_classes=10, seed=1)
    s = nb.Session(net, nb.make_batch(net, 128, 1), ctx=ctx)
    for _ in range(3):
        s.fisher(net)
    t = time.perf_counter()
    for _ in range(10):
        r = s.fisher(net)
    print(f"KWF={os.environ.get('NB_TC_KWF', '1')} 64ch@{hw}: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms total {r.total:.6e}")
