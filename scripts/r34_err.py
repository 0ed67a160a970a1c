"""Per-layer relative Fisher error of every precision mode at the bench
config (R34 chain, N=128) against tests/golden/r34_n128.* (GPU experiment)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from test_r34_parity import _nets
from paper_2102_06599_b200.workloads import resnet34_chain
o = resnet34_chain()
s = nb.Session(o, nb.make_batch(o, 128, 1), ctx=nb.Context(0))
for e, net, pc, probs in _nets():
    line = [f"{e['name']:8s} {e['kind']:16s}"]
    for name, p in ((nb.fp32_split(), Precision.FP32), ("simt", Precision.SIMT), ("tf32", Precision.TF32)):
        r = s.fisher(net, p)
        pl = np.array(e["per_layer"])
        le = np.abs(r.per_layer - pl) / np.abs(pl)
        line.append(f"{name} tot {(r.total - e['total']) / e['total']:+.2e} "
                    f"layer max {le.max():.1e}@{int(le.argmax())}")
    print("  ".join(line), flush=True)
