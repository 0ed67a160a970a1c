"""Halo-mode determinism probe: repeated whole-batch and sharded Fisher
evaluations of R34 networks must agree bitwise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
origin = resnet34_chain()
cands = load_candidates(fixture_path("r34_candidates.json"), origin)
batch = nb.make_batch(origin, 128, 1)
whole = nb.Session(origin, batch, ctx=nb.Context(0))
shards = [nb.Session(origin, b, ctx=nb.Context(0)) for b in nb.shard_batch(batch, 2)]
for name, net in [("origin", origin), ("c0", cands[0]), ("cmid", cands[len(cands) // 2])]:
    t = [whole.fisher(net).total for _ in range(3)]
    sh = [nb.fisher_sharded(shards, net).total for _ in range(2)]
    print(name, [repr(x) for x in t], [repr(x) for x in sh], "whole-det", len(set(t)) == 1,
          "shard==whole", sh[0] == t[0], flush=True)
    pl_w = whole.fisher(net).per_layer
    pl_s = nb.fisher_sharded(shards, net).per_layer
    bad = np.nonzero(pl_w != pl_s)[0]
    print("   layers differing:", bad[:20], flush=True)
