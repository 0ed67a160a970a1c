import os, sys
sys.path.insert(0, os.getcwd())
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
origin = resnet34_chain()
c0 = load_candidates(fixture_path("r34_candidates.json"), origin)[0]
batch = nb.make_batch(origin, 128, 1)
which = sys.argv[1]
if which == "whole":
    s = nb.Session(origin, batch, ctx=nb.Context(0)); print(s.fisher(c0).total)
else:
    sh = [nb.Session(origin, b, ctx=nb.Context(0)) for b in nb.shard_batch(batch, 2)]
    print(nb.fisher_sharded(sh, c0).total)
