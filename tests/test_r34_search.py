"""Decision parity of the GPU search driver at the benchmarked configuration:
the reference's per-layer neural search on the 33-layer ResNet-34 CIFAR chain
at batch N=128 (BASELINE configs[1]; north_star: "matching the reference's
selected candidates").

Goldens tests/golden/r34_search_m{M}.json (oracle/gen_r34_golden.py): the
reference's draw_candidates and evaluate_candidate gates, fisher_potential of
every neural candidate's network at N=128 by the fp64 oracle (pinned to the
reference), fisher_accepts (>=) and rank_survivors.  run_search_gpu
(integration/nestopt_b200.hpp, I/search.hpp:364-393) must give the same
statuses, the same survivors in the same order and the same selected
candidate; Fisher totals within the deep-chain tolerance
(paper_2102_06599_b200/api.py TOLERANCE_DEEP); any decision the golden puts
inside the documented tie band (api.py TIE_BAND) is exempt.
"""
import glob
import math
import os

import pytest

from conftest import GOLDEN, golden
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from paper_2102_06599_b200 import search as S

FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "r34_search_m*.json")))
NEEDS_LIB = pytest.mark.skipif(not os.path.exists(S.SO), reason="integration library not built")


@pytest.mark.parametrize("name", FILES)
def test_r34_search_golden_is_the_reference_pipeline(name):
    """CPU: the golden's config is the bench's per-layer search at N=128 and
    its report is internally consistent (statuses, counts, ranking rule)."""
    g = golden(name)
    cfg = g["config"]
    assert cfg["batch"] == {"n": 128, "seed": 1} and sum(cfg["layer_mask"]) == 1
    c = g["candidates"]
    assert len(c) == cfg["candidate_count"]
    surv = [x["index"] for x in c if x["status"] == "survivor"]
    assert len(surv) == g["stats"]["survivors"]
    assert sorted(surv, key=lambda i: (c[i]["macs"], -c[i]["fisher_total"], i)) == \
        g["survivors_ranked"]
    o = g["origin"]["fisher_total"]
    for x in c:
        if x["status"] == "rejected_fisher":
            assert x["fisher_total"] < o
        elif x["status"] == "survivor" and x["neural"]:
            assert x["fisher_total"] >= o


@pytest.mark.gpu
@NEEDS_LIB
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32], ids=["fp32_3xtf32", "tf32"])
@pytest.mark.parametrize("name", FILES)
def test_r34_search_matches_reference(name, prec):
    g = golden(name)
    rep = S.run_search_gpu(g["config"], "0", precision=prec)
    tol = nb.TOLERANCE_DEEP[prec]["total"]
    o = g["origin"]["fisher_total"]
    assert rep["origin"]["macs"] == g["origin"]["macs"]
    assert math.isclose(rep["origin"]["fisher_total"], o, rel_tol=tol)
    exempt = set()
    for a, b in zip(rep["candidates"], g["candidates"]):
        assert a["index"] == b["index"] and a["sequences"] == b["sequences"]
        assert a["macs"] == b["macs"] and a["neural"] == b["neural"]
        if b["status"] == "rejected_semantic":
            assert a["status"] == b["status"] and a.get("reason") == b.get("reason")
            continue
        assert math.isclose(a["fisher_total"], b["fisher_total"], rel_tol=max(tol, 3e-4)), \
            (b["index"], a["fisher_total"], b["fisher_total"])
        if a["status"] != b["status"]:
            assert abs(b.get("relative_margin", 0.0)) <= nb.TIE_BAND, (b["index"], a, b)
            exempt.add(b["index"])
    if not exempt:
        assert rep["stats"]["survivors"] == g["stats"]["survivors"]
        assert rep["stats"]["rejected_fisher"] == g["stats"]["rejected_fisher"]
        assert rep["survivors_ranked"] == g["survivors_ranked"]
    # the candidate the search selects (survivors_ranked.front(), I/search.hpp:381)
    assert rep["survivors_ranked"][0] == g["survivors_ranked"][0]
    assert rep["gpu"]["legality_host"] == 0
