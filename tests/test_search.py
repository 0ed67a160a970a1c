"""The GPU search driver (integration/nestopt_b200.hpp run_search_gpu) against
the reference's own search reports (tests/golden/search_toy_*.json,
generated from the unmodified reference by oracle/gen_golden.py and
oracle/gen_search_golden.py).

Decision parity: every candidate's status is identical to the reference's.
Candidates scored within the mode's stated tolerance of the origin (the
near-threshold band, nb.RECHECK_BAND) are re-scored in SIMT mode (fp32
FFMA, 1e-5 of the fp64 reference) before the decision, so only ties closer
than SIMT's tolerance could differ (none occur in these fixtures); networks
identical to the origin are exact ties by construction.  Fisher totals agree
within the mode's stated tolerance; reports are bitwise identical for any
number of GPU sessions.
"""
import json
import math
import os

import pytest

from conftest import golden
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from paper_2102_06599_b200 import search as S

TOL_TOTAL = nb.TOLERANCE[Precision.FP32]["total"]
NEEDS_LIB = pytest.mark.skipif(not os.path.exists(S.SO), reason="integration library not built")


@NEEDS_LIB
def test_integration_library_exports_and_fails_loudly_without_gpu():
    lib = S.load()
    for sym in ("nbi_run_search", "nbi_last_error", "nbi_free"):
        assert hasattr(lib, sym)
    import paper_2102_06599_b200 as nb
    if nb.device_count() > 0:
        pytest.skip("a GPU is visible")
    cfg = dict(golden("search_toy_100.json")["config"])
    cfg["network"] = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                                 "search_toy_1000.json")))["config"]["network"]
    with pytest.raises(Exception, match="no CUDA device|no CPU fallback"):
        S.run_search_gpu(cfg)


@NEEDS_LIB
def test_host_gates_match_reference_on_cpu():
    """nb200::host_gates (evaluate_candidate up to the Fisher call, re-composed
    from the reference's apply / check_semantic_legality / derived_spec) give
    the reference's semantic rejections (same reasons), non-neural survivors
    and MAC counts on the 1000-candidate toy search; every candidate they send
    to the GPU is one the reference scored."""
    g = golden("search_toy_1000.json")
    gated = S.gate_candidates(g["config"])
    assert len(gated) == len(g["candidates"])
    for i, (a, b) in enumerate(zip(gated, g["candidates"])):
        assert a["macs"] == b["macs"], i
        if a["status"] == "fisher":
            assert b["neural"] and b["status"] in ("survivor", "rejected_fisher"), i
            assert "network" in a
        else:
            assert a["status"] == b["status"], i
            assert a.get("reason", "") == b.get("reason", ""), i
            if a["status"] == "survivor":
                assert not b["neural"]


def _cfg100():
    g = golden("search_toy_100.json")
    cfg = dict(g["config"])
    cfg["network"] = golden("search_toy_1000.json")["config"]["network"]
    return g, cfg


def _reason_number(r):
    # "fisher potential dropped: A < B"
    return float(r.split(":")[1].split("<")[0])


def _check_candidates(got, want, origin, tol=TOL_TOTAL):
    near = 0
    simt = nb.TOLERANCE[Precision.SIMT]["total"]
    for i, (g, w) in enumerate(zip(got, want)):
        assert g["macs"] == w["macs"], i
        assert g["neural"] == w["neural"], i
        if "fisher_total" in w:
            assert math.isclose(g["fisher_total"], w["fisher_total"], rel_tol=tol), i
        if g["status"] != w["status"]:
            # only a tie closer than SIMT's tolerance may flip (none expected)
            assert abs(w["fisher_total"] - origin) / origin < simt, (i, g, w)
            near += 1
            continue
        if w["status"] == "rejected_fisher":
            assert math.isclose(_reason_number(g["reason"]), _reason_number(w["reason"]),
                                rel_tol=max(tol, 1e-5) + 1e-5)
        else:
            assert g.get("reason", "") == w.get("reason", ""), i
    return near


@pytest.mark.gpu
@NEEDS_LIB
def test_search_toy_100_matches_reference_report():
    g, cfg = _cfg100()
    rep = S.run_search_gpu(cfg, "0")
    assert rep["stats"] == g["stats"]
    assert rep["origin"]["macs"] == g["origin"]["macs"]
    assert math.isclose(rep["origin"]["fisher_total"], g["origin"]["fisher_total"],
                        rel_tol=TOL_TOTAL)
    for a, b in zip(rep["candidates"], g["candidates"]):
        assert a["sequences"] == b["sequences"] and a["index"] == b["index"]
    assert _check_candidates(rep["candidates"], g["candidates"],
                             g["origin"]["fisher_total"]) == 0
    assert rep["survivors_ranked"] == g["survivors_ranked"]
    assert rep["config"] == g["config"]


@pytest.mark.gpu
@NEEDS_LIB
def test_search_toy_1000_decisions_match_reference():
    """acceptance criterion 7 (T/acceptance.cpp:406-433): 220 survivors /
    100 semantic / 680 Fisher rejections, best index 103."""
    g = golden("search_toy_1000.json")
    rep = S.run_search_gpu(g["config"], "0", jobs=8)
    assert rep["stats"] == g["stats"]
    assert _check_candidates(rep["candidates"], g["candidates"],
                             g["origin"]["fisher_total"]) == 0
    assert rep["survivors_ranked"] == g["survivors_ranked"]
    assert rep["survivors_ranked"][0] == 103
    assert rep["gpu"]["deduplicated"] > 0
    # every semantic run of the all-kinds gates was checked on the GPU
    assert rep["gpu"]["legality_gpu"] > 0 and rep["gpu"]["legality_host"] == 0


@pytest.mark.gpu
@NEEDS_LIB
def test_search_report_independent_of_session_count():
    """T/test_search.cpp:83-94 (jobs=4 == jobs=1), for GPU sessions: the
    candidates are sharded by LPT over 1 or 3 sessions and the report (minus
    timing and the gpu block) is bitwise identical."""
    _, cfg = _cfg100()
    a = S.run_search_gpu(cfg, "0")
    b = S.run_search_gpu(cfg, "0,0,0")
    for r in (a, b):
        r.pop("timing")
        r.pop("gpu")
    assert json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)


@pytest.mark.gpu
@NEEDS_LIB
def test_tf32_search_with_near_tie_recheck_matches_reference():
    """The TF32 throughput mode plus the SIMT re-score of near-threshold
    candidates makes the reference's decisions on the 1000-candidate search."""
    g = golden("search_toy_1000.json")
    rep = S.run_search_gpu(g["config"], "0", precision=Precision.TF32, jobs=8)
    assert rep["stats"] == g["stats"]
    assert _check_candidates(rep["candidates"], g["candidates"], g["origin"]["fisher_total"],
                             tol=nb.TOLERANCE[Precision.TF32]["total"]) == 0
    assert rep["gpu"]["rechecked"] > 0


@NEEDS_LIB
def test_parallel_draw_matches_reference_draw():
    """nb200::draw_candidates (index-parallel) draws exactly
    the reference's draw_candidates (I/search.hpp:188-214): same steps for
    every candidate and layer, all kinds, two configs."""
    from paper_2102_06599_b200.workloads import resnet34_chain
    g = golden("search_toy_1000.json")
    assert S.draw_candidates(g["config"], 0) == S.draw_candidates(g["config"], 8)
    o = resnet34_chain().to_json()
    cfg = {"schema_version": 1, "candidate_count": 150, "max_seq_len": 6, "seed": 11,
           "batch": {"n": 8, "seed": 1}, "network": o}
    ref = S.draw_candidates(cfg, 0)
    assert ref == S.draw_candidates(cfg, 5)
    assert any(c["neural"] for c in ref)
