"""Semantic legality on the GPU (nb_semantic_legality, driven by
integration/nestopt_b200.hpp nb200::check_semantic_legality) against the
reference's check_semantic_legality (I/transforms.hpp:598-663).

tests/golden/legality_cases.json (oracle/gen_legality_golden.py) holds the
reference's verdict and reason for the reference tests' hand-injected
rewrites, random semantic runs and nests near the 1e6-instance cap.  The bar
is exact: same verdict, same reason string -- including which dependence is
reported first -- and the same CapExceeded throws.
"""
import json
import os

import pytest

from conftest import golden
from paper_2102_06599_b200 import search as S

NEEDS_LIB = pytest.mark.skipif(not os.path.exists(S.SO), reason="integration library not built")
CASES = golden("legality_cases.json")
SMALL = [c for c in CASES if not c["name"].startswith("big_")]


def _ids(cases):
    return [c["name"] for c in cases]


@NEEDS_LIB
@pytest.mark.parametrize("case", SMALL, ids=_ids(SMALL))
def test_host_check_reproduces_golden(case):
    """The fixtures are the reference's own verdicts (nest JSON round trip)."""
    res, _ = S.legality_nests(case["original"], case["transformed"], case["cap"], device=-1)
    assert res.pop("path", "host") == "host"
    assert res == case["expected"]


@NEEDS_LIB
def test_fixture_coverage():
    verdicts = {c["expected"].get("verdict", c["expected"].get("error")) for c in CASES}
    assert verdicts == {"legal", "illegal", "not_applicable", "CapExceeded"}
    reasons = {c["expected"].get("reason", "") for c in CASES}
    assert "transformed schedule duplicates an instance" in reasons
    assert any(r.startswith("dependence S1(0,14,0)") for r in reasons)
    assert sum(c["name"].startswith("big_") for c in CASES) >= 8


@NEEDS_LIB
@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=_ids(CASES))
def test_gpu_legality_matches_reference(case):
    res, ms = S.legality_nests(case["original"], case["transformed"], case["cap"], device=0)
    if "error" not in res:  # (CapExceeded is decided from instance counts first)
        assert res.pop("path") == "gpu", res  # answered by the device, no host fallback
    assert res == case["expected"], (res, case["expected"])
    if case["name"].startswith("big_") and "error" not in res:
        print(f'{case["name"]}: gpu {ms:.1f} ms vs reference host {case["host_ms"]:.0f} ms')


@NEEDS_LIB
@pytest.mark.gpu
def test_gpu_legality_through_dsl():
    """The DSL path (conv_nest + apply on the bridge side) at sizes around the
    kernel's limits: extents not powers of two, kernel 1x1 (no kh/kw loops),
    a neural prefix before the semantic run."""
    cases = [
        ({"ci": 3, "co": 5, "h": 7, "w": 9, "kh": 3, "kw": 3, "pad": 1}, "", "fuse(h,w) | tile(h_w,3)"),
        ({"ci": 16, "co": 8, "h": 14, "w": 14}, "", "interchange(co,ci) | unroll(w,7)"),
        ({"ci": 8, "co": 8, "h": 12, "w": 12, "kh": 3, "kw": 3, "pad": 1}, "bottleneck(co,2)",
         "strip_mine(ci,4) | interchange(ci_o,kw)"),
        ({"ci": 8, "co": 8, "h": 12, "w": 12, "kh": 3, "kw": 3, "pad": 1}, "group(co,ci,2)",
         "split(ci,1,3)"),
    ]
    for spec, pre, seq in cases:
        host, _ = S.legality(spec, seq, pre=pre, device=-1)
        gpu, _ = S.legality(spec, seq, pre=pre, device=0)
        assert host.pop("path") == "host" and gpu.pop("path") == "gpu"
        assert gpu == host, (spec, pre, seq)


@NEEDS_LIB
@pytest.mark.gpu
def test_gates_with_gpu_legality_match_host():
    """evaluate_candidate's gates with every semantic run checked on the GPU
    (no host fallback, whatever the nest size: the path counters prove it)
    give the same statuses, reasons and MACs as with the reference's host
    check, on the all-kinds toy search (the reference's default kinds)."""
    g = golden("search_toy_1000.json")
    cfg = dict(g["config"])
    cfg.pop("kinds", None)  # reference default: all seven kinds
    cfg["candidate_count"] = 300
    host, hc = S.gate_candidates(cfg, legal_device=-1, with_counts=True)
    gpu, gc = S.gate_candidates(cfg, legal_device=0, with_counts=True)
    assert hc["gpu"] == 0 and hc["host"] > 0
    assert gc["host"] == 0 and gc["gpu"] == hc["host"], gc
    assert [(c["status"], c.get("reason"), c["macs"]) for c in gpu] == \
           [(c["status"], c.get("reason"), c["macs"]) for c in host]
    assert any("reordered" in (c.get("reason") or "") or "duplicates" in (c.get("reason") or "")
               or c["status"] != "rejected_semantic" for c in host)
