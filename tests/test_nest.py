"""The general loop-nest executor (nb_nest_execute via the bridge's
nb200::execute) against the reference's execute (I/interp.hpp:67-145) on
conv nests rewritten by DSL sequences -- including the paper's Sequence 1,
which has no ConvSpec (tests/golden/nest_cases.json, generated from the
unmodified reference by oracle/gen_nest_golden.py).  int64: bit-exact;
fp64: 1e-12 relative (atomic accumulation order)."""
import os

import numpy as np
import pytest

from conftest import golden
from paper_2102_06599_b200 import ConvSpec
from paper_2102_06599_b200 import search as S

CASES = golden("nest_cases.json")["cases"]
NEEDS_LIB = pytest.mark.skipif(not os.path.exists(S.SO), reason="integration library not built")


def test_fixture_covers_forms_without_a_convspec():
    no_spec = [c for c in CASES if not c["has_spec"]]
    assert len(no_spec) >= 10 and all(c["dsl"].startswith("sequence1") for c in no_spec)


@NEEDS_LIB
def test_integration_exports_execute():
    assert hasattr(S.load(), "nbi_execute")


@pytest.mark.gpu
@NEEDS_LIB
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['seed']}-{c['dsl']}")
def test_gpu_execute_matches_reference(case):
    spec = ConvSpec.from_json(case["spec"])
    rng = np.random.default_rng(case["seed"])
    x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
    y = S.execute_gpu(spec, case["dsl"], x, w)
    assert y.ravel().tolist() == case["out_int"]
    yf = S.execute_gpu(spec, case["dsl"], x * 0.37, w * 1.3)
    np.testing.assert_allclose(yf.ravel(), case["out_f64"], rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@NEEDS_LIB
def test_gpu_execute_sequence1_structure():
    """Sequence 1 is spatially block-diagonal: in the
    top H/arity rows output-channel block g is computed only for row block g;
    the other cells stay zero, the bottom rows are a dense conv."""
    spec = ConvSpec(8, 16, 8, 8, 3, 3, 1, 1)
    x = np.ones((8, 8, 8), np.int64)
    w = np.ones((16, 8, 3, 3), np.int64)
    y = S.execute_gpu(spec, "sequence1(2,2)", x, w)
    dense = S.execute_gpu(spec, "", x, w)
    assert np.array_equal(y[:, 4:], dense[:, 4:])
    top = y[:, :4]
    assert (top == 0).any() and (top != 0).any()


# ---- the masked box executor (execute_boxes) ----------------

@pytest.mark.gpu
@NEEDS_LIB
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['seed']}-{c['dsl']}")
def test_gpu_box_executor_matches_reference(case):
    """Every golden nest (Sequence-1 forms included) on the tensor cores
    through execute_boxes: int64 bit-exact against the reference's execute;
    fp64 inputs within the FP32 tier's conv tolerance (relative to the
    output's scale); the boxes cover exactly the nest's MACs."""
    import paper_2102_06599_b200 as nb
    spec = ConvSpec.from_json(case["spec"])
    rng = np.random.default_rng(case["seed"])
    x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
    y, st = S.execute_boxes_gpu(spec, case["dsl"], x, w)
    assert y.ravel().tolist() == case["out_int"]
    assert st["box_macs"] == st["nest_macs"] == case["macs"] and st["boxes"] >= 1
    yf, _ = S.execute_boxes_gpu(spec, case["dsl"], x * 0.37, w * 1.3)
    ref = np.asarray(case["out_f64"])
    scale = np.abs(ref).max() or 1.0
    tol = nb.TOLERANCE[nb.Precision.FP32]["conv"]
    assert np.abs(yf.ravel() - ref).max() <= tol * scale * spec.ci * spec.kh * spec.kw


@pytest.mark.gpu
@NEEDS_LIB
def test_gpu_box_executor_sequence1_boxes():
    """Sequence 1 (arity 2, G 2) decomposes into one box per top row block
    (its output-channel block) and one dense box over the bottom half --
    G + 1 boxes, no MAC computed twice, none skipped."""
    spec = ConvSpec(8, 16, 8, 8, 3, 3, 1, 1)
    rng = np.random.default_rng(3)
    x = rng.integers(-3, 4, size=(8, 8, 8)).astype(np.int64)
    w = rng.integers(-3, 4, size=(16, 8, 3, 3)).astype(np.int64)
    y, st = S.execute_boxes_gpu(spec, "sequence1(2,2)", x, w)
    assert st["boxes"] == 3 and st["box_macs"] == st["nest_macs"]
    assert np.array_equal(y, S.execute_gpu(spec, "sequence1(2,2)", x, w))
