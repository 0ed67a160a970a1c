"""CPU tests: the oracle restatement pinned against the reference's golden
fixtures (tests/golden, generated from the unmodified reference by
oracle/gen_golden.py) and, where oracle/_ref is built, against the reference
itself; plus the product's host-side draws (init_weights / make_batch) being
bit-identical to the reference's."""
import math

import numpy as np
import pytest

from conftest import golden
from paper_2102_06599_b200.api import ChannelSplit, ConvSpec, Layer, Network, make_batch

GOLD_CONV = golden("conv_cases.json")["cases"]
GOLD_FISHER = golden("fisher_nets.json")["nets"]


def _inputs(seed, spec):
    rng = np.random.default_rng(seed)
    x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
    return x, w


@pytest.mark.parametrize("case", GOLD_CONV, ids=lambda c: str(c["seed"]))
def test_restatement_conv_matches_reference_golden(oracle, case):
    spec = ConvSpec.from_json(case["spec"])
    x, w = _inputs(case["seed"], spec)
    yi = oracle.conv(spec, x, w)
    assert yi.ravel().tolist() == case["out_int"]  # int64: bit-exact
    yf = oracle.conv(spec, x.astype(np.float64) * 0.37, w.astype(np.float64) * 1.3)
    np.testing.assert_allclose(yf.ravel(), case["out_f64"], rtol=1e-13, atol=1e-12)


def test_conv_kats(oracle):
    """T/test_interp.cpp:41-50, :73-82, :96-105."""
    s = ConvSpec(1, 1, 1, 1)
    assert oracle.conv(s, np.array([[[2]]]), np.array([[[[3]]]])).ravel().tolist() == [6]
    s = ConvSpec(4, 4, 1, 1, groups=2)
    y = oracle.conv(s, np.array([1, 10, 100, 1000]).reshape(4, 1, 1), np.ones((4, 4, 1, 1), int))
    assert y.ravel().tolist() == [11, 11, 1100, 1100]
    s = ConvSpec(1, 1, 2, 2, 3, 3, 1, 1)
    y = oracle.conv(s, np.array([1, 2, 3, 4]).reshape(1, 2, 2), np.ones((1, 1, 3, 3), int))
    assert y.ravel().tolist() == [10, 10, 10, 10]


@pytest.mark.parametrize("case", GOLD_FISHER, ids=lambda c: c["name"])
def test_restatement_fisher_matches_reference_golden(oracle, case):
    net = Network.from_json(case["network"])
    r = oracle.fisher(net, case["n"], case["batch_seed"])
    assert math.isclose(r["total"], case["total"], rel_tol=1e-12)
    assert math.isclose(r["loss"], case["loss"], rel_tol=1e-13)
    np.testing.assert_allclose(r["per_layer"], case["per_layer"], rtol=1e-11, atol=0)
    scale = max(case["per_layer"])
    np.testing.assert_allclose(r["per_channel"], case["per_channel"], rtol=1e-10,
                               atol=1e-12 * scale)
    np.testing.assert_allclose(r["probs"].ravel(), case["probs"], rtol=1e-12, atol=1e-15)


def test_restatement_gradients_match_reference(oracle, reference):
    """activation_gradients (I/nnet.hpp:201-247) on a net with every feature:
    stride 2, crops, groups, splits, depthwise, a ReLU-free layer."""
    net = Network([
        Layer(ConvSpec(3, 8, 9, 9, 3, 3, 2, 1)),
        Layer(ConvSpec(8, 8, 5, 5, 3, 3, 1, 1, groups=2, spatial_div_h=5), relu=False),
        Layer(ConvSpec(8, 6, 1, 5, 1, 3, 1, 0,
                       channel_splits=[ChannelSplit(0, 2, 2), ChannelSplit(2, 6, 1)])),
        Layer(ConvSpec(6, 6, 1, 3, 3, 3, 1, 1, groups=6)),
    ], num_classes=5, seed=11)
    r = reference.fisher(net, 3, 4, grads=True)
    o = oracle.fisher(net, 3, 4, grads=True)
    np.testing.assert_allclose(o["acts"], r["acts"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(o["grads"], r["grads"], rtol=1e-10, atol=1e-16)
    assert math.isclose(o["total"], r["total"], rel_tol=1e-12)


def test_host_draws_are_bit_identical_to_reference(reference):
    """init_weights (I/nnet.hpp:58-79) and make_batch (:87-101) through the
    product's host library equal the reference's doubles bit for bit."""
    net = Network.from_json(golden("fisher_nets.json")["nets"][0]["network"])
    w_ref, h_ref = reference.init_weights(net)
    net.init_weights()
    assert np.array_equal(np.concatenate([w.ravel() for w in net.weights]), w_ref)
    assert np.array_equal(net.head.ravel(), h_ref)
    x_ref, y_ref = reference.make_batch(net, 5, 3)
    b = make_batch(net, 5, 3)
    assert np.array_equal(b.inputs, x_ref) and np.array_equal(b.labels, y_ref)


def test_weight_prefix_property(oracle):
    """A candidate's weights are a prefix of the per-layer z-stream scaled by
    its own fan-in (what lets the device draw candidates from one cache)."""
    base = Network([Layer(ConvSpec(4, 8, 4, 4, 3, 3, 1, 1))], num_classes=3, seed=5)
    cand = Network([Layer(ConvSpec(4, 8, 4, 4, 3, 3, 1, 1, bottleneck_out=2))], num_classes=3,
                   seed=5)
    wb, _ = oracle.init_weights(base)
    wc, _ = oracle.init_weights(cand)
    assert np.array_equal(wc, wb[:wc.size])


def test_zero_weights_kat(oracle):
    """T/test_nnet.cpp:35-44 and :180-186: zero weights give loss ln(K) and
    Fisher 0."""
    net = Network([Layer(ConvSpec(2, 4, 5, 5, 3, 3, 1, 1)), Layer(ConvSpec(4, 4, 5, 5, 3, 3, 1, 1)),
                   Layer(ConvSpec(4, 3, 5, 5))], num_classes=4, seed=42)
    net.init_weights()
    net.weights = [np.zeros_like(w) for w in net.weights]
    net.head = np.zeros_like(net.head)
    r = oracle.fisher(net, 8, 1)
    assert math.isclose(r["loss"], math.log(4.0), rel_tol=1e-12)
    assert r["total"] == 0.0
