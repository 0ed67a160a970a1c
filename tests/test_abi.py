"""CPU tests of the C ABI: the library loads, exports exactly what
include/nb200.h declares, and its host-side logic (validation, MAC counts,
repair, LPT) matches the reference.  No compute calls without a GPU."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import abi


def test_library_exports_every_declared_symbol():
    lib = abi.load()
    hdr = open(os.path.join(ROOT, "include", "nb200.h")).read()
    declared = set(re.findall(r"\b(nb_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(abi.SIGNATURES), declared ^ set(abi.SIGNATURES)
    assert abi.load().nb_abi_version() == 2


def test_spec_validation_errors():
    with pytest.raises(nb.InvalidSpec, match="divisible by groups"):
        nb.ConvSpec(4, 6, 4, 4, groups=4).validate()
    with pytest.raises(nb.InvalidSpec, match="kernel larger"):
        nb.ConvSpec(1, 1, 1, 1, 3, 3).validate()
    with pytest.raises(nb.InvalidSpec, match="contiguous"):
        nb.ConvSpec(4, 4, 2, 2, channel_splits=[nb.ChannelSplit(1, 4, 1)]).validate()
    nb.ConvSpec(4, 8, 4, 4, 3, 3, 1, 1, groups=2, bottleneck_out=2).validate()


def test_network_validation_catches_shape_breaks():
    """T/test_nnet.cpp:56-63."""
    net = nb.Network([nb.Layer(nb.ConvSpec(2, 4, 5, 5, 3, 3, 1, 1)),
                      nb.Layer(nb.ConvSpec(4, 4, 5, 5, 3, 3, 1, 1))], num_classes=4)
    net.validate()
    net.layers[1].spec.ci = 3
    with pytest.raises(nb.ConfigError):
        net.validate()
    net.layers[1].spec.ci = 4
    net.layers[1].spec.h = 4
    with pytest.raises(nb.ConfigError):
        net.validate()


@pytest.mark.parametrize("case", golden("conv_cases.json")["cases"], ids=lambda c: str(c["seed"]))
def test_macs_match_reference_count_macs(case):
    assert nb.count_macs(nb.ConvSpec.from_json(case["spec"])) == case["macs"]


def test_derived_spec_macs_match_reference():
    for c in golden("sequences.json")["cases"]:
        if c["derived_spec"] is not None:
            assert nb.count_macs(nb.ConvSpec.from_json(c["derived_spec"])) == c["macs"], c["dsl"]


def test_repair_propagates_shapes():
    """T/test_nnet.cpp:202-215."""
    net = nb.Network([nb.Layer(nb.ConvSpec(2, 4, 5, 5, 3, 3, 1, 1)),
                      nb.Layer(nb.ConvSpec(4, 4, 5, 5, 3, 3, 1, 1)),
                      nb.Layer(nb.ConvSpec(4, 3, 5, 5))], num_classes=4, seed=42)
    net.layers[0].spec.bottleneck_out = 2
    nb.repair_network(net)
    assert net.layers[1].spec.ci == 2
    net.init_weights()
    assert net.weights[1].shape == (4, 2, 3, 3)
    net.layers[1].spec.set_bottleneck_spatial(5)
    nb.repair_network(net)
    assert (net.layers[2].spec.h, net.layers[2].spec.w) == (1, 1)


def test_lpt_is_deterministic_and_balanced():
    rng = np.random.default_rng(0)
    costs = rng.uniform(1, 10, 200)
    a = nb.schedule_lpt(costs, 8)
    assert a == nb.schedule_lpt(costs, 8)
    loads = np.bincount(a, weights=costs, minlength=8)
    assert loads.max() - loads.min() <= costs.max()
    assert loads.max() / loads.mean() < 1.05


def test_fisher_flops_is_fprop_plus_dgrad():
    net = nb.Network([nb.Layer(nb.ConvSpec(3, 8, 8, 8, 3, 3, 1, 1)),
                      nb.Layer(nb.ConvSpec(8, 8, 8, 8, 3, 3, 1, 1))])
    m0, m1 = (nb.count_macs(l.spec) for l in net.layers)
    assert nb.fisher_flops(net, 4) == 2 * 4 * (m0 + m1 + m1)
    assert nb.network_macs(net) == m0 + m1


@pytest.mark.skipif(abi.load().nb_device_count() > 0, reason="a GPU is visible")
def test_no_cpu_fallback_without_gpu():
    """Every compute entry point fails loudly (NoDevice) without a B200."""
    with pytest.raises(nb.NoDevice):
        nb.Context(0)
