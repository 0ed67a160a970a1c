"""Edge cases of the GPU path: degenerate shapes the transformation search
produces (1x1 crops, Co_eff = 1, G = Ci depthwise at 512 channels, 16
channel ranges), single-example and large batches, and the error classes
of the reference for bad inputs (I/errors.hpp)."""
import math

import numpy as np
import pytest

import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ChannelSplit, ConvSpec, Layer, Network, Precision

pytestmark = pytest.mark.gpu
TOT = nb.TOLERANCE[Precision.FP32]["total"]


def _check(ctx, oracle, net, n, prec=Precision.FP32, seed=1):
    batch = nb.make_batch(net, n, seed)
    rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
    o = oracle.fisher(net, n, batch=batch)
    tol = nb.TOLERANCE[prec]["total"]
    if o["total"] == 0.0:
        assert rep.total == 0.0
    else:
        assert math.isclose(rep.total, o["total"], rel_tol=tol), (rep.total, o["total"])
    assert math.isclose(rep.loss, o["loss"], rel_tol=1e-6)


def test_crop_to_one_pixel_and_single_output_channel(ctx, oracle):
    """SURVEY finding 12: a 32x crop leaves out_h = 1; bottleneck can take
    Co_eff down to 1."""
    net = Network([Layer(ConvSpec(3, 32, 32, 32, 3, 3, 1, 1, spatial_div_h=32, spatial_div_w=32)),
                   Layer(ConvSpec(32, 64, 1, 1, 3, 3, 1, 1, bottleneck_out=64)),
                   Layer(ConvSpec(1, 8, 1, 1, 1, 1, 1, 0))], num_classes=10, seed=42)
    _check(ctx, oracle, net, 4)


def test_wide_depthwise_and_many_groups(ctx, oracle):
    net = Network([Layer(ConvSpec(3, 512, 8, 8, 3, 3, 1, 1)),
                   Layer(ConvSpec(512, 512, 8, 8, 3, 3, 1, 1, groups=512)),
                   Layer(ConvSpec(512, 256, 8, 8, 3, 3, 2, 1, groups=128)),
                   Layer(ConvSpec(256, 256, 4, 4, 3, 3, 1, 1, groups=64))], num_classes=10, seed=7)
    _check(ctx, oracle, net, 3)


def test_sixteen_channel_ranges(ctx, oracle):
    splits = [ChannelSplit(4 * i, 4 * i + 4, 2 if i % 2 else 1) for i in range(16)]
    net = Network([Layer(ConvSpec(4, 64, 6, 6, 3, 3, 1, 1, channel_splits=splits)),
                   Layer(ConvSpec(64, 8, 6, 6, 3, 3, 1, 1))], num_classes=5, seed=3)
    _check(ctx, oracle, net, 2)


def test_more_than_sixteen_ranges_is_unsupported(ctx):
    splits = [ChannelSplit(i, i + 1, 1) for i in range(17)]
    net = Network([Layer(ConvSpec(4, 17, 4, 4, 3, 3, 1, 1, channel_splits=splits))],
                  num_classes=3, seed=1)
    with pytest.raises(nb.Unsupported):
        nb.fisher_potential(net, nb.make_batch(net, 1, 1), ctx=ctx)


@pytest.mark.parametrize("n", [1, 2, 129])
def test_batch_sizes(ctx, oracle, n):
    net = Network([Layer(ConvSpec(3, 32, 8, 8, 3, 3, 1, 1)), Layer(ConvSpec(32, 32, 8, 8, 3, 3, 1, 1)),
                   Layer(ConvSpec(32, 64, 8, 8, 3, 3, 2, 1))], num_classes=10, seed=42)
    _check(ctx, oracle, net, n)


def test_no_relu_chain_and_two_classes(ctx, oracle):
    net = Network([Layer(ConvSpec(2, 32, 5, 5, 3, 3, 1, 1), relu=False),
                   Layer(ConvSpec(32, 32, 5, 5, 3, 3, 1, 1), relu=False)], num_classes=2, seed=9)
    for prec in (Precision.SIMT, Precision.FP32):
        _check(ctx, oracle, net, 3, prec)


def test_error_classes(ctx):
    net = Network([Layer(ConvSpec(3, 8, 4, 4, 3, 3, 1, 1))], num_classes=4, seed=1)
    with pytest.raises(nb.ConfigError):
        nb.fisher_potential(net, nb.Batch(np.zeros((0, 3, 4, 4)), np.zeros(0, np.int32)), ctx=ctx)
    with pytest.raises(nb.ConfigError, match="label"):
        nb.fisher_potential(net, nb.Batch(np.zeros((1, 3, 4, 4)), np.array([7], np.int32)),
                            ctx=ctx)
    bad = Network([Layer(ConvSpec(3, 8, 4, 4, 3, 3, 1, 1)), Layer(ConvSpec(4, 8, 4, 4))],
                  num_classes=4)
    with pytest.raises(nb.ConfigError, match="input shape"):
        nb.fisher_potential(bad, nb.make_batch(net, 1, 1), ctx=ctx)
    with pytest.raises(nb.InvalidSpec):
        nb.reference_conv(ConvSpec(4, 6, 4, 4, groups=4), np.zeros((4, 4, 4)), np.zeros((6, 4, 1, 1)),
                          ctx=ctx)
    with pytest.raises(nb.ShapeMismatch):
        nb.reference_conv(ConvSpec(4, 4, 4, 4), np.zeros((3, 4, 4)), np.zeros((4, 4, 1, 1)), ctx=ctx)
    sess = nb.Session(net, nb.make_batch(net, 2, 1), ctx=ctx)
    other = Network([Layer(ConvSpec(3, 8, 5, 5, 3, 3, 1, 1))], num_classes=4)
    with pytest.raises(nb.ShapeMismatch):
        sess.fisher(other)
