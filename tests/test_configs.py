"""Parity at the shapes of every BASELINE.json config (the non-headline
configs are parity cases, not bench lines):

  C1  single 3x3 conv 64->64 32x32 N=8, standard / grouped g=4 / bottleneck b=2
      -- Fisher totals of the UNMODIFIED reference (BASELINE.md section 2,
      measured with oracle/_ref during the survey);
  C2  the ResNet-34 CIFAR chain -- the reference's N=1 total and
      the fp64 oracle at N=2;
  C3  the ResNeXt-29 (2x64d) chain, grouped 3x3 convs, and its Sequence-3
      (channel-split) / Sequence-2 (grouped) rewrites of a block;
  C4  DenseNet-161 dense layers (2-conv chains) with bottleneck / depthwise
      candidates;
  C5  ImageNet-shape convs (56/28/14/7 spatial, groups 1..C): conv fprop and
      dgrad against the oracle.

Tolerances are the precision tiers of tests/test_gpu_parity.py.
"""
import math

import numpy as np
import pytest

import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ChannelSplit, ConvSpec, Layer, Network, Precision
from paper_2102_06599_b200.workloads import (c1_network, densenet161_layer_chains,
                                             resnet34_chain, resnext29_chain)

pytestmark = pytest.mark.gpu
TOT = {p: t["total"] for p, t in nb.TOLERANCE.items()}
LAYER = {p: t["layer"] for p, t in nb.TOLERANCE.items()}

# BASELINE.md section 2 (reference fisher_potential, N=8, batch seed 1, net seed 42)
C1_REF = {(1, 1): 1.0650840122724437e-3, (4, 1): 2.6306236713211252e-4,
          (1, 2): 1.2464151317626677e-3}


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.SIMT, Precision.TF32])
@pytest.mark.parametrize("gb", sorted(C1_REF), ids=lambda gb: f"g{gb[0]}b{gb[1]}")
def test_c1_fisher_matches_reference(ctx, gb, prec):
    net = c1_network(groups=gb[0], bottleneck=gb[1])
    rep = nb.fisher_potential(net, nb.make_batch(net, 8, 1), precision=prec, ctx=ctx)
    assert math.isclose(rep.total, C1_REF[gb], rel_tol=TOT[prec]), (rep.total, C1_REF[gb])


def _vs_oracle(ctx, oracle, net, n, prec):
    batch = nb.make_batch(net, n, 1)
    rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
    o = oracle.fisher(net, n, batch=batch)
    assert math.isclose(rep.total, o["total"], rel_tol=TOT[prec]), (rep.total, o["total"])
    np.testing.assert_allclose(rep.per_layer, o["per_layer"], rtol=LAYER[prec])
    assert math.isclose(rep.loss, o["loss"], rel_tol=1e-6)
    return rep, o


def test_r34_chain_reference_total_n1(ctx):
    """reference fisher_potential of the R34 chain at N=1 =
    8.2040586242701433e-12 (loss 2.3025833612483151)."""
    net = resnet34_chain()
    rep = nb.fisher_potential(net, nb.make_batch(net, 1, 1), ctx=ctx)
    assert math.isclose(rep.total, 8.2040586242701433e-12, rel_tol=TOT[Precision.FP32])
    assert math.isclose(rep.loss, 2.3025833612483151, rel_tol=1e-9)


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32])
def test_r34_chain_vs_oracle_n2(ctx, oracle, prec):
    _vs_oracle(ctx, oracle, resnet34_chain(), 2, prec)


def test_resnext29_chain_vs_oracle(ctx, oracle):
    _vs_oracle(ctx, oracle, resnext29_chain(), 2, Precision.FP32)


def test_resnext29_sequence_rewrites_vs_oracle(ctx, oracle):
    """A ResNeXt block's 3x3 grouped conv rewritten to the paper's Sequence 3
    (channel splits g2 | g4, I/transforms.hpp:560-582) and Sequence 2
    (grouped G=2 + unroll hint), then shape-repaired."""
    base = resnext29_chain()
    for splits in ([ChannelSplit(0, 64, 2), ChannelSplit(64, 128, 4)],
                   [ChannelSplit(0, 32, 1), ChannelSplit(32, 128, 8)]):
        net = base.copy()
        net.layers[2].spec.channel_splits = splits
        nb.repair_network(net)
        _vs_oracle(ctx, oracle, net, 2, Precision.FP32)


@pytest.mark.parametrize("which", [0, 6, 18, 54, 77])
def test_densenet_dense_layers_vs_oracle(ctx, oracle, which):
    chain = densenet161_layer_chains()[which]
    _vs_oracle(ctx, oracle, chain, 4, Precision.FP32)
    # bottleneck / depthwise candidates of the 3x3 conv (SURVEY finding 12)
    for mut in ("b2", "dw", "crop"):
        net = chain.copy()
        s = net.layers[1].spec
        if mut == "b2":
            s.bottleneck_out = 2
        elif mut == "dw":
            net.layers[0].spec.co = s.ci = 48
            s.groups = 48
            s.co = 48
        else:
            if s.h % 2:
                continue
            s.spatial_div_h = s.spatial_div_w = 2
        nb.repair_network(net)
        _vs_oracle(ctx, oracle, net, 4, Precision.FP32)


IMAGENET = [(64, 56, 1), (64, 56, 64), (128, 28, 1), (128, 28, 32), (256, 14, 8),
            (256, 14, 256), (512, 7, 1), (512, 7, 2)]


@pytest.mark.parametrize("c,hw,g", IMAGENET, ids=lambda v: str(v))
def test_imagenet_shape_convs_vs_oracle(ctx, oracle, c, hw, g):
    spec = ConvSpec(c, c, hw, hw, 3, 3, 1, 1, groups=g)
    rng = np.random.default_rng(c + hw + g)
    x = np.maximum(rng.standard_normal((2, c, hw, hw)), 0)
    w = rng.standard_normal((c, c, 3, 3)) / math.sqrt(c * 9 / g)
    y = nb.reference_conv(spec, x, w, ctx=ctx)
    dy = rng.standard_normal((2, c, hw, hw))
    dx = nb.conv_dgrad(spec, dy, w, ctx=ctx)
    for i in range(2):
        scale = oracle.conv(spec, np.abs(x[i]), np.abs(w))
        assert np.all(np.abs(y[i] - oracle.conv(spec, x[i], w)) <= 1e-5 * scale + 1e-30)
        dscale = oracle.conv_dgrad(spec, np.abs(dy[i]), np.abs(w))
        assert np.all(np.abs(dx[i] - oracle.conv_dgrad(spec, dy[i], w)) <= 1e-5 * dscale + 1e-30)
