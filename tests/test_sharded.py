"""Example sharding (nb_fisher_sharded, SURVEY.md 8(e) secondary axis): one
network's fisher_potential (I/nnet.hpp:321-350) with the batch split over
sessions on distinct contexts.  Each shard divides dz by the whole batch's N
and plans its launches for it, and the per-example sums are reduced on the
root in the unsharded kernel's order, so the bar is bitwise equality with
one session holding the whole batch -- per_channel, per_layer, total, loss
and probabilities.  (One GPU here: the shards' contexts share device 0; the
gather is then a device-local copy instead of a peer copy.)"""
import numpy as np
import pytest

import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision


def test_shard_batch_slices_in_order():
    net = Network([Layer(ConvSpec(3, 4, 4, 4, 3, 3, 1, 1))], num_classes=3)
    x = np.arange(7 * 3 * 4 * 4, dtype=np.float64).reshape(7, 3, 4, 4)
    b = nb.Batch(x, np.arange(7, dtype=np.int32) % 3, 5)
    parts = nb.shard_batch(b, 3)
    assert [len(p) for p in parts] == [2, 2, 3]
    assert np.array_equal(np.concatenate([p.inputs for p in parts]), x)
    assert all(p.seed == 5 for p in parts)
    with pytest.raises(nb.ConfigError):
        nb.shard_batch(b, 8)
    del net


def _same(a, b):
    assert a.total == b.total, (a.total, b.total)
    assert a.loss == b.loss
    assert np.array_equal(a.per_layer, b.per_layer)
    for x, y in zip(a.per_channel, b.per_channel):
        assert np.array_equal(x, y)
    assert np.array_equal(a.probs, b.probs)


def _tc_chain():
    return Network([
        Layer(ConvSpec(3, 32, 16, 16, 3, 3, 1, 1)),
        Layer(ConvSpec(32, 64, 16, 16, 3, 3, 1, 1)),
        Layer(ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=2)),
        Layer(ConvSpec(64, 128, 16, 16, 3, 3, 2, 1)),
        Layer(ConvSpec(128, 128, 8, 8, 3, 3, 1, 1, bottleneck_out=2)),
        Layer(ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, spatial_div_h=2, spatial_div_w=2)),
        Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1, groups=64)),
        Layer(ConvSpec(64, 64, 4, 4, 3, 3, 1, 1)),
    ], num_classes=10, seed=42)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32, Precision.SIMT])
@pytest.mark.parametrize("count", [2, 3])
def test_sharded_chain_bitwise_equals_whole_batch(prec, count):
    net = _tc_chain()
    batch = nb.make_batch(net, 12, 1)
    whole = nb.Session(net, batch, ctx=nb.Context(0))
    ref = whole.fisher(net, prec)
    shards = [nb.Session(net, b, ctx=nb.Context(0)) for b in nb.shard_batch(batch, count)]
    _same(nb.fisher_sharded(shards, net, prec), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("count", [2, 3, 4])
def test_sharded_r34_bitwise_equals_whole_batch(count):
    """The R34 origin and two bench candidates at N=128: the shards' smaller
    per-launch tile counts would pick other split-K factors if they planned
    for their own N."""
    from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
    origin = resnet34_chain()
    cands = load_candidates(fixture_path("r34_candidates.json"), origin)
    batch = nb.make_batch(origin, 128, 1)
    whole = nb.Session(origin, batch, ctx=nb.Context(0))
    shards = [nb.Session(origin, b, ctx=nb.Context(0)) for b in nb.shard_batch(batch, count)]
    for net in [origin, cands[0], cands[len(cands) // 2]]:
        _same(nb.fisher_sharded(shards, net), whole.fisher(net))


@pytest.mark.gpu
def test_sharded_rejects_shared_context_and_mixed_batches():
    net = _tc_chain()
    batch = nb.make_batch(net, 4, 1)
    c = nb.Context(0)
    a, b = nb.shard_batch(batch, 2)
    s1, s2 = nb.Session(net, a, ctx=c), nb.Session(net, b, ctx=c)
    with pytest.raises(nb.ConfigError):
        nb.fisher_sharded([s1, s2], net)
    other = nb.make_batch(net, 2, 9)
    s3 = nb.Session(net, other, ctx=nb.Context(0))
    with pytest.raises(nb.ConfigError):
        nb.fisher_sharded([s1, s3], net)
