"""Parity at the benchmarked configuration (BASELINE configs[1]): the 33-conv
ResNet-34 CIFAR chain at batch N=128 -- the size bench.py times, where every
tensor-core launch has more output tiles than the 148 SMs and each CTA of
the persistent kernel runs several tiles (TMEM accumulator ping-pong,
cross-tile barrier phases, epilogue/mainloop overlap).

Goldens (oracle/gen_r34_golden.py): the fp64 restatement oracle/nb_oracle.cpp
(pinned to the unmodified reference to 1e-12 by tests/test_oracle.py) on the
origin and on bench-pool candidates covering depthwise, crop, bottleneck
(co_eff down to 1), grouped G<=8 (densified tensor-core plans) and G>8
(FFMA), masks on the stem, a stride-2 layer and the 512-channel stage.

Stated tolerances (paper_2102_06599_b200/api.py TOLERANCE_DEEP, DESIGN.md
3): totals / per-layer relative, per-channel against the largest layer's
value, loss 1e-6 relative, probabilities 1e-6 absolute.  At this depth true
fp32 (SIMT) itself sits ~1e-4 from fp64 (ReLU-mask flips of near-zero
activations re-route the gradient), which sets the floor of every mode.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Precision

N = 128
HAVE = os.path.exists(os.path.join(GOLDEN, "r34_n128.json"))
needs_golden = pytest.mark.skipif(not HAVE, reason="r34_n128 golden not generated")


def _nets():
    from paper_2102_06599_b200.workloads import fixture_path, load_candidates, resnet34_chain
    g = golden("r34_n128.json")
    origin = resnet34_chain()
    pool = load_candidates(fixture_path("r34_candidates.json"), origin)
    arrays = np.load(os.path.join(GOLDEN, "r34_n128.npz"))
    out = []
    for e in g["networks"]:
        net = origin if e["pool_index"] < 0 else pool[e["pool_index"]]
        out.append((e, net, arrays[e["name"] + "_per_channel"], arrays[e["name"] + "_probs"]))
    return out


@needs_golden
def test_r34_golden_is_consistent():
    """CPU: the golden's entries are the pool networks they name, and its
    totals are the sums of its per-layer values (no GPU needed)."""
    for e, net, pc, probs in _nets():
        assert len(e["per_layer"]) == len(net.layers) == 33
        assert pc.shape == (sum(l.spec.co_eff() for l in net.layers),)
        assert probs.shape == (N, 10)
        assert math.isclose(sum(e["per_layer"]), e["total"], rel_tol=1e-12)
    kinds = {e["kind"] for e, *_ in _nets()}
    for k in ("origin", "dw", "g8", "b2", "b64"):
        assert k in kinds, kinds


@pytest.fixture(scope="module")
def r34_session():
    from paper_2102_06599_b200.workloads import resnet34_chain
    origin = resnet34_chain()
    ctx = nb.Context(0)
    s = nb.Session(origin, nb.make_batch(origin, N, 1), ctx=ctx)
    yield s
    s.close()


@pytest.mark.gpu
@needs_golden
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.SIMT, Precision.TF32],
                         ids=["fp32_3xtf32", "simt", "tf32"])
def test_r34_n128_fisher_matches_oracle(r34_session, prec):
    tol = nb.TOLERANCE_DEEP[prec]
    reps = {}
    for e, net, pc, probs in _nets():
        rep = r34_session.fisher(net, prec)
        reps[e["name"]] = rep
        assert math.isclose(rep.total, e["total"], rel_tol=tol["total"]), \
            (e["name"], e["kind"], rep.total, e["total"])
        if prec == Precision.TF32:
            continue
        np.testing.assert_allclose(rep.per_layer, e["per_layer"], rtol=tol["layer"],
                                   err_msg=e["name"])
        np.testing.assert_allclose(np.concatenate(rep.per_channel), pc, rtol=0,
                                   atol=tol["layer"] * max(e["per_layer"]), err_msg=e["name"])
        assert math.isclose(rep.loss, e["loss"], rel_tol=1e-6), e["name"]
        np.testing.assert_allclose(rep.probs, probs, atol=1e-6, err_msg=e["name"])
    # fisher_accepts (I/nnet.hpp:356-359) against the origin: the decision of
    # every candidate outside the mode's near-threshold band is the oracle's
    o_gpu, o_ref = reps["origin"].total, golden("r34_n128.json")["networks"][0]["total"]
    for e, *_ in _nets()[1:]:
        margin = (e["total"] - o_ref) / o_ref
        if abs(margin) <= max(nb.RECHECK_BAND[prec], nb.TIE_BAND):
            continue  # decided by the search driver's SIMT recheck
        assert (reps[e["name"]].total >= o_gpu) == (e["total"] >= o_ref), (e["name"], margin)


@pytest.mark.gpu
@needs_golden
def test_r34_n128_simt_decisions_exact(r34_session):
    """The SIMT tier (the near-tie recheck's arithmetic) decides every golden
    candidate outside the documented tie band exactly as the fp64 oracle."""
    o_ref = golden("r34_n128.json")["networks"][0]["total"]
    o = r34_session.fisher(_nets()[0][1], Precision.SIMT).total
    for e, net, *_ in _nets()[1:]:
        if abs(e["total"] - o_ref) / o_ref <= nb.TIE_BAND:
            continue
        got = r34_session.fisher(net, Precision.SIMT).total
        assert (got >= o) == (e["total"] >= o_ref), e["name"]


# --------------------------------------------------------------------------
# multi-tile tensor-core launches, integer-exact (split-K stays off when the
# output tiles exceed 2 x the SMs, engine.cu choose_ksplit; the persistent
# grid is min(units, SMs), so every CTA runs 2-4 tiles here)

MULTI_TILE = [
    (ConvSpec(64, 64, 32, 32, 3, 3, 1, 1), 64),      # kw-fused N=192 plan: 512 tiles
    (ConvSpec(128, 128, 16, 16, 3, 3, 1, 1), 256),   # BN=128: 512 tiles
    (ConvSpec(256, 256, 8, 8, 3, 3, 1, 1), 512),     # BN=128 x 2 N tiles: 512 tiles
    (ConvSpec(512, 512, 4, 4, 3, 3, 1, 1), 1024),    # 4 N tiles: 128 M x 4 = 512 tiles
    (ConvSpec(64, 128, 32, 32, 3, 3, 2, 1), 256),    # stride 2 (dgrad: 4 phases)
    (ConvSpec(128, 128, 16, 16, 3, 3, 1, 1, groups=2), 256),  # grouped, per-group GEMMs
]


def _tiles(spec, n):
    bn = 192 if spec.co_eff() == 64 else min(128, spec.co_eff() // spec.groups)
    n_tiles = max(1, spec.co_eff() // bn) if spec.co_eff() != 64 else 1
    return (n * spec.out_h() * spec.out_w() + 127) // 128 * n_tiles


@pytest.mark.parametrize("spec,n", MULTI_TILE, ids=lambda v: str(v))
def test_multi_tile_cases_exceed_two_waves(spec, n):
    assert _tiles(spec, n) > 2 * 148


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32], ids=["fp32_3xtf32", "tf32"])
@pytest.mark.parametrize("spec,n", MULTI_TILE,
                         ids=[f"{s.ci}x{s.co}@{s.h}s{s.stride}g{s.groups}n{n}"
                              for s, n in MULTI_TILE])
def test_multi_tile_tc_conv_integer_exact(ctx, oracle, spec, n, prec):
    """fprop and dgrad of launches with 2-7 tiles per CTA reproduce
    reference_conv<int64> / the dgrad MAC loop bit for bit on every image."""
    rng = np.random.default_rng(spec.ci + n)
    x = rng.integers(-3, 4, size=(n, spec.ci, spec.h, spec.w)).astype(np.float64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.float64)
    dy = rng.integers(-3, 4, size=(n,) + spec.output_shape()).astype(np.float64)
    ctx.set_profiling(True)
    ctx.reset_stats()
    y = nb.reference_conv(spec, x, w, precision=prec, ctx=ctx)
    g = nb.conv_dgrad(spec, dy, w, precision=prec, ctx=ctx)
    names = set(ctx.kernel_stats())
    ctx.set_profiling(False)
    assert any("fprop_tc" in k for k in names) and any("dgrad_tc" in k for k in names), names
    wi = w.astype(np.int64)
    for i in range(0, n, max(1, n // 16)):  # 16 images spread over the batch
        assert np.array_equal(y[i], oracle.conv(spec, x[i].astype(np.int64), wi)), i
        assert np.array_equal(g[i], oracle.conv_dgrad(spec, dy[i], w)), i
    # the last image (the last tile of the last CTA)
    assert np.array_equal(y[-1], oracle.conv(spec, x[-1].astype(np.int64), wi))
    assert np.array_equal(g[-1], oracle.conv_dgrad(spec, dy[-1], w))
