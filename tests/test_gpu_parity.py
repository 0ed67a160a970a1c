"""GPU parity tests: the sm_100a kernels (through the C ABI) against the
reference's golden fixtures and the fp64 oracle restatement.

Stated tolerances, per arithmetic mode:

  NB_PREC_SIMT  fp32 FFMA everywhere (round-to-nearest fp32 accumulation):
    conv outputs |gpu - ref| <= 2e-6 * sum|w||x|; Fisher totals 1e-5 relative,
    per layer 1e-4, per channel 1e-4 of the largest layer; loss 1e-6.
  NB_PREC_FP32  3xTF32 on the tensor cores (hi/lo split products, fp32
    accumulation inside tcgen05.mma, measured rms 4e-7..9e-7 of sum|w||x| for
    K = 576..4608 vs 3e-8 for SIMT -- scripts/experiments/precision_probe.py):
    conv outputs 1e-5 * sum|w||x|; Fisher totals 5e-4 (measured 1.3e-5 on
    10 layers, 1.0e-4 on the 33-layer R34 chain), per layer 5e-3, per channel
    5e-3 of the largest layer; loss 1e-6.
  NB_PREC_TF32  1xTF32 throughput mode: totals 5e-2, per layer 2e-1 (measured
    7e-4..7.3e-3 on <= 10 layers, 3.1e-2 on the R34 chain).

Small-integer conv inputs are bit-exact in every mode (products exact in
tf32, every partial sum < 2^24).
"""
import math

import numpy as np
import pytest

from conftest import golden
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ChannelSplit, ConvSpec, Layer, Network, Precision

pytestmark = pytest.mark.gpu

GOLD_CONV = golden("conv_cases.json")["cases"]
GOLD_FISHER = golden("fisher_nets.json")["nets"]
EXACT_PRECS = [Precision.FP32, Precision.SIMT]
# (total, per_layer, per_channel-of-max-layer, conv-vs-sum|w||x|)
TOL = {p: (t["total"], t["layer"], t["layer"], t["conv"]) for p, t in nb.TOLERANCE.items()}


def _inputs(seed, spec):
    rng = np.random.default_rng(seed)
    x = rng.integers(-3, 4, size=(spec.ci, spec.h, spec.w)).astype(np.int64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.int64)
    return x, w


@pytest.mark.parametrize("prec", EXACT_PRECS)
@pytest.mark.parametrize("case", GOLD_CONV, ids=lambda c: str(c["seed"]))
def test_conv_matches_reference_conv(ctx, case, prec):
    spec = ConvSpec.from_json(case["spec"])
    x, w = _inputs(case["seed"], spec)
    y = nb.reference_conv(spec, x.astype(np.float64), w.astype(np.float64), precision=prec,
                          ctx=ctx)
    assert np.array_equal(y.ravel(), np.asarray(case["out_int"], np.float64))
    xf, wf = x * 0.37, w * 1.3
    yf = nb.reference_conv(spec, xf, wf, precision=prec, ctx=ctx)
    scale = nb.reference_conv(spec, np.abs(xf), np.abs(wf), precision=Precision.SIMT, ctx=ctx)
    assert np.all(np.abs(yf.ravel() - case["out_f64"]) <= TOL[prec][3] * scale.ravel() + 1e-30)


def test_conv_kats_and_batching(ctx):
    """T/test_interp.cpp KATs, batched with distinct images per example."""
    s = ConvSpec(4, 4, 1, 1, groups=2)
    x = np.stack([np.array([1, 10, 100, 1000.]).reshape(4, 1, 1) * k for k in (1, 2, 3)])
    y = nb.reference_conv(s, x, np.ones((4, 4, 1, 1)), ctx=ctx)
    assert y[:, :, 0, 0].tolist() == [[11, 11, 1100, 1100], [22, 22, 2200, 2200],
                                      [33, 33, 3300, 3300]]
    s = ConvSpec(1, 1, 2, 2, 3, 3, 1, 1)
    y = nb.reference_conv(s, np.arange(1, 5.).reshape(1, 2, 2), np.ones((1, 1, 3, 3)), ctx=ctx)
    assert y.ravel().tolist() == [10, 10, 10, 10]


@pytest.mark.parametrize("prec", EXACT_PRECS)
def test_dgrad_matches_oracle(ctx, oracle, prec):
    rng = np.random.default_rng(3)
    for case in GOLD_CONV:
        spec = ConvSpec.from_json(case["spec"])
        dy = rng.integers(-3, 4, size=spec.output_shape()).astype(np.float64)
        w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(
            np.float64)
        got = nb.conv_dgrad(spec, dy, w, precision=prec, ctx=ctx)
        want = oracle.conv_dgrad(spec, dy, w)
        assert np.array_equal(got, want), case["spec"]


@pytest.mark.parametrize("prec", EXACT_PRECS)
@pytest.mark.parametrize("case", GOLD_FISHER, ids=lambda c: c["name"])
def test_fisher_matches_reference_golden(ctx, case, prec):
    net = Network.from_json(case["network"])
    batch = nb.make_batch(net, case["n"], case["batch_seed"])
    rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
    t_tot, t_layer, t_chan, _ = TOL[prec]
    assert math.isclose(rep.total, case["total"], rel_tol=t_tot), (rep.total, case["total"])
    np.testing.assert_allclose(rep.per_layer, case["per_layer"], rtol=t_layer)
    scale = max(case["per_layer"])
    np.testing.assert_allclose(np.concatenate(rep.per_channel), case["per_channel"], rtol=0,
                               atol=t_chan * scale)
    assert math.isclose(rep.loss, case["loss"], rel_tol=1e-6)
    np.testing.assert_allclose(rep.probs.ravel(), case["probs"], atol=1e-6)
    assert rep.seed == case["batch_seed"]


def test_tf32_mode_within_stated_tolerance(ctx):
    for case in GOLD_FISHER:
        net = Network.from_json(case["network"])
        batch = nb.make_batch(net, case["n"], case["batch_seed"])
        rep = nb.fisher_potential(net, batch, precision=Precision.TF32, ctx=ctx)
        assert math.isclose(rep.total, case["total"], rel_tol=TOL[Precision.TF32][0]), case["name"]


def _feature_net(seed=11):
    return Network([
        Layer(ConvSpec(3, 8, 9, 9, 3, 3, 2, 1)),
        Layer(ConvSpec(8, 8, 5, 5, 3, 3, 1, 1, groups=2, spatial_div_h=5), relu=False),
        Layer(ConvSpec(8, 6, 1, 5, 1, 3, 1, 0,
                       channel_splits=[ChannelSplit(0, 2, 2), ChannelSplit(2, 6, 1)])),
        Layer(ConvSpec(6, 6, 1, 3, 3, 3, 1, 1, groups=6)),
    ], num_classes=5, seed=seed)


@pytest.mark.parametrize("prec", EXACT_PRECS)
def test_activation_gradients_match_oracle(ctx, oracle, prec):
    net = _feature_net()
    batch = nb.make_batch(net, 3, 4)
    acts, grads = nb.activation_gradients(net, batch, precision=prec, ctx=ctx)
    o = oracle.fisher(net, 3, batch=batch, grads=True)
    off = 0
    f = 10.0 if prec == Precision.FP32 else 1.0
    for a, g in zip(acts, grads):
        k = a.size
        ra, rg = o["acts"][off:off + k], o["grads"][off:off + k]
        np.testing.assert_allclose(a.ravel(), ra, rtol=1e-5 * f, atol=1e-6 * f * np.abs(ra).max())
        np.testing.assert_allclose(g.ravel(), rg, rtol=1e-4 * f, atol=1e-5 * f * np.abs(rg).max())
        off += k


def test_gradients_agree_with_finite_differences(ctx, oracle):
    """acceptance criterion 5 (T/acceptance.cpp:333-369): the GPU's analytic
    activation gradients against central differences of the fp64 loss."""
    net = Network([Layer(ConvSpec(2, 4, 5, 5, 3, 3, 1, 1)), Layer(ConvSpec(4, 4, 5, 5, 3, 3, 1, 1)),
                   Layer(ConvSpec(4, 3, 5, 5))], num_classes=4, seed=42)
    batch = nb.make_batch(net, 3, 11)
    acts, grads = nb.activation_gradients(net, batch, ctx=ctx)
    net.init_weights()
    eps = 1e-5
    probes = 0
    for l in range(len(net.layers)):
        n = l % 3
        sub = Network(net.layers[l + 1:], num_classes=4, seed=42) if l + 1 < len(net.layers) else None
        for p in range(6):
            i = (p * 17 + l * 5) % acts[l][n].size
            loss = []
            for sgn in (1, -1):
                a = acts[l][n].ravel().copy()
                a[i] += sgn * eps
                a = a.reshape(acts[l][n].shape)
                if sub is None:
                    z = net.head @ a.reshape(a.shape[0], -1).mean(axis=1)
                else:
                    sub.weights = net.weights[l + 1:]
                    sub.head = net.head
                    from paper_2102_06599_b200.api import Batch
                    fwd = oracle.fisher(sub, 1, batch=Batch(a[None], batch.labels[n:n + 1], 0))
                    z = None
                    loss.append(fwd["loss"])
                    continue
                pz = np.exp(z - z.max())
                pz /= pz.sum()
                loss.append(-math.log(max(pz[batch.labels[n]], 1e-300)))
            fd = (loss[0] - loss[1]) / (2 * eps) / 3.0  # other examples' terms cancel
            g = grads[l][n].ravel()[i]
            assert abs(g - fd) <= 1e-4 * max(abs(fd), 1e-3), (l, i, g, fd)
            probes += 1
    assert probes == 18


def test_zero_weights_and_relu_killed(ctx):
    """T/test_nnet.cpp:35-44, :145-157, :180-186."""
    net = Network([Layer(ConvSpec(2, 4, 5, 5, 3, 3, 1, 1)), Layer(ConvSpec(4, 4, 5, 5, 3, 3, 1, 1)),
                   Layer(ConvSpec(4, 3, 5, 5))], num_classes=4, seed=42)
    net.init_weights()
    zero = net.copy()
    zero.weights = [np.zeros_like(w) for w in net.weights]
    zero.head = np.zeros_like(net.head)
    batch = nb.make_batch(net, 8, 1)
    rep = nb.fisher_potential(zero, batch, ctx=ctx)
    assert math.isclose(rep.loss, math.log(4.0), rel_tol=1e-12)
    assert rep.total == 0.0
    killed = net.copy()
    killed.weights[1] = np.full_like(net.weights[1], -10.0)
    acts, grads = nb.activation_gradients(killed, nb.make_batch(net, 2, 3), ctx=ctx)
    assert np.all(acts[1] == 0.0)
    assert np.all(grads[0] == 0.0)


def test_determinism_and_exact_ties(ctx):
    """Identical networks score bit-identically, so fisher_accepts(origin,
    origin) holds exactly (T/test_nnet.cpp:188-200)."""
    case = GOLD_FISHER[0]
    net = Network.from_json(case["network"])
    batch = nb.make_batch(net, 8, 1)
    a = nb.fisher_potential(net, batch, ctx=ctx)
    b = nb.fisher_potential(net, batch, ctx=ctx)
    assert a.total == b.total
    assert all(np.array_equal(x, y) for x, y in zip(a.per_channel, b.per_channel))
    assert nb.fisher_accepts(a, b) and nb.legality_fisher(net, net, batch, ctx=ctx)


def test_session_and_scheduler_match_single_calls(ctx):
    """evaluate (the evaluate_all replacement) == per-network calls, with
    duplicates answered by dedupe (T/test_search.cpp:83-94 analogue)."""
    base = Network.from_json(GOLD_FISHER[1]["network"])
    batch = nb.make_batch(base, 4, 1)
    variants = []
    for b, g in [(1, 1), (2, 1), (1, 2), (1, 1), (2, 1)]:
        n = base.copy()
        n.layers[1].spec.bottleneck_out = b
        n.layers[2].spec.groups = g
        nb.repair_network(n)
        variants.append(n)
    sess = nb.Session(base, batch, ctx=ctx)
    reps, stats = nb.evaluate([sess], variants)
    assert stats.evaluated == 3 and stats.deduplicated == 2
    for n, r in zip(variants, reps):
        single = nb.fisher_potential(n, batch, ctx=ctx)
        assert single.total == r.total
        assert sess.fisher(n).total == r.total


def test_larger_chain_matches_oracle(ctx, oracle):
    """A 10-layer 16->32 channel chain at N=4 (the mid10 shape, larger batch)."""
    net = Network.from_json([c for c in GOLD_FISHER if c["name"] == "mid10"][0]["network"])
    batch = nb.make_batch(net, 4, 2)
    for prec in (Precision.SIMT, Precision.FP32):
        rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
        o = oracle.fisher(net, 4, batch=batch)
        assert math.isclose(rep.total, o["total"], rel_tol=TOL[prec][0])
        np.testing.assert_allclose(rep.per_layer, o["per_layer"], rtol=TOL[prec][1])


# ---------------------------------------------------------------------------
# tensor-core (tcgen05) shaped cases: 32-channel K chunks, 16-aligned N

TC_SPECS = [
    ConvSpec(32, 32, 8, 8, 3, 3, 1, 1),
    ConvSpec(64, 64, 16, 16, 3, 3, 1, 1),
    ConvSpec(64, 128, 16, 16, 3, 3, 2, 1),                     # stride 2 (TMA element strides)
    ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, groups=2),              # grouped, slice_ci = 32
    ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, bottleneck_out=2),    # Co_eff = 32
    ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, spatial_div_h=4, spatial_div_w=2),  # crop
    ConvSpec(64, 64, 4, 4, 3, 3, 1, 1),                        # 8 images per M tile
    ConvSpec(32, 64, 7, 7, 3, 3, 1, 1),                        # 49-pixel images (partial tiles)
    ConvSpec(64, 64, 8, 8, 1, 1, 1, 0),                        # 1x1
    ConvSpec(64, 96, 8, 8, 3, 3, 1, 1,
             channel_splits=[ChannelSplit(0, 32, 1), ChannelSplit(32, 96, 2)]),
    ConvSpec(128, 128, 2, 2, 3, 3, 1, 1),                      # 32 images per M tile
    ConvSpec(64, 64, 9, 9, 3, 3, 2, 1),                        # stride 2, odd input
    ConvSpec(32, 64, 16, 16, 3, 3, 2, 1, spatial_div_h=2),     # stride 2 + crop
    ConvSpec(64, 64, 8, 8, 1, 1, 2, 0),                        # 1x1 s2: empty dgrad phases
    ConvSpec(64, 64, 32, 32, 3, 3, 1, 1),                      # kw-fused fprop + dgrad (N=192)
    ConvSpec(128, 64, 32, 32, 3, 3, 1, 1),                     # kw-fused fprop, K = 3 x 128
    ConvSpec(64, 64, 12, 32, 3, 3, 1, 1, spatial_div_h=2),     # kw-fused, short rows + crop
    ConvSpec(64, 64, 8, 8, 3, 3, 1, 1),                        # kw-fused, 8-pixel rows (4 per warp)
    ConvSpec(128, 64, 6, 16, 3, 3, 1, 1),                      # kw-fused, 16-pixel rows, partial tiles
]
# padded plans: K per tap rounded up to 32-channel chunks (TMA zero fill),
# the last N tile narrower than BN (DenseNet's 48-channel growth)
PAD_SPECS = [
    ConvSpec(144, 192, 8, 8, 1, 1, 1, 0),                      # K 144 -> 160
    ConvSpec(192, 48, 8, 8, 3, 3, 1, 1),                       # N 48 of 64; dgrad K 48 -> 64
    ConvSpec(48, 80, 16, 16, 3, 3, 2, 1),                      # both padded, stride 2
    ConvSpec(20, 16, 7, 7, 3, 3, 1, 1),                        # K 20 -> 32, N 16 of 32
    ConvSpec(64, 48, 8, 8, 3, 3, 1, 1,
             channel_splits=[ChannelSplit(0, 16, 1), ChannelSplit(16, 48, 1)]),  # padded range
    # 64-wide outputs over power-of-two rows (kw-fused shape) with a padded K:
    # fprop K 16 / 48 -> 32 / 64, dgrad K (= Co) 16 -> 32 (round 2: R34 bottleneck
    # candidates, b4 into a 64-channel stage; the kw-fused plan must not take these)
    ConvSpec(16, 64, 32, 32, 3, 3, 1, 1),
    ConvSpec(16, 64, 16, 8, 3, 3, 1, 1),
    ConvSpec(48, 64, 8, 8, 3, 3, 1, 1),
    ConvSpec(64, 16, 32, 32, 3, 3, 1, 1),
]
# densified grouped ranges: a few groups of slices off the 32-channel chunk
# run as one GEMM over block-diagonal weights
DENSE_SPECS = [
    ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, groups=4),              # slices of 16
    ConvSpec(64, 64, 16, 16, 3, 3, 1, 1, groups=8),            # slices of 8
    ConvSpec(32, 48, 8, 8, 3, 3, 2, 1, groups=2),              # 16 -> 24 per group, stride 2
    ConvSpec(128, 128, 4, 4, 3, 3, 1, 1, groups=8, bottleneck_out=2),  # 16 -> 8 per group
    ConvSpec(64, 96, 8, 8, 3, 3, 1, 1,
             channel_splits=[ChannelSplit(0, 32, 1), ChannelSplit(32, 96, 4)]),  # densified range
]
TC_SPECS += PAD_SPECS + DENSE_SPECS


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32])
@pytest.mark.parametrize("spec", TC_SPECS, ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}g{s.groups}")
def test_tc_conv_integer_exact(ctx, oracle, spec, prec):
    """Small integers are exact in tf32 and their sums exact in fp32, so the
    tensor-core path must reproduce reference_conv<int64> bit for bit."""
    rng = np.random.default_rng(spec.ci * 7 + spec.co)
    n = 3
    x = rng.integers(-3, 4, size=(n, spec.ci, spec.h, spec.w)).astype(np.float64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.float64)
    y = nb.reference_conv(spec, x, w, precision=prec, ctx=ctx)
    for i in range(n):
        want = oracle.conv(spec, x[i].astype(np.int64), w.astype(np.int64))
        assert np.array_equal(y[i], want.astype(np.float64)), i


@pytest.mark.parametrize("spec", PAD_SPECS + DENSE_SPECS,
                         ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}g{s.groups}")
def test_padded_specs_run_on_tensor_cores(spec):
    """The padded and densified shapes are lowered to the tcgen05 kernel, not
    the FFMA fallback (fprop; dgrad too where Ci is a multiple of 16)."""
    c = nb.Context(0)
    net = Network([Layer(ConvSpec(spec.ci, spec.ci, spec.h, spec.w, 1, 1, 1, 0)), Layer(spec)],
                  num_classes=10, seed=3)
    s = nb.Session(net, nb.make_batch(net, 4, 1), ctx=c)
    c.set_profiling(True)
    s.fisher(net)
    names = set(c.kernel_stats())
    split = nb.fp32_split()  # "3xbf16" (default) or "3xtf32"
    assert f"conv_fprop_tc_{split}" in names, names
    if spec.ci % 16 == 0 and not spec.channel_splits:
        assert f"conv_dgrad_tc_{split}_fisher" in names, names
        assert "conv_dgrad_direct_fisher" not in names, names


@pytest.mark.parametrize("spec", TC_SPECS, ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}g{s.groups}")
def test_tc_conv_fp32_accuracy(ctx, oracle, spec):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, spec.ci, spec.h, spec.w))
    w = rng.standard_normal((spec.co_eff(), spec.ci, spec.kh, spec.kw)) / np.sqrt(spec.ci * 9)
    y3 = nb.reference_conv(spec, x, w, precision=Precision.FP32, ctx=ctx)
    y1 = nb.reference_conv(spec, x, w, precision=Precision.TF32, ctx=ctx)
    scale = np.stack([oracle.conv(spec, np.abs(x[i]), np.abs(w)) for i in range(2)])
    want = np.stack([oracle.conv(spec, x[i], w) for i in range(2)])
    assert np.all(np.abs(y3 - want) <= TOL[Precision.FP32][3] * scale + 1e-30)  # 3xTF32
    assert np.all(np.abs(y1 - want) <= TOL[Precision.TF32][3] * scale + 1e-30)  # 1xTF32


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32])
@pytest.mark.parametrize("spec", [s for s in TC_SPECS if not s.channel_splits],
                         ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}g{s.groups}")
def test_tc_dgrad_integer_exact(ctx, oracle, spec, prec):
    rng = np.random.default_rng(11)
    dy = rng.integers(-3, 4, size=(2,) + spec.output_shape()).astype(np.float64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.float64)
    got = nb.conv_dgrad(spec, dy, w, precision=prec, ctx=ctx)
    for i in range(2):
        assert np.array_equal(got[i], oracle.conv_dgrad(spec, dy[i], w)), i


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


@pytest.mark.parametrize("prec", [Precision.SIMT, Precision.FP32, Precision.TF32])
def test_tc_chain_fisher_matches_oracle(ctx, oracle, prec):
    net = _tc_chain()
    batch = nb.make_batch(net, 4, 1)
    rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
    o = oracle.fisher(net, 4, batch=batch)
    t_tot, t_layer, _, _ = TOL[prec]
    assert math.isclose(rep.total, o["total"], rel_tol=t_tot), (rep.total, o["total"])
    np.testing.assert_allclose(rep.per_layer, o["per_layer"], rtol=t_layer)
    assert math.isclose(rep.loss, o["loss"], rel_tol=t_tot)


# chains that lower to every tensor-core plan family inside the Fisher
# pipeline (kw-fused, padded K in fprop and dgrad, bottleneck into a kw-fused
# width, densified groups, col stem), scored against the oracle layer by layer
PLAN_CHAINS = {
    "padded_into_kwf": [ConvSpec(3, 16, 32, 32, 3, 3, 1, 1), ConvSpec(16, 64, 32, 32, 3, 3, 1, 1),
                        ConvSpec(64, 64, 32, 32, 3, 3, 1, 1)],
    "b4_g2_into_64": [ConvSpec(3, 64, 32, 32, 3, 3, 1, 1),
                      ConvSpec(64, 64, 32, 32, 3, 3, 1, 1, groups=2, bottleneck_out=4),
                      ConvSpec(16, 64, 32, 32, 3, 3, 1, 1), ConvSpec(64, 64, 32, 32, 3, 3, 1, 1)],
    "crop_rows_8": [ConvSpec(3, 64, 16, 16, 3, 3, 1, 1),
                    ConvSpec(64, 48, 16, 16, 3, 3, 1, 1, spatial_div_w=2),
                    ConvSpec(48, 64, 16, 8, 3, 3, 1, 1), ConvSpec(64, 64, 16, 8, 3, 3, 1, 1)],
    "dense_g4_s2": [ConvSpec(3, 32, 16, 16, 3, 3, 1, 1),
                    ConvSpec(32, 64, 16, 16, 3, 3, 2, 1, groups=4),
                    ConvSpec(64, 64, 8, 8, 3, 3, 1, 1, groups=8)],
}


@pytest.mark.parametrize("prec", [Precision.SIMT, Precision.FP32, Precision.TF32])
@pytest.mark.parametrize("name", sorted(PLAN_CHAINS))
def test_plan_family_chains_match_oracle(ctx, oracle, name, prec):
    net = Network([Layer(s) for s in PLAN_CHAINS[name]], num_classes=10, seed=42)
    for n in (4, 33):
        batch = nb.make_batch(net, n, 1)
        rep = nb.fisher_potential(net, batch, precision=prec, ctx=ctx)
        o = oracle.fisher(net, n, batch=batch)
        t_tot, t_layer, _, _ = TOL[prec]
        assert math.isclose(rep.total, o["total"], rel_tol=t_tot), (n, rep.total, o["total"])
        np.testing.assert_allclose(rep.per_layer, o["per_layer"], rtol=t_layer, err_msg=str(n))


def test_tc_chain_gradients_match_oracle(ctx, oracle):
    net = _tc_chain()
    batch = nb.make_batch(net, 2, 3)
    acts, grads = nb.activation_gradients(net, batch, precision=Precision.FP32, ctx=ctx)
    o = oracle.fisher(net, 2, batch=batch, grads=True)
    off = 0
    for a, g in zip(acts, grads):
        k = a.size
        ra, rg = o["acts"][off:off + k], o["grads"][off:off + k]
        np.testing.assert_allclose(a.ravel(), ra, rtol=0, atol=1e-4 * np.abs(ra).max())
        np.testing.assert_allclose(g.ravel(), rg, rtol=0, atol=1e-3 * np.abs(rg).max())
        off += k


STEM_SPECS = [
    ConvSpec(3, 64, 32, 32, 3, 3, 1, 1),     # the R34 stem (k_fprop_blocked<64>)
    ConvSpec(4, 64, 9, 9, 3, 3, 2, 1),       # stride 2, partial last block
    ConvSpec(14, 64, 5, 5, 3, 3, 1, 1),      # K = 126 <= 128
    ConvSpec(3, 64, 7, 7, 3, 3, 1, 1, spatial_div_h=7),  # crop
    ConvSpec(64, 128, 16, 16, 3, 3, 2, 1, groups=8),     # grouped s2, slice_ci 8 (float4 path)
    ConvSpec(96, 96, 6, 6, 3, 3, 2, 1, groups=12),       # grouped s2, slice 8
    ConvSpec(36, 72, 5, 5, 3, 3, 2, 1, groups=3),        # slice_ci 12 (float4, K = 108)
]


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.SIMT])
@pytest.mark.parametrize("spec", STEM_SPECS, ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}")
def test_stem_fprop_integer_exact(ctx, oracle, spec, prec):
    """The direct fprop of stem-shaped layers (k_fprop_blocked, outputs staged
    through shared memory) against reference_conv<int64>, small integers so
    fp32 sums are exact."""
    rng = np.random.default_rng(spec.ci * 3 + spec.h)
    n = 3
    x = rng.integers(-3, 4, size=(n, spec.ci, spec.h, spec.w)).astype(np.float64)
    w = rng.integers(-3, 4, size=(spec.co_eff(), spec.ci, spec.kh, spec.kw)).astype(np.float64)
    y = nb.reference_conv(spec, x, w, precision=prec, ctx=ctx)
    for i in range(n):
        want = oracle.conv(spec, x[i].astype(np.int64), w.astype(np.int64))
        assert np.array_equal(y[i], want.astype(np.float64)), i


# the session path lowers narrow stems (Ci*KH*KW <= 32) to a 1x1 tensor-core
# GEMM over the resident batch's im2col copy
COL_STEMS = [
    ConvSpec(3, 64, 32, 32, 3, 3, 1, 1),                    # the R34 stem
    ConvSpec(3, 32, 17, 17, 3, 3, 2, 1),                    # stride 2, odd size
    ConvSpec(3, 16, 9, 9, 3, 3, 1, 1, spatial_div_h=3),     # crop, N 16 of 32
    ConvSpec(2, 48, 8, 8, 3, 3, 1, 1),                      # K 18, N 48 of 64
    ConvSpec(3, 8, 6, 6, 1, 1, 1, 0),                       # 1x1 stem, N 8 of 32
    ConvSpec(3, 16, 8, 8, 3, 3, 1, 1, bottleneck_out=4),    # co_eff 4: N 4 of 32
]


@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32])
@pytest.mark.parametrize("spec", COL_STEMS, ids=lambda s: f"{s.ci}x{s.co}x{s.h}s{s.stride}")
def test_col_stem_integer_exact(oracle, spec, prec):
    c = nb.Context(0)
    net = Network([Layer(spec, relu=False)], num_classes=4, seed=5)
    net.init_weights()
    rng = np.random.default_rng(spec.co + spec.h)
    w = rng.integers(-3, 4, size=net.weights[0].shape).astype(np.float64)
    net.weights[0] = w
    n = 3
    x = rng.integers(-3, 4, size=(n, spec.ci, spec.h, spec.w)).astype(np.float64)
    batch = nb.Batch(x, np.arange(n, dtype=np.int32) % 4, 1)
    c.set_profiling(True)
    acts, _ = nb.activation_gradients(net, batch, precision=prec, ctx=c)
    names = set(c.kernel_stats())
    assert "conv_fprop_direct" not in names, names
    y = acts[0].reshape((n,) + spec.output_shape())
    for i in range(n):
        want = oracle.conv(spec, x[i].astype(np.int64), w.astype(np.int64))
        assert np.array_equal(y[i], want.astype(np.float64)), i
