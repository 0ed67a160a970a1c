"""The candidate scheduler (nb_evaluate, paper_2102_06599_b200/csrc/sched.cpp),
the B200 replacement of evaluate_all (I/search.hpp:315-334): dedupe, one
LPT-ordered queue pulled by every session as it frees up, re-queue of a
failed session's candidate, per-session statistics, and the search driver's
near-threshold band (integration/nestopt_b200.hpp near_threshold)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision
from paper_2102_06599_b200 import search as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NEEDS_LIB = pytest.mark.skipif(not os.path.exists(S.SO), reason="integration library not built")


@NEEDS_LIB
@pytest.mark.parametrize("prec", [Precision.FP32, Precision.TF32])
def test_near_threshold_band_covers_opposite_errors(prec):
    """a candidate and the origin can each be off by the mode's
    total tolerance in opposite directions; such a pair must be re-scored."""
    tol = nb.TOLERANCE_DEEP[prec]["total"]
    flips = 0
    for d in np.linspace(-3 * tol, 3 * tol, 121):
        cand_true, origin_true = 1.0 + d, 1.0
        for ec in (-tol, 0.0, tol):
            for eo in (-tol, 0.0, tol):
                cand, origin = cand_true * (1 + ec), origin_true * (1 + eo)
                if (cand >= origin) != (cand_true >= origin_true):
                    flips += 1  # a decision the mode alone would get wrong ...
                    assert S.near_threshold(cand, origin, prec), (d, ec, eo)  # ... is rechecked
    assert flips > 0
    assert not S.near_threshold(1.0 + 3 * tol, 1.0, prec)
    assert nb.RECHECK_BAND[prec] >= 2 * tol
    assert not S.near_threshold(1.0, 1.0, Precision.SIMT)


def _nets(k=12):
    out = []
    for i in range(k):
        g = [1, 2, 4][i % 3]
        out.append(Network([
            Layer(ConvSpec(3, 16, 16, 16, 3, 3, 1, 1)),
            Layer(ConvSpec(16, 32, 16, 16, 3, 3, 1 + i % 2, 1, groups=g)),
            Layer(ConvSpec(32, 32, 16 // (1 + i % 2), 16 // (1 + i % 2), 3, 3, 1, 1,
                           bottleneck_out=1 + (i // 3) % 2)),
        ], num_classes=10, seed=5))
    out.append(out[0].copy())  # a duplicate: answered by dedupe
    return out


@pytest.mark.gpu
def test_sessions_must_not_share_a_context():
    net = _nets()[0]
    b = nb.make_batch(net, 4, 1)
    c = nb.Context(0)
    s1, s2 = nb.Session(net, b, ctx=c), nb.Session(net, b, ctx=c)
    with pytest.raises(nb.ConfigError, match="share a context"):
        nb.evaluate([s1, s2], [net], Precision.FP32)


@pytest.mark.gpu
def test_sessions_must_hold_the_same_batch():
    net = _nets()[0]
    s1 = nb.Session(net, nb.make_batch(net, 4, 1), ctx=nb.Context(0))
    s2 = nb.Session(net, nb.make_batch(net, 5, 1), ctx=nb.Context(0))
    with pytest.raises(nb.ConfigError, match="different batches"):
        nb.evaluate([s1, s2], [net], Precision.FP32)
    s3 = nb.Session(net, nb.make_batch(net, 4, 2), ctx=nb.Context(0))
    with pytest.raises(nb.ConfigError, match="different batches"):
        nb.evaluate([s1, s3], [net], Precision.FP32)


@pytest.mark.gpu
def test_more_than_sixteen_sessions_and_per_session_stats():
    nets = _nets()
    b = nb.make_batch(nets[0], 4, 1)
    one = nb.Session(nets[0], b, ctx=nb.Context(0))
    want, _ = nb.evaluate([one], nets, Precision.FP32)
    many = [nb.Session(nets[0], b, ctx=nb.Context(0)) for _ in range(20)]
    got, st = nb.evaluate(many, nets, Precision.FP32)
    for a, w in zip(got, want):
        assert a.total == w.total and np.array_equal(a.per_layer, w.per_layer)
    distinct = len({str([(l.spec.to_json(), l.relu) for l in n.layers]) for n in nets})
    assert st.evaluated == distinct and st.deduplicated == len(nets) - distinct
    assert sum(st.evaluations) == st.evaluated
    assert len(st.busy_ms) == 20 and sum(st.busy_ms) > 0
    for k in range(20):
        assert (st.busy_ms[k] > 0) == (st.evaluations[k] > 0)
    assert st.requeued == 0 and st.failed_sessions == 0


FAULT = r"""
import sys
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from test_sched import _nets
nets = _nets()
b = nb.make_batch(nets[0], 4, 1)
ss = [nb.Session(nets[0], b, ctx=nb.Context(0)) for _ in range(3)]
got, st = nb.evaluate(ss, nets, Precision.FP32)
ref, _ = nb.evaluate(ss[:1], nets, Precision.FP32)
assert st.requeued == 1 and st.failed_sessions == 1, (st.requeued, st.failed_sessions)
assert st.evaluations[1] == 0, st.evaluations
for a, w in zip(got, ref):
    assert a.total == w.total and np.array_equal(a.per_channel[-1], w.per_channel[-1])
only = [nb.Session(nets[0], b, ctx=nb.Context(0))]
import os
os.environ["NB_SCHED_FAULT"] = "0"
try:
    nb.evaluate(only, nets, Precision.FP32)
    raise SystemExit("a call with no session left must fail")
except nb.CudaError as e:
    assert "injected" in str(e)
print("ok")
"""


@pytest.mark.gpu
def test_failed_session_candidates_are_requeued():
    """NB_SCHED_FAULT=1: session 1's first evaluation fails as a device
    error; it is retired, its candidate re-runs elsewhere and the report is
    bitwise the single-session one.  With no session left the call fails."""
    env = dict(os.environ, NB_SCHED_FAULT="1")
    r = subprocess.run([sys.executable, "-c", FAULT % (ROOT, os.path.join(ROOT, "tests"))],
                       env=env, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.stdout[-2000:],
                                                                    r.stderr[-2000:])


@pytest.mark.gpu
@pytest.mark.skipif(nb.device_count() < 2, reason="needs two GPUs")
def test_distinct_devices_match_single_device():
    """nb_evaluate and nb_fisher_sharded across two real devices give the
    single-device reports bitwise (skipped on a one-GPU box)."""
    nets = _nets()
    b = nb.make_batch(nets[0], 4, 1)
    one = [nb.Session(nets[0], b, ctx=nb.Context(0))]
    two = [nb.Session(nets[0], b, ctx=nb.Context(d)) for d in (0, 1)]
    want, _ = nb.evaluate(one, nets, Precision.FP32)
    got, st = nb.evaluate(two, nets, Precision.FP32)
    for a, w in zip(got, want):
        assert a.total == w.total
    assert all(e > 0 for e in st.evaluations)
    shards = [nb.Session(nets[0], x, ctx=nb.Context(d))
              for d, x in zip((0, 1), nb.shard_batch(b, 2))]
    r = nb.fisher_sharded(shards, nets[1])
    assert r.total == one[0].fisher(nets[1]).total
