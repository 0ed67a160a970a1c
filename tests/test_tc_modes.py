"""The tcgen05 kernel's experimental launch modes (environment switches read
once per process, so each runs in a subprocess with a deadline): CTA pairs,
multicast-B clusters, converter stage alternation, no split-K, no PDL, the
kw-fused plans switched off, the 3xTF32 / 3xBF16 splits, the row-per-tap A
operand (halo tiles off), the 256-wide single-accumulator tile and the kw-fused dgrad with one
epilogue column group (debug bit 2^21).  Each must reproduce reference_conv<int64>
bit for bit on tensor-core-shaped layers (including a kw-fused shape) and
finish -- a hang here is a barrier-count bug."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, sys
sys.path.insert(0, %r)
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Precision
from oracle.oracle import Restatement
O = Restatement()
ctx = nb.Context(0)
specs = [ConvSpec(64, 128, 8, 8, 3, 3, 1, 1), ConvSpec(128, 128, 4, 4, 3, 3, 1, 1),
         ConvSpec(64, 64, 32, 32, 3, 3, 1, 1), ConvSpec(64, 128, 9, 9, 3, 3, 2, 1),
         ConvSpec(256, 256, 8, 8, 3, 3, 1, 1)]
rng = np.random.default_rng(3)
for prec in (Precision.FP32, Precision.TF32):
    for s in specs:
        x = rng.integers(-3, 4, size=(2, s.ci, s.h, s.w)).astype(np.float64)
        w = rng.integers(-3, 4, size=(s.co_eff(), s.ci, s.kh, s.kw)).astype(np.float64)
        y = nb.reference_conv(s, x, w, precision=prec, ctx=ctx)
        dy = rng.integers(-3, 4, size=(2,) + s.output_shape()).astype(np.float64)
        g = nb.conv_dgrad(s, dy, w, precision=prec, ctx=ctx)
        for i in range(2):
            assert np.array_equal(y[i], O.conv(s, x[i].astype(np.int64), w.astype(np.int64))), s
            assert np.array_equal(g[i], O.conv_dgrad(s, dy[i], w)), s
print("ok")
""" % ROOT

# comma-separated environment assignments; the CTA-pair modes run under the
# 3xTF32 split (the 16-bit splits plan single-CTA or multicast launches only)
MODES = ["NB_TC_SPLIT=tf32,NB_TC_PAIR=1", "NB_TC_SPLIT=tf32,NB_TC_PAIR=2", "NB_TC_MC=1",
         "NB_TC_MC=2", "NB_TC_SPLIT=tf32,NB_TC_MC=1", "NB_TC_CONVH=0", "NB_TC_CONVH=1",
         "NB_TC_CONVH=2", "NB_TC_KSPLIT=0", "NB_TC_PDL=0", "NB_TC_KWF=0", "NB_TC_SPLIT=tf32",
         "NB_TC_SPLIT=bf16", "NB_TC_HALO=0", "NB_TC_HALO=0,NB_TC_CONVH=1",
         "NB_TC_HALO=0,NB_TC_SPLIT=tf32", "NB_TC_BN3=256", "NB_TC_SPLIT=tf32,NB_TC_BN3=256",
         "NB_TC_HALO=0,NB_TC_MC=1", "NB_TC_DEBUG=16384,NB_TC_HALO=0", "NB_TC_DEBUG=2097152"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES)
def test_tc_mode_exact_and_terminates(mode):
    env = dict(os.environ, **dict(kv.split("=") for kv in mode.split(",")))
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                       timeout=240, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (mode, r.stdout[-2000:],
                                                                    r.stderr[-2000:])
