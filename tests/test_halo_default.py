"""The halo-tile A operand is the default tensor-core path: on the R34 origin
Fisher evaluation at N=128 most launches take it (NB_TC_HALO_LOG prints each
launch's decision: every stride-1 multi-tap phase grid whose box fits, including
the stride-2 dgrads' sub-pixel phases), and NB_TC_HALO=0 turns it off.  The totals of both A operands agree within the
FP32 tier's tolerance (they only differ in the K order)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, %r)
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import Precision
from paper_2102_06599_b200.workloads import resnet34_chain
net = resnet34_chain()
ctx = nb.Context(0)
batch = nb.make_batch(net, 128, 1)
print("total", repr(nb.fisher_potential(net, batch, precision=Precision.FP32, ctx=ctx).total))
""" % ROOT


def run(env):
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=dict(os.environ, **env), cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    total = float(next(l for l in r.stdout.splitlines() if l.startswith("total")).split()[1])
    modes = [l.split() for l in r.stderr.splitlines() if l.startswith("tc mode")]
    return total, [(int(m[16]), int(m[18]), int(m[20])) for m in modes]  # (ksplit, taps, halo)


@pytest.mark.gpu
def test_halo_is_the_default_and_agrees():
    t_on, on = run({"NB_TC_HALO_LOG": "1"})
    t_off, off = run({"NB_TC_HALO_LOG": "1", "NB_TC_HALO": "0"})
    assert on and off and len(on) == len(off)
    assert sum(h for _, _, h in on) >= len(on) // 3, on   # most 3x3 stride-1 launches
    assert all(h == 0 for _, _, h in off)
    assert abs(t_on - t_off) <= 5e-4 * abs(t_off)          # TOLERANCE[FP32] on totals
