"""Accuracy probe of the conv kernels (fp32 SIMT / 3xTF32 / 1xTF32) against the
fp64 oracle: max and rms of |gpu - ref| / (sum |w||x|) per output, for fprop
and dgrad at K up to 4608.  Test infrastructure (uses oracle/)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Precision
from oracle.oracle import Restatement

O = Restatement()
ctx = nb.Context(0)
specs = [ConvSpec(64, 64, 16, 16, 3, 3, 1, 1), ConvSpec(256, 256, 8, 8, 3, 3, 1, 1),
         ConvSpec(512, 512, 4, 4, 3, 3, 1, 1)]
rng = np.random.default_rng(0)
for s in specs:
    x = np.maximum(rng.standard_normal((2, s.ci, s.h, s.w)), 0)
    w = rng.standard_normal((s.co_eff(), s.ci, s.kh, s.kw)) / np.sqrt(s.ci * 9)
    want = np.stack([O.conv(s, x[i], w) for i in range(2)])
    scale = np.stack([O.conv(s, np.abs(x[i]), np.abs(w)) for i in range(2)])
    dy = rng.standard_normal((2,) + s.output_shape())
    dwant = np.stack([O.conv_dgrad(s, dy[i], w) for i in range(2)])
    dscale = np.stack([O.conv_dgrad(s, np.abs(dy[i]), np.abs(w)) for i in range(2)])
    for name, p in [("simt", Precision.SIMT), ("3xtf32", Precision.FP32), ("tf32", Precision.TF32)]:
        y = nb.reference_conv(s, x, w, precision=p, ctx=ctx)
        e = np.abs(y - want) / scale
        d = nb.conv_dgrad(s, dy, w, precision=p, ctx=ctx)
        de = np.abs(d - dwant) / dscale
        sb = np.mean(y - want) / np.mean(scale)
        print(f"K={s.ci*9:5d} {name:7s} fprop max {e.max():.2e} rms {np.sqrt((e**2).mean()):.2e} "
              f"bias {sb:+.2e} | dgrad max {de.max():.2e} rms {np.sqrt((de**2).mean()):.2e}", flush=True)
