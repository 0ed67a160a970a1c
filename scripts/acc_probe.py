"""Accumulation-error probe of the tensor-core conv path (GPU experiment).

1x1 convs with K = Ci input channels and tf32-exact operands, so every
product is exact and any error is the accumulation's.  For K in a sweep and
for all-positive / random-sign operands, prints the mean signed relative error
(bias) and the rms relative error of TF32 / 3xTF32 / SIMT outputs against the
exact fp64 sum.  N*H*W = 32768 output pixels = 256 M tiles, so no split-K.
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Precision


def tf32(a):
    b = a.astype(np.float32).view(np.uint32)
    b = (b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    return b.view(np.float32).astype(np.float64)


ctx = nb.Context(0)
rng = np.random.default_rng(0)
print("K sign mode bias rms(rel |y|) rms(rel sum|wx|)")
for K in (64, 512, 2048, 4096):
    s = ConvSpec(K, 128, 32, 32, 1, 1, 1, 0)
    for sign in ("pos", "rand"):
        x = rng.standard_normal((32, K, 32, 32))
        w = rng.standard_normal((128, K, 1, 1))
        if sign == "pos":
            x, w = np.abs(x), np.abs(w)
        x, w = tf32(x), tf32(w)
        exact = np.einsum("nchw,oc->nohw", x, w[:, :, 0, 0])
        scale = np.einsum("nchw,oc->nohw", np.abs(x), np.abs(w[:, :, 0, 0]))
        for name, p in (("tf32", Precision.TF32), (nb.fp32_split(), Precision.FP32),
                        ("simt", Precision.SIMT)):
            y = nb.reference_conv(s, x, w, precision=p, ctx=ctx)
            m = np.abs(exact) > 1e-3 * scale
            rel = (y - exact)[m] / np.abs(exact[m])
            print(f"{K:5d} {sign:4s} {name:6s} bias {np.mean(np.sign(exact[m]) * rel):+.3e} "
                  f"rms {np.sqrt(np.mean(rel ** 2)):.3e} "
                  f"rms/sum {np.sqrt(np.mean(((y - exact) / scale) ** 2)):.3e}", flush=True)
