"""BASELINE configs[4]: ImageNet-shape (N=256) transformed-conv kernel sweep
over channels / groups against the HBM and tensor-pipe rooflines.

For each (C @ HW, G) a one-layer network runs forward (conv + head) and
forward+backward (Fisher: adds the dgrad) on a resident N=256 batch; the
conv kernels' device times come from per-launch CUDA events (kernel_stats).
Algorithmic FLOPs = 2*N*count_macs; bytes = 4*(N*H*W*C in + N*H*W*C out +
weights).  Prints one JSON line per point and a markdown table."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb
from paper_2102_06599_b200 import ConvSpec, Layer, Network, Precision

N = int(os.environ.get("SWEEP_N", "256"))
PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
HBM, BF16 = PEAKS["hbm_gbs"], PEAKS["bf16_tflops"]
prec = {"fp32": Precision.FP32, "tf32": Precision.TF32, "simt": Precision.SIMT}[
    os.environ.get("SWEEP_PREC", "fp32")]
ctx = nb.Context(0)
rows = []
for c, hw in [(64, 56), (128, 28), (256, 14), (512, 7)]:
    shape = Network([Layer(ConvSpec(c, c, hw, hw, 3, 3, 1, 1))], num_classes=10, seed=42)
    sess = nb.Session(shape, nb.make_batch(shape, N, 1), ctx=ctx)
    # SWEEP_GROUPS=dw: the depthwise points only
    for g in ([c] if os.environ.get("SWEEP_GROUPS") == "dw" else sorted({1, 2, 4, 8, 32, c})):
        net = Network([Layer(ConvSpec(c, c, hw, hw, 3, 3, 1, 1, groups=g))], num_classes=10, seed=42)
        macs = nb.count_macs(net.layers[0].spec)
        flops = 2.0 * N * macs
        bytes_ = 4.0 * (2 * N * hw * hw * c + c * (c // g) * 9)
        for _ in range(2):
            sess.forward(net, prec)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(5):
            sess.forward(net, prec)
        ctx.set_profiling(False)
        st = {k: v for k, v in ctx.kernel_stats().items() if k.startswith("conv_")}
        ms = sum(v["ms"] for v in st.values()) / 5
        fam = max(st, key=lambda k: st[k]["ms"])
        tfs = flops / (ms / 1e3) / 1e12
        gbs = bytes_ / (ms / 1e3) / 1e9
        tc = "tc" in fam
        # dgrad: the target conv as layer 2 behind two 1x1 convs, timed through
        # a Fisher evaluation -- a middle layer's dgrad: it reads dpre and
        # a_prev and writes the masked dpre of layer 1 (layer 0 has no dgrad)
        net2 = Network([Layer(ConvSpec(c, c, hw, hw, 1, 1, 1, 0)),
                        Layer(ConvSpec(c, c, hw, hw, 1, 1, 1, 0)),
                        Layer(ConvSpec(c, c, hw, hw, 3, 3, 1, 1, groups=g))], num_classes=10, seed=42)
        sess.fisher(net2, prec)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(3):
            sess.fisher(net2, prec)
        ctx.set_profiling(False)
        # the target layer's dgrad launches only (layer 1's 1x1 dgrad is a
        # separate record: the stats are per kernel family, so time the
        # target alone by subtracting a run of the 1x1 pair)
        dst = {k: v for k, v in ctx.kernel_stats().items() if k.startswith("conv_dgrad")}
        net3 = Network([Layer(ConvSpec(c, c, hw, hw, 1, 1, 1, 0)),
                        Layer(ConvSpec(c, c, hw, hw, 1, 1, 1, 0))], num_classes=10, seed=42)
        sess.fisher(net3, prec)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(3):
            sess.fisher(net3, prec)
        ctx.set_profiling(False)
        base = {k: v for k, v in ctx.kernel_stats().items() if k.startswith("conv_dgrad")}
        dms = (sum(v["ms"] for v in dst.values()) - sum(v["ms"] for v in base.values())) / 3
        dfam = max(dst, key=lambda k: dst[k]["ms"] - base.get(k, {"ms": 0.0})["ms"])
        # dpre read + a_prev read + masked dpre write (no dX store) + weights
        dbytes = 4.0 * (3 * N * hw * hw * c + c * (c // g) * 9)
        row = {"C": c, "HW": hw, "G": g, "family": fam, "us": round(ms * 1e3, 2),
               "dgrad_family": dfam, "dgrad_us": round(dms * 1e3, 2),
               "dgrad_tflops": round(flops / (dms / 1e3) / 1e12, 2),
               "dgrad_gbs": round(dbytes / (dms / 1e3) / 1e9, 1),
               "dgrad_frac_hbm": round(dbytes / (dms / 1e3) / 1e9 / HBM, 3),
               "tflops": round(tfs, 2), "gbs": round(gbs, 1),
               "frac_tensor_bf16": round(tfs / BF16, 4), "frac_hbm": round(gbs / HBM, 4),
               "bound": "tensor" if tc else "hbm", "ai_flop_per_byte": round(flops / bytes_, 1)}
        rows.append(row)
        print(json.dumps(row), flush=True)
print()
print(f"| C@HW | G | fprop kernel | us | TFLOP/s | GB/s | frac bf16 | frac HBM | AI | dgrad kernel | us | TFLOP/s | GB/s | frac HBM |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print(f"| {r['C']}@{r['HW']} | {r['G']} | `{r['family']}` | {r['us']} | {r['tflops']} | {r['gbs']} | "
          f"{r['frac_tensor_bf16']:.3f} | {r['frac_hbm']:.3f} | {r['ai_flop_per_byte']} | "
          f"`{r['dgrad_family']}` | {r['dgrad_us']} | {r['dgrad_tflops']} | {r['dgrad_gbs']} | {r['dgrad_frac_hbm']} |")
