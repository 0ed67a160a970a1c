"""Per-evaluation timings of SURVEY 8(d)'s configs beside the bench's C2
search: C1 (single 3x3 conv 64->64 32x32, N=8: std / g4 / b2 / dw), C2 (R34
origin, N=128), C3 (ResNeXt-29 origin, N=128) and C4 (the 78 DenseNet-161
dense layers, each a 2-conv chain, N=128).

For each: fisher_potential through a session (synchronous call: the wall
time includes host launch and the result copies) and, separately, the sum of
the device time of its kernels (CUDA events per launch, one profiled pass);
forward only (inference) the same way.  Algorithmic FLOPs are nb_fisher_flops
/ 2*N*network_macs (count_macs, padded taps included).  Prints a markdown
table."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06599_b200 as nb  # noqa: E402
from paper_2102_06599_b200 import Precision  # noqa: E402
from paper_2102_06599_b200.workloads import (c1_network, densenet161_layer_chains,  # noqa: E402
                                             resnet34_chain, resnext29_chain)

PREC = {"fp32": Precision.FP32, "tf32": Precision.TF32}[sys.argv[1] if len(sys.argv) > 1 else "fp32"]
REPS = 10


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(REPS):
        t = time.perf_counter()
        fn()
        ts.append(1e3 * (time.perf_counter() - t))
    return statistics.median(ts)


def device_ms(ctx, fn):
    ctx.reset_stats()
    ctx.set_profiling(True)
    fn()
    ctx.set_profiling(False)
    return sum(v["ms"] for k, v in ctx.kernel_stats().items() if not k.startswith("host_"))


def measure(ctx, nets, n):
    """Sum over `nets` (each its own session) of wall / device ms."""
    fw = fd = iw = idv = fl = ifl = 0.0
    for net in nets:
        s = nb.Session(net, nb.make_batch(net, n, 1), ctx=ctx)
        fw += timed(lambda: s.fisher(net, PREC))
        fd += device_ms(ctx, lambda: s.fisher(net, PREC))
        iw += timed(lambda: s.forward(net, PREC))
        idv += device_ms(ctx, lambda: s.forward(net, PREC))
        fl += nb.fisher_flops(net, n)
        ifl += 2.0 * n * nb.network_macs(net)
        s.close()
    return fw, fd, fl, iw, idv, ifl


def main():
    ctx = nb.Context(0)
    rows = [
        ("C1 std (N=8)", [c1_network()], 8),
        ("C1 g4 (N=8)", [c1_network(groups=4)], 8),
        ("C1 b2 (N=8)", [c1_network(bottleneck=2)], 8),
        ("C1 dw (N=8)", [c1_network(groups=64)], 8),
        ("C2 R34 origin (N=128)", [resnet34_chain()], 128),
        ("C3 ResNeXt-29 origin (N=128)", [resnext29_chain()], 128),
        ("C4 DenseNet-161, 78 dense layers (N=128)", densenet161_layer_chains(), 128),
    ]
    print(f"precision {'fp32 (3xTF32)' if PREC == Precision.FP32 else 'tf32'}\n")
    print("| config | Fisher GFLOP | Fisher wall ms | Fisher device ms | TFLOP/s (device) "
          "| inference GFLOP | inference wall ms | inference device ms | TFLOP/s (device) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name, nets, n in rows:
        fw, fd, fl, iw, idv, ifl = measure(ctx, nets, n)
        print(f"| {name} | {fl / 1e9:.1f} | {fw:.3f} | {fd:.3f} | {fl / fd / 1e9:.1f} "
              f"| {ifl / 1e9:.1f} | {iw:.3f} | {idv:.3f} | {ifl / idv / 1e9:.1f} |", flush=True)


if __name__ == "__main__":
    main()
