"""The masked box executor beside the interpreter: wall
time per call of execute (nb_nest_execute, one thread per MAC instance,
int64 atomics) and execute_boxes (cell pass + tensor-core box convs,
FP32 tier) on Sequence-1 forms of growing layers; both calls include the
bridge's nest rewriting, the reference-layout copies and a fresh context."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2102_06599_b200 import ConvSpec
from paper_2102_06599_b200 import search as S

print("| spec | dsl | nest MACs | boxes | interpreter ms | box executor ms | equal |")
print("|---|---|---|---|---|---|---|")
for ci, co, hw, dsl in [(16, 32, 16, "sequence1(2,2)"), (64, 64, 32, "sequence1(2,2)"),
                        (64, 128, 32, "sequence1(2,4)"), (128, 128, 32, "sequence1(4,2)")]:
    spec = ConvSpec(ci, co, hw, hw, 3, 3, 1, 1)
    rng = np.random.default_rng(0)
    x = rng.integers(-3, 4, size=(ci, hw, hw)).astype(np.int64)
    w = rng.integers(-3, 4, size=(co, ci, 3, 3)).astype(np.int64)
    t = []
    for fn in (lambda: S.execute_gpu(spec, dsl, x, w), lambda: S.execute_boxes_gpu(spec, dsl, x, w)[0]):
        fn()
        t0 = time.perf_counter()
        for _ in range(3):
            y = fn()
        t.append((1e3 * (time.perf_counter() - t0) / 3, y))
    _, st = S.execute_boxes_gpu(spec, dsl, x, w)
    print(f"| {ci}->{co} @{hw} | {dsl} | {st['nest_macs']} | {st['boxes']} | {t[0][0]:.1f} | "
          f"{t[1][0]:.1f} | {np.array_equal(t[0][1], t[1][1])} |", flush=True)
