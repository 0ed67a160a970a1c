"""TEST INFRASTRUCTURE: tests/golden/nest_cases.json -- execute<T>
(I/interp.hpp:67-145) of the UNMODIFIED reference (oracle/_ref) on conv
nests rewritten by DSL sequences, including the paper's Sequence 1 (no
ConvSpec: derived_spec == nullopt), in int64 and fp64, on seeded inputs."""
import json, os, sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Reference  # noqa: E402
from paper_2102_06599_b200.api import ConvSpec  # noqa: E402

SPECS = [ConvSpec(4, 16, 8, 8, 3, 3, 1, 1), ConvSpec(8, 8, 8, 6, 3, 3, 1, 1),
         ConvSpec(8, 16, 9, 9, 3, 3, 2, 1), ConvSpec(6, 12, 4, 4, 1, 1, 1, 0),
         ConvSpec(16, 32, 8, 8, 3, 3, 1, 1)]
DSLS = ["sequence1", "sequence1(2,2)", "sequence1(4,2)", "sequence1(2,4)", "sequence1(4,4)",
        "sequence2(4,2)", "sequence3(2,4)", "interchange(co,ci) | unroll(co,4)",
        "tile(ci,2) | interchange(w,kh)", "group(co,ci,2) | interchange(h,w)"]


def main():
    R = Reference()
    cases = []
    for si, s in enumerate(SPECS):
        for dsl in DSLS:
            rng = np.random.default_rng(1000 * si + len(cases))
            x = rng.integers(-3, 4, size=(s.ci, s.h, s.w)).astype(np.int64)
            w = rng.integers(-3, 4, size=(s.co_eff(), s.ci, s.kh, s.kw)).astype(np.int64)
            try:
                yi = R.execute(s, dsl, x, w)
            except Exception as e:  # the rewrite does not apply to this spec
                print("skip", s.to_json(), dsl, str(e)[:60])
                continue
            yf = R.execute(s, dsl, x * 0.37, w * 1.3)
            d = R.derived_spec(s, dsl)
            cases.append({"spec": s.to_json(), "dsl": dsl, "seed": 1000 * si + len(cases),
                          "has_spec": bool(d), "macs": R.count_macs(s, dsl),
                          "out_int": yi.ravel().tolist(), "out_f64": yf.ravel().tolist()})
    out = os.path.join(os.path.dirname(HERE), "tests", "golden", "nest_cases.json")
    json.dump({"generator": "oracle/gen_nest_golden.py (execute, I/interp.hpp:67)",
               "cases": cases}, open(out, "w"), separators=(",", ":"))
    print(len(cases), "cases,", sum(not c["has_spec"] for c in cases), "without a ConvSpec")


if __name__ == "__main__":
    main()
