"""Per-stage breakdown of an NB_TC_TRACE capture (CTA 0, clock64 cycles):
medians over the steady-state stages.  Roles (kernels_tc.cu trace()):
0 issue, 1/2 converter group 0 start/done, 3/4 MMA ready/commit,
5/6 group 1 start/done, 7/8 group 0 wait begin / A landed."""
import sys
import numpy as np
t = np.array([[int(x) for x in l.split()[1:]] for l in open(sys.argv[1]) if not l.startswith("#")],
             dtype=np.int64)
t = t[(t[:, 4] > 0) & (t[:, 0] > 0)]
s = t[4:-4] if len(t) > 12 else t
m = lambda a: int(np.median(a))
print(f"issue-gap {m(np.diff(s[:, 0]))} commit-gap {m(np.diff(s[:, 4]))} | g0: wait-A {m(s[:, 8] - s[:, 7])}"
      f" wait-tfree {m(s[:, 1] - s[:, 8])} conv {m(s[:, 2] - s[:, 1])} done->next-wait {m(s[1:, 7] - s[:-1, 2])}"
      f" | g1: conv {m(s[:, 6] - s[:, 5])} start-skew(g1-g0) {m(s[:, 5] - s[:, 1])}"
      f" | ready->mma {m(s[:, 3] - np.maximum(s[:, 2], s[:, 6]))} mma {m(s[:, 4] - s[:, 3])}"
      f" | issue->A-landed {m(s[:, 8] - s[:, 0])}")
for r in s[:5]:
    print("   ", " ".join(f"{x - s[0, 0]:6d}" for x in r))
