"""Summarise an NB_TC_TRACE capture (nb_tc_trace.txt + nb_tc_ctas.txt):
stage period of CTA 0 (median cycles between MMA commits), MMA wait for
ready (converter/TMA latency), and the CTA timeline (first start, median and
max MMA-done / end) in us."""
import sys
import numpy as np
tr = [l.split() for l in open(sys.argv[1]) if not l.startswith("#")]
hdr = open(sys.argv[1]).readline().strip()
t = np.array([[int(x) for x in r[1:]] for r in tr], dtype=np.int64)
t = t[t[:, 4] > 0]
per = np.diff(t[:, 4])
ct = np.array([[int(x) for x in l.split()] for l in open(sys.argv[2])], dtype=np.int64)
t0 = ct[:, 2].min()
print(f"{hdr} | stages {len(t)} period med {np.median(per):.0f} p90 {np.percentile(per, 90):.0f} cyc"
      f" | conv lat med {np.median(t[:, 2] - t[:, 1]):.0f} | ctas {len(ct)} start max {(ct[:,2].max()-t0)/1e3:.1f}"
      f" mma-done med {(np.median(ct[:, 3]) - t0)/1e3:.1f} max {(ct[:, 3].max() - t0)/1e3:.1f}"
      f" end med {(np.median(ct[:, 4]) - t0)/1e3:.1f} max {(ct[:, 4].max() - t0)/1e3:.1f} us")
