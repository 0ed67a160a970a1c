"""Epilogue events of CTA 0 (trace role 9, NB_TC_TRACE capture): per tile,
cycles from the accumulator wait to each 16-column chunk's end, the final
partial sums and the accumulator release."""
import sys
import numpy as np
rows = [l.split() for l in open(sys.argv[1]) if not l.startswith("#")]
e = np.array([int(r[-1]) for r in rows], dtype=np.int64)
for t in range(10):
    s = e[t * 24:(t + 1) * 24]
    if s[0] == 0:
        break
    base = s[1]
    ch = [int(x - base) for x in s[2:18] if x]
    print(f"tile {t}: wait {s[1] - s[0]} | chunks {ch} | sums {s[18] - base if s[18] else '-'}"
          f" | release {s[19] - base}")
