NB_TC_HALO=${H:-0} NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
python - <<'PY'
import numpy as np
t = np.array([[int(x) for x in l.split()[1:]] for l in open("nb_tc_trace.txt") if not l.startswith("#")], dtype=np.int64)
t = t[(t[:, 0] > 0)][:72]
t0 = t[0, 0]
print("kb issue  cs   ce   mmaR mmaC | commit-gap  conv-start-minus-issue  mmaR-minus-ce")
prev = None
for i, r in enumerate(t):
    cs, ce = (r[1], r[2]) if r[1] > 0 else (r[5], r[6])
    print(i, " ".join(f"{x - t0:6d}" for x in [r[0], cs, ce, r[3], r[4]]), "|", (r[4] - prev) if prev else 0, cs - r[0], r[3] - ce)
    prev = r[4]
PY
