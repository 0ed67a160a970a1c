NB_TC_HALO=1 NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
python - <<'PY'
import numpy as np
t = np.array([[int(x) for x in l.split()[1:]] for l in open("nb_tc_trace.txt") if not l.startswith("#")], dtype=np.int64)
t = t[(t[:, 0] > 0)][:40]
t0 = t[0, 0]
print("kb issue g0s g0e mmaR mmaC g1s g1e g0wait")
for i, r in enumerate(t):
    print(i, " ".join(f"{(x - t0) if x > 0 else -1:7d}" for x in [r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7]]))
PY
