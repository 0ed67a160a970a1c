for h in 0 1; do
NB_TC_HALO=$h NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
echo "== halo $h"
python - <<'PY'
import numpy as np
t = np.array([[int(x) for x in l.split()[1:]] for l in open("nb_tc_trace.txt") if not l.startswith("#")], dtype=np.int64)
t = t[(t[:, 0] > 0)][:40]
t0 = t[0, 0]
print("kb  issue  wait7   cs    ce   mmaR  mmaC | c-gap  cs-issue  cs-wait  mmaR-ce")
prev = None
for i, r in enumerate(t):
    cs, ce = (r[1], r[2]) if r[1] > 0 else (r[5], r[6])
    w7 = r[7] if r[7] > 0 else 0
    print(f"{i:2d} {r[0]-t0:6d} {(w7-t0) if w7 else -1:6d} {cs-t0:6d} {ce-t0:6d} {r[3]-t0:6d} {r[4]-t0:6d} | {(r[4]-prev) if prev else 0:5d} {cs-r[0]:6d} {(cs-w7) if w7 else -1:6d} {r[3]-ce:6d}")
    prev = r[4]
PY
done
