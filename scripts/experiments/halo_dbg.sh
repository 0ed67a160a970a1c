for cfg in "0 0" "1 0" "1 32" "1 1024" "0 32"; do
  set -- $cfg
  NB_TC_HALO=$1 NB_TC_DEBUG=$2 NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo -n "halo $1 dbg $2: "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-150
  python - <<'PY'
import numpy as np
t = np.array([[int(x) for x in l.split()[1:]] for l in open("nb_tc_trace.txt") if not l.startswith("#")], dtype=np.int64)
t = t[(t[:, 0] > 0)][4:40]
g0 = t[t[:, 1] > 0]; g1 = t[t[:, 5] > 0]
print("   g0 conv", int(np.median(g0[:, 2] - g0[:, 1])), " g1 conv", int(np.median(g1[:, 6] - g1[:, 5])))
PY
done
