mkdir -p gpurun_out
for dbg in ${DBGS:-0}; do
  NB_TC_TRACE=${IDX:-250} NB_TC_DEBUG=$dbg timeout 120 python scripts/origin_fisher.py 3 > /dev/null 2>&1
  cp nb_tc_ctas.txt gpurun_out/ctasd_${IDX:-250}_$dbg.txt
done
