# trace launch IDX under several NB_TC_DEBUG settings
mkdir -p gpurun_out
for dbg in ${DBGS:-0 4 8}; do
  NB_TC_TRACE=${IDX:-192} NB_TC_DEBUG=$dbg timeout 120 python scripts/origin_fisher.py 3 ${PREC:-fp32} > /dev/null 2>&1
  cp nb_tc_trace.txt gpurun_out/trace_mix_${IDX:-192}_$dbg.txt
done
