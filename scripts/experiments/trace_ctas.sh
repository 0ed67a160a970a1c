mkdir -p gpurun_out
for idx in ${IDXS:-192 200 212 224 228 240 252}; do
  NB_TC_TRACE=$idx timeout 120 python scripts/origin_fisher.py 3 ${PREC:-fp32} > /dev/null 2>&1
  cp nb_tc_ctas.txt gpurun_out/ctas_$idx.txt; cp nb_tc_trace.txt gpurun_out/trace_idx$idx.txt
done
