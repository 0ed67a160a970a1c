# epilogue event timeline of CTA 0 for a few origin-Fisher TC launches
for idx in ${IDXS:-131 139 171 194 236 254}; do
  NB_TC_TRACE=$idx timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  head -1 nb_tc_trace.txt | cut -c1-150
  python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-140
  python scripts/experiments/epi_trace.py nb_tc_trace.txt
done
