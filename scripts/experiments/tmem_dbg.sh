for dbg in 0 512 32 2 514; do
  NB_TC_HALO=0 NB_TC_DEBUG=$dbg NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo -n "dbg $dbg: "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-110
done
