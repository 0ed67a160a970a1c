# dgrad L1 (kw-fused, fused Fisher epilogue): launch time under epilogue debug bits
for dbg in 0 2048 4096 8192 14336 16; do
  NB_TC_DEBUG=$dbg NB_TC_TRACE=${IDX:-254} timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo -n "dbg=$dbg "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-140
done
