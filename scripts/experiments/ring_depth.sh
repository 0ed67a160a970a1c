# stage period vs ring depth (NB_TC_DEBUG bits 16..19 cap the stages) and without B / A loads
for h in 0 1; do
for dbg in 0 $((5 << 16)) $((4 << 16)) 8 4; do
  NB_TC_HALO=$h NB_TC_DEBUG=$dbg NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo -n "halo $h dbg $dbg: "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-110
done; done
