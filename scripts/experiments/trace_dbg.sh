mkdir -p gpurun_out
for dbg in ${DBGS:-0 32 12 44}; do
  NB_TC_TRACE=200 NB_TC_DEBUG=$dbg timeout 120 python scripts/origin_fisher.py 3 > /dev/null 2>&1
  echo "debug=$dbg"; head -1 nb_tc_trace.txt
  awk 'NR>22 && NR<120 {d=$6-$5; s+=d; n++; if (p) {g+=$5-p; m++}; p=$6} END {printf "  MMA issue/stage %.0f  gap %.0f  period %.0f\n", s/n, g/m, (s+g)/n}' nb_tc_trace.txt
  cp nb_tc_trace.txt gpurun_out/trace_dbg$dbg.txt
done
