# stage period of one launch under the NB_TC_DEBUG experiment bits, per split
for sp in ${SPLITS:-tf32 bf16}; do
  for dbg in 0 32 12 44 2 34 4 8; do
    NB_TC_DEBUG=$dbg NB_TC_SPLIT=$sp NB_TC_TRACE=${IDX:-214} timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
    echo -n "$sp dbg=$dbg "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/'
  done
done
