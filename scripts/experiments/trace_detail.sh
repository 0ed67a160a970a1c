for sp in tf32 bf16; do for dbg in 0 2; do
  NB_TC_DEBUG=$dbg NB_TC_SPLIT=$sp NB_TC_TRACE=${IDX:-214} timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo "$sp dbg=$dbg"; python scripts/trace_detail.py nb_tc_trace.txt
done; done
