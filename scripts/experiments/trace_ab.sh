# stage periods and CTA timelines of origin-evaluation TC launches, per split
mkdir -p gpurun_out
for sp in ${SPLITS:-tf32 bf16}; do
  echo "== split $sp"; NB_TC_SPLIT=$sp timeout 120 python scripts/origin_fisher.py 3 fp32 | head -4
  for idx in ${IDXS:-196 206 214 222 226 236 246 254}; do
    NB_TC_SPLIT=$sp NB_TC_TRACE=$idx timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
    echo -n "$idx "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt
  done
done
