# per-launch CTA timelines, halo off / on, for launches of the 4th origin evaluation
for idx in ${IDXS:-196 200 206 210 214 222 226 236 240 246 250 254}; do
  for h in 0 1; do
    NB_TC_HALO=$h NB_TC_TRACE=$idx timeout 120 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
    echo -n "$idx h$h "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | cut -c1-250
  done
done
