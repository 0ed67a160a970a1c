# per-stage traces of several tcgen05 launches (indices into the launch
# order of scripts/origin_fisher.py 3: 4 evaluations x 64 TC launches)
mkdir -p gpurun_out
for idx in ${IDXS:-192 200 212 224 228 240 252}; do
  NB_TC_TRACE=$idx timeout 120 python scripts/origin_fisher.py 3 ${PREC:-fp32} > /dev/null 2>&1
  cp nb_tc_trace.txt gpurun_out/trace_idx$idx.txt
done
