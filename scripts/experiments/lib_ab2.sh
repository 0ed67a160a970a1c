for lib in libnb200_head.so libnb200_v1.so libnb200.so; do
  NB200_LIB=$lib NB_TC_HALO=0 NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of.txt 2>&1
  echo "== $lib: $(sed -n 3p gpurun_out/of.txt)"; python scripts/trace_detail.py nb_tc_trace.txt 2>/dev/null | head -4
done
