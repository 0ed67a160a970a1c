for cfg in "libnb200_head.so 0" "libnb200.so 0" "libnb200.so 1"; do
  set -- $cfg
  NB200_LIB=$1 NB_TC_HALO=$2 NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of.txt 2>&1
  echo "== $1 halo=$2: $(sed -n 3p gpurun_out/of.txt)"; python scripts/trace_detail.py nb_tc_trace.txt 2>/dev/null | head -1 | cut -c1-40
done
NB_TC_HALO=1 timeout 300 python -m pytest tests/test_sharded.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
