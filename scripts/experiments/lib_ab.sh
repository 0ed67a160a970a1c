# same-box A/B of two builds (NB200_LIB) on the origin evaluation and the bench
mkdir -p gpurun_out
for lib in libnb200_head.so libnb200.so; do
  for h in 1 0; do
    NB200_LIB=$lib NB_TC_HALO=$h NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of.txt 2>&1
    echo "== $lib halo=$h: $(sed -n 3p gpurun_out/of.txt)"; python scripts/trace_detail.py nb_tc_trace.txt 2>/dev/null | head -1 | cut -c1-40
    [ "$lib" = libnb200_head.so ] && break
  done
done
NB_TC_HALO=0 timeout 300 python -m pytest tests/test_sharded.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
NB_TC_HALO=1 timeout 300 python -m pytest tests/test_sharded.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
