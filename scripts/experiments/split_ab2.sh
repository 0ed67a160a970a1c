mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_r34_parity.py tests/test_tc_modes.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
timeout 400 python scripts/r34_err.py > gpurun_out/r34_err_f16.txt 2>&1; echo "r34 rc=$?"; cut -c1-75 gpurun_out/r34_err_f16.txt
for sp in f16 bf16 tf32; do
  NB_TC_SPLIT=$sp NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of_$sp.txt 2>&1
  echo "$sp"; head -4 gpurun_out/of_$sp.txt; python scripts/trace_detail.py nb_tc_trace.txt | head -1
  NB_TC_SPLIT=$sp timeout 300 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench_$sp.log 2>&1
  echo "bench $sp rc=$?"; tail -1 gpurun_out/bench_$sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['e2e']['value'], r['kernel'], r['achieved'], r['launch_ms'], d['inference_ms'])"
done
