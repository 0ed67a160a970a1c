timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_r34_parity.py tests/test_sharded.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for idx in 254 236; do
  NB_TC_TRACE=$idx timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  echo -n "$idx "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-140
done
for i in 1 2; do
  timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1))")"
done
