timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tc_modes.py tests/test_r34_parity.py tests/test_sharded.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for dbg in 16384 0 16384 0; do
  NB_TC_DEBUG=$dbg timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB_TC_DEBUG=$dbg timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "dbg=$dbg origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'dgrad', round(r['achieved'],1))")"
done
