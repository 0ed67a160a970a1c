for ch in 0 0; do
  NB_TC_CONVH=$ch timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB_TC_CONVH=$ch NB_TC_TRACE=214 timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  t=$(python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-100)
  NB_TC_CONVH=$ch timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "convh=$ch origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1))") | $t"
done
