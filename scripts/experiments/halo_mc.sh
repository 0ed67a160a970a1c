NB_TC_HALO=1 NB_TC_MC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "integer" 2>&1 | tail -1
for cfg in "0 0" "1 0" "0 1" "1 1" "1 2"; do
  set -- $cfg
  NB_TC_HALO=$1 NB_TC_MC=$2 timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB_TC_HALO=$1 NB_TC_MC=$2 NB_TC_TRACE=214 timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  t=$(python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/.*| stages/stages/' | cut -c1-100)
  NB_TC_HALO=$1 NB_TC_MC=$2 timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "halo=$1 mc=$2 origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1))") | $t"
done
