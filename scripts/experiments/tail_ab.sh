# tail-epilogue helpers on / off (NB_TC_DEBUG bit 2^21): bench and launch timelines
for dbg in 0 16777216; do
  for i in 1 2; do
    NB_TC_DEBUG=$dbg timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
    echo "dbg=$dbg $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1))")"
  done
done
