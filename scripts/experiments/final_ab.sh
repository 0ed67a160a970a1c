# same-box A/B: builds x halo mode, single-stream origin Fisher and the 4-session bench
for cfg in "libnb200_head.so 0" "libnb200_g2.so 0" "libnb200_g2.so 1" "libnb200.so 0" "libnb200.so 1"; do
  set -- $cfg
  NB200_LIB=$1 NB_TC_HALO=$2 timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB200_LIB=$1 NB_TC_HALO=$2 timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "$1 halo=$2 origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'dgrad', round(r['achieved'],1), 'inf', round(d['inference_ms'],3))")"
done
