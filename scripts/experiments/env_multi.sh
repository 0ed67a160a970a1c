# same-box comparison of several environment settings (ENVS: ';'-separated)
IFS=';' read -ra SETS <<< "${ENVS:-NB_NONE=0;NB_NONE=1}"
for round in 1 2; do
for envs in "${SETS[@]}"; do
  env $envs timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  env $envs timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks --no-inference > gpurun_out/bench.log 2>&1
  echo "$envs origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'dgrad', round(r['achieved'],1))" 2>/dev/null)"
done
done
