# same-box A/B of library builds (NB200_LIB): origin Fisher (1 stream) and the 4-session bench
for round in 1 2; do
for lib in ${LIBS:-libnb200_A.so libnb200_B.so libnb200.so}; do
  NB200_LIB=$lib timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB200_LIB=$lib timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "$lib origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'dgrad', round(r['achieved'],1), 'inf', round(d['inference_ms'],3), 'inf_origin', round(d['inference_origin_ms'],3))")"
done
done
