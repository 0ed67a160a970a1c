for k in 1 0 1 0; do
  NB_TC_KWF=$k timeout 60 python scripts/origin_fisher.py 6 fp32 > gpurun_out/of.txt 2>&1
  o=$(grep "fisher [3-5]" gpurun_out/of.txt | awk '{print $3}' | sort -n | head -1)
  NB_TC_KWF=$k timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "kwf=$k origin_ms=$o $(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1), 'inf', round(d['inference_ms'],3))")"
done
