# converter group mode A/B: NB_TC_CONVH=1 (both groups, channel halves) vs 0 (alternate stages)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_modes.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
for cfg in "f16 1" "f16 0" "bf16 0" "tf32 0"; do
  set -- $cfg
  NB_TC_CONVH=$2 NB_TC_SPLIT=$1 NB_TC_TRACE=214 timeout 120 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of.txt 2>&1
  echo "== $1 convh=$2: $(sed -n 3p gpurun_out/of.txt)"; python scripts/trace_detail.py nb_tc_trace.txt 2>/dev/null | head -1
  NB_TC_CONVH=$2 NB_TC_SPLIT=$1 timeout 300 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), round(d['e2e']['value'],1), r['kernel'], round(r['achieved'],1), round(d['inference_ms'],3))"
done
