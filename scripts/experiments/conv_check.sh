# converter rework: parity subset, stage traces, bench A/B of the splits
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_modes.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
bash scripts/trace_detail.sh
for sp in bf16 tf32; do
  NB_TC_SPLIT=$sp timeout 300 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench_$sp.log 2>&1
  echo "bench $sp rc=$?"; tail -1 gpurun_out/bench_$sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['e2e']['value'], r['kernel'], r['achieved'], r['launch_ms'], d['inference_ms'])"
done
