# FP32-tier splits (3xf16 default, 3xbf16, 3xtf32): parity tests, accuracy probes, bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/split_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/split_pytest.log
timeout 300 python scripts/acc_probe.py > gpurun_out/acc_f16.txt 2>&1; echo "acc rc=$?"; grep -v simt gpurun_out/acc_f16.txt | grep -v " tf32 "
timeout 400 python scripts/r34_err.py > gpurun_out/r34_err_f16.txt 2>&1; echo "r34 rc=$?"; cut -c1-75 gpurun_out/r34_err_f16.txt
for sp in f16 tf32; do
  NB_TC_SPLIT=$sp timeout 300 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench_$sp.log 2>&1
  echo "bench $sp rc=$?"; tail -1 gpurun_out/bench_$sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], d['e2e']['value'], r['kernel'], r['achieved'], r['launch_ms'], d['inference_ms'])"
done
