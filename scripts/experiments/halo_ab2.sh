mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_tc_modes.py tests/test_r34_parity.py tests/test_sharded.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
timeout 400 python scripts/r34_err.py 2>&1 | cut -c1-75 | head -14
bash scripts/halo_dbg.sh 2>&1 | head -4
for h in 1 0; do
  NB_TC_HALO=$h timeout 300 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('halo $h bench', round(d['value'],1), round(d['e2e']['value'],1), r['kernel'], round(r['achieved'],1), round(d['inference_ms'],3))"
done
