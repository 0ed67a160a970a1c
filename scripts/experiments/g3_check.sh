mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_tc_modes.py tests/test_r34_parity.py tests/test_sharded.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pt.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pt.log
[ $rc -ne 0 ] && grep -E "^FAILED|Timeout" gpurun_out/pt.log | head -3
for h in 0 1; do
  NB_TC_HALO=$h timeout 60 python scripts/origin_fisher.py 3 fp32 > gpurun_out/of.txt 2>&1 || { echo "origin halo $h FAILED/timeout"; continue; }
  echo "halo $h origin $(sed -n 3p gpurun_out/of.txt)"
  for idx in 196 206 214 226 246 254; do
    NB_TC_HALO=$h NB_TC_TRACE=$idx timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1 || break
    echo -n "  $idx "; python scripts/trace_sum.py nb_tc_trace.txt nb_tc_ctas.txt | sed 's/ # bn=\([0-9]*\).*tiles=\([0-9]*\) kblocks.tile=\([0-9]*\) | stages [0-9]* period med/ bn\1 t\2 k\3 per/; s/ctas/c/; s/conv lat med/conv/' | cut -c1-140
  done
  NB_TC_HALO=$h timeout 200 python bench.py --steps 20 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('  bench', round(d['value'],1), round(d['e2e']['value'],1), r['kernel'], round(r['achieved'],1), round(d['inference_ms'],3))"
done
