# A/B of two in-tree builds (NB200_LIB) on the bench, alternating runs.
mkdir -p gpurun_out
for i in 1 2 3; do
  for lib in libnb200_prev.so libnb200.so; do
    NB200_LIB=$lib python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$lib', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'inf', round(d['inference_ms'],3))"
  done
done
for lib in libnb200_prev.so libnb200.so; do NB200_LIB=$lib python scripts/origin_fisher.py 4 | grep -E "fisher 3"; done
