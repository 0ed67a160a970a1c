# A/B of two in-tree builds (NB200_LIB): origin Fisher + bench, alternating
for i in 1 2; do
  for lib in libnb200_prev.so libnb200.so; do
    echo "== $lib"; NB200_LIB=$lib python scripts/origin_fisher.py 4 ${PREC:-fp32} | grep -E "fisher 3|conv_.*tc"
    NB200_LIB=$lib python bench.py --no-cpu-baseline --precision ${PREC:-fp32} ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('bench', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
  done
done
