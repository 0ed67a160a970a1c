# A/B of an environment setting on the bench, alternating runs:
#   ENV_A="" ENV_B="NB_SCHED_THREADS=1" bash scripts/ab_env.sh
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in "${ENV_A:-NONE=0}" "${ENV_B:-NONE=0}"; do
    env $v python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); k=d.get('kernels',{})
print('$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],3), {n: round(k[n]['ms'],1) for n in k if n.startswith('host')})"
  done
done
