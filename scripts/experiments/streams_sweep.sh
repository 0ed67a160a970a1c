mkdir -p gpurun_out
for s in ${STREAMS:-2 4 6 8}; do
  python bench.py --no-cpu-baseline --streams $s > gpurun_out/ss.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ss.log').read().strip().splitlines()[-1]); print('streams $s', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
