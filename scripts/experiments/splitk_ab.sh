# split-K epilogue: launch list share (ncu) and bench
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:splitk --csv --log-file gpurun_out/sk.csv python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/sk.csv')) if len(r)>10 and r[-3]=='gpu__time_duration.sum']
v=[float(r[-1]) for r in rows]
print('splitk launches', len(v), 'avg', sum(v)/max(1,len(v)), 'unit', rows[0][-2] if rows else '')
P
for i in 1 2; do
  timeout 200 python bench.py --steps 40 --warmup 5 --no-modes --no-cpu-baseline --no-peaks > gpurun_out/bench.log 2>&1
  echo "$(tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('bench', round(d['value'],1), 'dgrad', round(r['achieved'],1))")"
done
