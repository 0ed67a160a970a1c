# GPU tests, then the default bench and A/B variants given as env strings
mkdir -p gpurun_out; rm -f gpurun_out/ab_quick.txt
[ -n "$SKIP_TESTS" ] || timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_quick.txt
tail -3 gpurun_out/ab_tests.log >> gpurun_out/ab_quick.txt
for env in "X=0" "$@"; do
  tag=$(echo "$env" | tr ' =' '__')
  env $env timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_$tag.log 2>&1
  python - "$env" "gpurun_out/ab_$tag.log" >> gpurun_out/ab_quick.txt <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"], 1), round(d["e2e"]["value"], 1), round(d["roofline"]["achieved"], 1),
      round(d["inference_ms"], 3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
