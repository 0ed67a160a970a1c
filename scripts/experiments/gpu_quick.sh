mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 120 python scripts/origin_fisher.py 4 2>&1 | grep -E "fisher 3|conv_"
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench64.log 2>&1; python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench64.log").read().strip().splitlines()[-1])
print(round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "ms/step", round(d["ms_per_step"],3), "inf", round(d["inference_ms"],3), {k:round(v["ms"],1) for k,v in d["kernels"].items()})
PY
