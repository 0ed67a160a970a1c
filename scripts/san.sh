mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for tool in initcheck memcheck racecheck; do
  timeout 600 $S --tool $tool --print-limit 20 python scripts/san_fisher.py simt > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -5 gpurun_out/san_$tool.log
done
