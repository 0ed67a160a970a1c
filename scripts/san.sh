# compute-sanitizer over a small Fisher chain (tensor-core 3xF16 path and the
# SIMT path): memcheck, racecheck, synccheck, initcheck.  Summaries land in
# gpurun_out/san_<tool>_<prec>.log.
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for prec in fp32 simt; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 $S --tool $tool --print-limit 20 python scripts/san_fisher.py $prec > gpurun_out/san_${tool}_$prec.log 2>&1
    echo "$prec $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_$prec.log | tail -1)"
  done
done
