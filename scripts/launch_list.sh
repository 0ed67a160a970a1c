# per-launch durations of one origin R34 Fisher evaluation (the 4th of
# scripts/origin_fisher.py 3) -- ncu launch list, cold-cache, serialised
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launch_list.csv python scripts/origin_fisher.py 3 ${PREC:-fp32} > /dev/null 2>&1
echo rc=$?
