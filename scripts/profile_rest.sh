# Round evidence without the default bench line: single-stream bench launch
# list, per-launch DRAM/tensor metrics, and four ncu --set full captures of
# the origin evaluation (see round_profile.sh for the launch offsets).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --streams 1 --no-cpu-baseline --no-modes --no-peaks --no-inference \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
STEPS=12 timeout 900 bash scripts/ncu_traffic.sh
rm -f gpurun_out/prof_r2_*.ncu-rep
for spec in "1:fprop_L1" "9:fprop_L9" "41:dgrad_L24" "64:dgrad_L1"; do
  off=${spec%%:*}; name=${spec##*:}
  timeout 300 $NCU --set full --clock-control none --import-source on -k regex:k_conv_tc \
    -s $((130 + off)) -c 1 -o gpurun_out/prof_r2_$name -f python scripts/origin_fisher.py 3 \
    > gpurun_out/ncu_r2_$name.log 2>&1; echo "$name rc=$?"
done
du -sh gpurun_out
