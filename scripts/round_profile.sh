# Round evidence in one call: default bench JSON, launch list of a
# single-stream bench, per-launch DRAM/tensor metrics, and full ncu captures
# of a BN=128 dgrad and a BN=64 fprop launch of the origin evaluation.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --streams 1 --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
STEPS=12 bash scripts/ncu_traffic.sh
rm -f gpurun_out/prof_r1c_*.ncu-rep
for spec in "0:fprop_L1" "8:fprop_L9" "40:dgrad_L24" "63:dgrad_L1"; do
  off=${spec%%:*}; name=${spec##*:}
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_conv_tc \
    -s $((128 + off)) -c 1 -o gpurun_out/prof_r1c_$name -f python scripts/origin_fisher.py 3 \
    > gpurun_out/ncu_r1c_$name.log 2>&1; echo "$name rc=$?"
done
du -sh gpurun_out
