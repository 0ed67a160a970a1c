# Round evidence in one call: default bench JSON, launch list of a
# single-stream bench, per-launch DRAM/tensor metrics, and full ncu captures
# of four tcgen05 launches of the origin evaluation (the third of
# scripts/origin_fisher.py 3; 65 k_conv_tc launches per evaluation: the
# im2col stem, fprop of layers 1-32, dgrad of layers 32..1).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-300
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --streams 1 --no-cpu-baseline --no-modes --no-peaks --no-inference \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
STEPS=12 bash scripts/ncu_traffic.sh
rm -f gpurun_out/prof_r2_*.ncu-rep
for spec in "1:fprop_L1" "9:fprop_L9" "41:dgrad_L24" "64:dgrad_L1"; do
  off=${spec%%:*}; name=${spec##*:}
  timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_conv_tc \
    -s $((130 + off)) -c 1 -o gpurun_out/prof_r2_$name -f python scripts/origin_fisher.py 3 \
    > gpurun_out/ncu_r2_$name.log 2>&1; echo "$name rc=$?"
done
du -sh gpurun_out
