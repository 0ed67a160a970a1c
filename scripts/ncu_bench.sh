# ncu evidence for the bench workload (1 GPU): launch list + one full capture.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_conv_tc -s ${SKIP:-120} -c ${COUNT:-4} \
  -o gpurun_out/prof_tc -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out
