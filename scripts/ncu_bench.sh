# ncu evidence for the bench workload (1 GPU): launch list of a single-stream
# bench (the device time of every kernel), then one full capture per major
# tcgen05 variant.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps ${STEPS:-32} --warmup 4 --streams 1 --no-cpu-baseline \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "launches rc=$?"
