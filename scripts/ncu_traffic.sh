# Per-launch DRAM traffic, duration and tensor-pipe activity of every nb200
# kernel in a short single-stream bench (metrics only: small output).
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg \
  --clock-control none --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps ${STEPS:-12} --warmup 2 --streams 1 --no-cpu-baseline --no-kernel-events --no-modes --no-peaks --no-inference \
  > gpurun_out/ncu_traffic.log 2>&1
echo "rc=$?"; wc -l gpurun_out/traffic.csv
