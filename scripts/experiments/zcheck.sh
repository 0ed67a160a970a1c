mkdir -p gpurun_out
nproc > gpurun_out/z.txt
python /root/repo/scripts/z_time.py >> gpurun_out/z.txt 2>&1
( time timeout 300 integration/_build/nb200_search scripts/r34_search_all_kinds.json --candidates 1000 ) >> gpurun_out/z.txt 2>&1
bash scripts/gpu_check.sh
