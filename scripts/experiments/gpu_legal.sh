mkdir -p gpurun_out
nproc
timeout 900 python -m pytest tests/test_legality.py -m gpu -q -p no:cacheprovider -x -s > gpurun_out/pytest_legal.log 2>&1; echo "pytest rc=$?"; grep -E "gpu .* ms|passed|failed|Error" gpurun_out/pytest_legal.log | head -30
timeout 900 python scripts/gate_timing.py 200 0 1 2>&1 | tail -3
