mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "tc_" > gpurun_out/pair_tc.log 2>&1; echo "tc tests rc=$?"; tail -3 gpurun_out/pair_tc.log
timeout 120 python scripts/origin_fisher.py 4 > gpurun_out/of_pair.log 2>&1; echo "of rc=$?"; tail -12 gpurun_out/of_pair.log
NB_TC_PAIR=0 timeout 120 python scripts/origin_fisher.py 4 2>&1 | grep -E "fisher 3|conv_"
NB_TC_PAIR_BN=256 timeout 120 python scripts/origin_fisher.py 4 2>&1 | grep -E "fisher 3|conv_"
timeout 120 python scripts/origin_fisher.py 4 tf32 2>&1 | grep -E "fisher 3|conv_"
NB_TC_PAIR=0 timeout 120 python scripts/origin_fisher.py 4 tf32 2>&1 | grep -E "fisher 3|conv_"
