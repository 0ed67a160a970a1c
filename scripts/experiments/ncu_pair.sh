mkdir -p gpurun_out
rm -f gpurun_out/prof_pair*.ncu-rep
NCU=/usr/local/cuda/bin/ncu
for pr in 1 0; do
  NB_TC_PAIR=$pr $NCU --set full --clock-control none --import-source on -k regex:k_conv_tc \
    -s $((128 + 8)) -c 1 -o gpurun_out/prof_pair${pr}_L9 -f python scripts/origin_fisher.py 3 > /dev/null 2>&1
  NB_TC_PAIR=$pr $NCU --set full --clock-control none -k regex:k_conv_tc \
    -s $((128 + 16)) -c 1 -o gpurun_out/prof_pair${pr}_L17 -f python scripts/origin_fisher.py 3 > /dev/null 2>&1
done
ls gpurun_out/prof_pair*
