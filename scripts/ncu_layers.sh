# Full ncu captures of selected tcgen05 launches of one R34 origin Fisher
# evaluation (launch order: fprop L1..L32, then dgrad L32..L1).
mkdir -p gpurun_out
rm -f gpurun_out/prof_layers*.ncu-rep
for spec in "0:fprop_L1" "8:fprop_L9" "16:fprop_L17" "28:fprop_L29" "32:dgrad_L32" "36:dgrad_L28" "48:dgrad_L16" "56:dgrad_L8" "63:dgrad_L1"; do
  off=${spec%%:*}; name=${spec##*:}
  /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_conv_tc \
    -s $((128 + off)) -c 1 -o gpurun_out/prof_$name -f python scripts/origin_fisher.py 3 ${PREC:-fp32} \
    > gpurun_out/ncu_$name.log 2>&1; echo "$name rc=$?"
done
du -sh gpurun_out
