# depthwise fprop: output columns per thread (NB_DW3_OWB) on the C5 depthwise points
for owb in ${OWBS:-1 2 4}; do
  echo "OWB=$owb"
  NB_DW3_OWB=$owb SWEEP_GROUPS=dw timeout 300 python scripts/sweep_c5.py 2>&1 | grep "^|" | grep -v "C@HW\|---" | cut -d"|" -f2-14
done
