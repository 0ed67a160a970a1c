# fprop tail epilogue (launch 139, BN=128): chunk timeline under debug bits
for dbg in 0 2097152 6291456 10485760 14680064; do
  echo "dbg=$dbg"
  NB_TC_DEBUG=$dbg NB_TC_TRACE=139 timeout 60 python scripts/origin_fisher.py 3 fp32 > /dev/null 2>&1
  python scripts/experiments/epi_trace.py nb_tc_trace.txt
done
