# origin R34 Fisher (single stream) under two environments, alternating
for i in 1 2; do
  for v in "${ENV_A:-NONE=0}" "${ENV_B:-NONE=0}"; do
    echo "== $v"; env $v python scripts/origin_fisher.py 4 ${PREC:-fp32} | grep -E "fisher 3|conv_|split|head|reduce"
  done
done
