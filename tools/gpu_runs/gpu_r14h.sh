# pair vs single-CTA tiles with pre-split operands
set -x
for b in "2MM 2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" "CORR 2048,2048"; do
  set -- $b
  for pr in 1 0; do echo "$1 pair=$pr $(PF_TC_PAIR=$pr timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"; done
done
