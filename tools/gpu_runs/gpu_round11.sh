# GEMM 512^3 tcgen05 fixed-cost split (kernel durations under ncu launch list)
set -x
for pair in 1 0; do for d in 0 8 6 14 15; do
  echo "pair=$pair diag=$d"
  PF_TC_PAIR=$pair PF_TC_DIAG=$d timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 3 2>/dev/null | grep -E "tc_tma|tc_prescale" | cut -d, -f5,9,15 | tail -2
done; done
PF_TC_DIAG=0 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 3 2>/dev/null | grep -E "tc_tma|tc_prescale" | cut -d, -f5,9,15 | tail -2
