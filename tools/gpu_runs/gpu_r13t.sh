# flat beta pre-pass
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "SYRK or SYR2K or GEMM" 2>&1 | tail -2
for b in "SYRK 2048,2048" "SYR2K 2048,2048" "GEMM 512,512,512"; do
  set -- $b; echo "$1 $2 $(timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py SYRK 2048,2048 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -4
