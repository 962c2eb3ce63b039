# lo image of D from the epilogue for chained products (2MM, 3MM)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "2MM or 3MM or GEMM or SYRK or SYR2K or tensor_core or config_paths" 2>&1 | tail -2
for b in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048"; do
  set -- $b; echo "$1 $(timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py 3MM 2048,2048,2048,2048,2048 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -9
