# ordered split-K (split 0 stores, flag, others add): parity + timings
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GEMM or 2MM or 3MM or SYRK or SYR2K or CORR or COVAR or tensor_core or config_paths" 2>&1 | tail -3
for b in "GEMM 512,512,512" "GEMM 1024,1024,1024" "CORR 2048,2048" "COVAR 2048,2048" "2MM 2048,2048,2048,2048"; do
  set -- $b; echo "$1 $2 $(timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py GEMM 512,512,512 stage=2 2 2>/dev/null | python tools/ncu_list.py | tail -3
