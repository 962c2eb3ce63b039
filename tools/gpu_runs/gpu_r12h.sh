# pre-split lo operands (PF_TC_PRESPLIT=1) vs in-kernel converters
set -x
mkdir -p gpurun_out
PF_TC_PRESPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GEMM or 2MM or 3MM or SYRK or SYR2K or tensor_core" 2>&1 | tail -3
for b in "2MM 2048,2048,2048,2048" "3MM 2048,2048,2048,2048,2048" "SYRK 2048,2048" "SYR2K 2048,2048" "GEMM 512,512,512"; do
  set -- $b
  for ps in 0 1; do
    echo "$1 presplit=$ps $(PF_TC_PRESPLIT=$ps timeout 120 python tools/profile_kernels.py $1 $2 stage=2 10 2>&1 | tail -1)"
  done
done
PF_TC_PRESPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 2 2>/dev/null | python tools/ncu_list.py | tail -8
