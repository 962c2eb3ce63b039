# 3DCONV cp.async ring candidate (PF_C3=9) vs direct form; split pass timing
set -x
PF_C3=9 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "3DCONV" 2>&1 | tail -3
for m in 9 0; do echo "3DCONV mode=$m $(PF_C3=$m timeout 120 python tools/profile_kernels.py 3DCONV 256,256,256 stage=2 10 2>&1 | tail -1)"; done
echo "2MM $(timeout 120 python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 10 2>&1 | tail -1)"
echo "3MM $(timeout 120 python tools/profile_kernels.py 3MM 2048,2048,2048,2048,2048 stage=2 10 2>&1 | tail -1)"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py 2MM 2048,2048,2048,2048 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -6
