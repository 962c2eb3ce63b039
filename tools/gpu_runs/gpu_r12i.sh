# GRAMSCHM barrier-free factorisation + FDTD temporal blocking: parity + timing
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM or FDTD" 2>&1 | tail -4
echo "GRAMSCHM v3 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
for tb in 1 0; do echo "FDTD tb=$tb $(PF_FDTD_TB=$tb timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/profile_kernels.py FDTD-2D 2048,2048,20 stage=2 1 2>/dev/null | python tools/ncu_list.py | tail -6
