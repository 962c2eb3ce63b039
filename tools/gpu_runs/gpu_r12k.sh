# FDTD temporal blocking, float4 form: parity (forced on) + timing
set -x
PF_FDTD_TB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -4
for tb in 1 0; do echo "FDTD tb=$tb $(PF_FDTD_TB=$tb timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
echo "GRAMSCHM v2 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 3 2>&1 | tail -1)"
