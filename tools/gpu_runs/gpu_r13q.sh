# FDTD temporal blocking: load-then-compute phases with shuffled neighbours
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1
PF_FDTD_TB=8 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1
for d in 4 8 0; do echo "FDTD tb=$d $(PF_FDTD_TB=$d timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
