# register-tiled FDTD temporal blocking
set -x
for d in 22 23 24; do PF_FDTD_TB=$d timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1; done
for d in 4 22 23 24; do echo "FDTD tb=$d $(PF_FDTD_TB=$d timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
