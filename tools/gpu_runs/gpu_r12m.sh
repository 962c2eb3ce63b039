# GRAMSCHM per-column lookahead for the critical panel; FDTD blocking depth sweep
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "GRAMSCHM or FDTD" 2>&1 | tail -3
for d in 8 2; do PF_FDTD_TB=$d timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1; done
echo "GRAMSCHM v4 $(timeout 300 python tools/profile_kernels.py GRAMSCHM 2048,2048 stage=2,vec=1 5 2>&1 | tail -1)"
for d in 4 8 2 0; do echo "FDTD tb=$d $(PF_FDTD_TB=$d timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
