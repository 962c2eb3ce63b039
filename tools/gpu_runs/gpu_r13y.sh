set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1
PF_FDTD_TB=4 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "FDTD" 2>&1 | tail -1
for d in -1 4 0; do echo "FDTD tb=$d $(PF_FDTD_TB=$d timeout 300 python tools/profile_kernels.py FDTD-2D 2048,2048,500 stage=2 5 2>&1 | tail -1)"; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_rt -s 2 -c 1 \
   -o gpurun_out/prof_FDTD_rt python tools/profile_kernels.py FDTD-2D 2048,2048,24 stage=2 1 > /dev/null 2>&1
